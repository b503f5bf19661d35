// xfer.cu — K6: the attention -> MoE dispatch and MoE -> attention combine
// inside one NVLink/NVSwitch box, as peer-memory kernels.
//
// The reference only prices this exchange (src/comm.cpp; "No bytes move",
// include/moesim/comm.hpp:11-14).  Its semantics are kept:
//   * token ownership on the attention side: even split, remainder to the lowest
//     instance ids (comm.cpp:76-81, janus_shard_tokens);
//   * gating is MoE-side, so every MoE instance receives every token's full
//     activation (comm.hpp:12-14; test_comm.cpp:35-64) — here with its routing
//     (top-k ids) and gate weights, which the scheduler on each MoE GPU needs
//     (it runs replicated on identical inputs);
//   * the MoE side's per-token aggregation "plays the all-reduce role" on the
//     way back (comm.hpp:96-98): each MoE GPU pushes its partial sums for the
//     tokens an attention GPU owns; the owner adds the M partials in a fixed
//     instance order.
//
// Transport: every rank allocates one exchange region (identical layout on all
// ranks, CUDA IPC handle exchanged once); kernels store straight into peers'
// regions over NVLink (P2P), fused with the copy / combine math, then publish
// with a system-scope release store of the step's epoch into the receiver's
// flag.  Receivers wait with acquire loads (bounded: a stuck peer sets an error
// flag instead of hanging the GPU).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "internal.h"

namespace janus {
namespace {

constexpr int kMaxPeers = 16;
constexpr unsigned long long kWaitTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s

struct PeerPtrs {
  unsigned char *base[kMaxPeers];
};

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Shard rule (comm.cpp:76-81) on the device.
__device__ __forceinline__ void shard_of(long long T, int A, long long t, int &a, long long &first) {
  const long long base = T / A, rem = T % A;
  const long long big = rem * (base + 1);
  if (t < big) {
    a = (int)(t / (base + 1));
    first = (long long)a * (base + 1);
  } else {
    a = (int)(rem + (t - big) / base);
    first = big + (long long)(a - rem) * base;
  }
}

// Grid-wide completion: the last block to finish publishes the flags.
// Every thread fences its own peer stores (system scope) before the block
// counts itself done; the last block fences again (acquire side) before it
// publishes.
__device__ __forceinline__ bool last_block(unsigned *counter) {
  __shared__ bool last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    last = prev == gridDim.x - 1;
    if (last) {
      __threadfence_system();
      *counter = 0;  // re-arm for the next step (stream-ordered)
    }
  }
  __syncthreads();
  return last;
}

// Attention rank `a`: push this shard's rows, routing and gate weights into
// every MoE rank's receive buffers at the shard's token offset, then raise
// flag_dispatch[a] = epoch on each MoE rank.
// Destinations: the M MoE ranks' IPC regions (P2P), or the one multicast
// mapping (NVLS: the switch replicates each store to every rank).
struct DispatchDst {
  unsigned char *base[kMaxPeers];
  int n;
  size_t x_off, ex_off, gw_off;
};

__global__ void dispatch_kernel(DispatchDst dst, PeerPtrs peers, int M, int moe0, int a,
                                const uint4 *__restrict__ x, const int32_t *__restrict__ ex,
                                const float *__restrict__ gw, long long first, long long Ta,
                                int vec, int k, XferLayout L, unsigned long long epoch,
                                unsigned *counter) {
  const long long nx = Ta * vec, ns = Ta * k;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // 4 independent 16-B chunks per thread per round: 4 loads in flight, then
  // 4*M posted peer stores.
  constexpr int U = 4;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < nx;
       i0 += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i < nx) v[u] = __ldg(x + i);
    }
    for (int g = 0; g < dst.n; ++g) {
      uint4 *d = reinterpret_cast<uint4 *>(dst.base[g] + dst.x_off) + first * vec;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long i = i0 + u * stride;
        if (i < nx) d[i] = v[u];
      }
    }
  }
  // routing rows (absent when the MoE side gates: it computes them from x)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; ex && i < ns;
       i += stride) {
    const int32_t e = __ldg(ex + i);
    const float w = __ldg(gw + i);
    for (int g = 0; g < dst.n; ++g) {
      reinterpret_cast<int32_t *>(dst.base[g] + dst.ex_off)[first * k + i] = e;
      reinterpret_cast<float *>(dst.base[g] + dst.gw_off)[first * k + i] = w;
    }
  }
  if (last_block(counter) && threadIdx.x < M) {
    unsigned long long *flag =
        reinterpret_cast<unsigned long long *>(peers.base[moe0 + threadIdx.x] + L.flag_dispatch_off) +
        a;
    st_release_sys(flag, epoch);
  }
}

// Wait until flags[0..n) all reach epoch (one warp).  On timeout, record an
// error instead of hanging.
__global__ void wait_flags_kernel(const unsigned long long *flags, int n,
                                  unsigned long long epoch, int *err) {
  const int lane = threadIdx.x;
  const unsigned long long t0 = gtimer();
  bool done = false;
  while (!done) {
    bool mine = true;
    for (int i = lane; i < n; i += 32) mine = mine && ld_acquire_sys(flags + i) >= epoch;
    done = __all_sync(0xffffffffu, mine);
    if (!done) {
      if (gtimer() - t0 > kWaitTimeoutNs) {
        if (lane == 0) atomicExch(err, 1);
        return;
      }
      __nanosleep(200);
    }
  }
}

// MoE rank g: partial[t] = sum over this instance's slots of w * y (fixed j
// order, fp32), stored as bf16 straight into the owning attention rank's
// part_recv[g][t - first]; then raise flag_combine[g] = epoch there.
__global__ void combine_push_kernel(PeerPtrs peers, int A, int g, const __nv_bfloat16 *__restrict__ y,
                                    const int32_t *__restrict__ slot_row,
                                    const int32_t *__restrict__ slot_inst,
                                    const float *__restrict__ gw, long long T, int k, int d_h,
                                    long long ta_max, XferLayout L, size_t part_off,
                                    unsigned long long epoch, unsigned *counter) {
  const int vec = d_h / 8;
  const long long n = T * vec;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long t = idx / vec;
    const int c = (int)(idx % vec);
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int j = 0; j < k; ++j) {
      const long long s = t * k + j;
      if (__ldg(slot_inst + s) != g) continue;
      const float w = __ldg(gw + s);
      const uint4 v =
          __ldg(reinterpret_cast<const uint4 *>(y + (size_t)__ldg(slot_row + s) * d_h) + c);
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        acc[2 * e] += w * f.x;
        acc[2 * e + 1] += w * f.y;
      }
    }
    uint4 o;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
    int a;
    long long first;
    shard_of(T, A, t, a, first);
    uint4 *dst = reinterpret_cast<uint4 *>(peers.base[a] + part_off) +
                 ((long long)g * ta_max + (t - first)) * vec;
    dst[c] = o;
  }
  if (last_block(counter) && threadIdx.x < A) {
    unsigned long long *flag =
        reinterpret_cast<unsigned long long *>(peers.base[threadIdx.x] + L.flag_combine_off) + g;
    st_release_sys(flag, epoch);
  }
}

// Attention rank: out[t] = sum_g part_recv[g][t] in instance order (fp32).
__global__ void reduce_partials_kernel(const __nv_bfloat16 *__restrict__ part, int M,
                                       long long Ta, long long ta_max, int d_h,
                                       __nv_bfloat16 *__restrict__ out) {
  const int vec = d_h / 8;
  const long long n = Ta * vec;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int g = 0; g < M; ++g) {
      const uint4 v = reinterpret_cast<const uint4 *>(part + (size_t)g * ta_max * d_h)[idx];
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        acc[2 * e] += f.x;
        acc[2 * e + 1] += f.y;
      }
    }
    uint4 o;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
    reinterpret_cast<uint4 *>(out)[idx] = o;
  }
}

// MoE rank g (multicast path): its partial sums are already in its own backing
// (K5 with the instance filter); publish flag_combine[g] = epoch on every
// attention rank.  The release store is cumulative over the preceding kernel's
// writes (stream order), so the switch-side reads see them.
__global__ void signal_combine_kernel(PeerPtrs peers, int A, int g, XferLayout L,
                                      unsigned long long epoch) {
  __threadfence_system();
  if (threadIdx.x < A) {
    unsigned long long *flag =
        reinterpret_cast<unsigned long long *>(peers.base[threadIdx.x] + L.flag_combine_off) + g;
    st_release_sys(flag, epoch);
  }
}

// Attention rank (multicast path): out[t] = sum over every rank's backing of
// part[first + t], reduced by the NVSwitch (multimem.ld_reduce, fp32
// accumulation, one rounding to bf16).  Ranks that hold no partial for a row
// contribute zeros.
__global__ void reduce_mc_kernel(const uint4 *__restrict__ mc_part, long long n,
                                 uint4 *__restrict__ out) {
  constexpr int U = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i < n)
        asm volatile(
            "multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
            : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
            : "l"(mc_part + i)
            : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i < n) out[i] = v[u];
    }
  }
}

int grid_for(long long work, int per_block = 256) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long b = (work + per_block - 1) / per_block;
  return (int)std::max<long long>(1, std::min<long long>(b, (long long)sms * 8));
}

PeerPtrs peer_ptrs(const XferState &x) {
  PeerPtrs p{};
  for (int r = 0; r < x.world && r < kMaxPeers; ++r)
    p.base[r] = static_cast<unsigned char *>(x.peer_base[r]);
  return p;
}

}  // namespace

XferLayout xfer_layout(int A, int M, long long T_max, int d_h, int k) {
  XferLayout L{};
  auto up = [](size_t v) { return (v + 255) & ~size_t(255); };
  const long long ta_max = (T_max + A - 1) / A;
  size_t o = 0;
  L.flag_dispatch_off = o;
  o = up(o + 8 * (size_t)A);
  L.flag_combine_off = o;
  o = up(o + 8 * (size_t)M);
  const size_t slot0 = o;
  L.x_off = o;
  o = up(o + (size_t)T_max * d_h * 2);
  L.ex_off = o;
  o = up(o + (size_t)T_max * k * 4);
  L.gw_off = o;
  o = up(o + (size_t)T_max * k * 4);
  L.part_off = o;
  o = up(o + (size_t)M * ta_max * d_h * 2);
  L.slot_stride = o - slot0;
  L.bytes = o + L.slot_stride;
  L.ta_max = ta_max;
  return L;
}

cudaError_t launch_dispatch(const XferState &x, const void *d_x, const int32_t *d_ex,
                            const float *d_gw, long long T, unsigned long long epoch,
                            cudaStream_t s) {
  const int a = x.rank;
  long long first = 0, Ta = 0;
  {
    const long long base = T / x.A, rem = T % x.A;
    Ta = base + (a < rem ? 1 : 0);
    first = a * base + std::min<long long>(a, rem);
  }
  const int vec = x.d_h / 8;
  DispatchDst dst{};
  if (x.mc) {  // one store per element; the NVSwitch replicates it to every rank
    const size_t so = xfer_slot(epoch) * x.mslot;
    dst.base[0] = reinterpret_cast<unsigned char *>(x.mc_va);
    dst.n = 1;
    dst.x_off = x.mx_off + so;
    dst.ex_off = x.mex_off + so;
    dst.gw_off = x.mgw_off + so;
  } else {
    const size_t so = xfer_slot(epoch) * x.L.slot_stride;
    for (int g = 0; g < x.M; ++g)
      dst.base[g] = static_cast<unsigned char *>(x.peer_base[x.moe0 + g]);
    dst.n = x.M;
    dst.x_off = x.L.x_off + so;
    dst.ex_off = x.L.ex_off + so;
    dst.gw_off = x.L.gw_off + so;
  }
  dispatch_kernel<<<grid_for(std::max<long long>(Ta * vec, 1)), 256, 0, s>>>(
      dst, peer_ptrs(x), x.M, x.moe0, a, reinterpret_cast<const uint4 *>(d_x), d_ex, d_gw, first, Ta,
      vec, x.k, x.L, epoch, x.counter);
  return cudaGetLastError();
}

cudaError_t launch_wait(const XferState &x, bool dispatch_flags, unsigned long long epoch,
                        cudaStream_t s) {
  unsigned char *base = static_cast<unsigned char *>(x.local);
  const unsigned long long *flags = reinterpret_cast<const unsigned long long *>(
      base + (dispatch_flags ? x.L.flag_dispatch_off : x.L.flag_combine_off));
  wait_flags_kernel<<<1, 32, 0, s>>>(flags, dispatch_flags ? x.A : x.M, epoch, x.err);
  return cudaGetLastError();
}

cudaError_t launch_combine_push(const XferState &x, const void *y, const int32_t *slot_row,
                                const int32_t *slot_inst, const float *gw, long long T,
                                unsigned long long epoch, cudaStream_t s) {
  const int g = x.rank - x.moe0;
  combine_push_kernel<<<grid_for(std::max<long long>(T * (x.d_h / 8), 1)), 256, 0, s>>>(
      peer_ptrs(x), x.A, g, reinterpret_cast<const __nv_bfloat16 *>(y), slot_row, slot_inst, gw,
      T, x.k, x.d_h, x.L.ta_max, x.L, x.L.part_off + xfer_slot(epoch) * x.L.slot_stride, epoch,
      x.counter);
  return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const XferState &x, void *d_out, long long Ta,
                                   unsigned long long epoch, cudaStream_t s) {
  if (Ta == 0) return cudaSuccess;
  const unsigned char *base = static_cast<const unsigned char *>(x.local);
  reduce_partials_kernel<<<grid_for(Ta * (x.d_h / 8)), 256, 0, s>>>(
      reinterpret_cast<const __nv_bfloat16 *>(base + x.L.part_off +
                                               xfer_slot(epoch) * x.L.slot_stride),
      x.M, Ta, x.L.ta_max, x.d_h,
      reinterpret_cast<__nv_bfloat16 *>(d_out));
  return cudaGetLastError();
}

cudaError_t launch_signal_combine(const XferState &x, unsigned long long epoch, cudaStream_t s) {
  signal_combine_kernel<<<1, 32, 0, s>>>(peer_ptrs(x), x.A, x.rank - x.moe0, x.L, epoch);
  return cudaGetLastError();
}

cudaError_t launch_reduce_mc(const XferState &x, void *d_out, long long first, long long Ta,
                             unsigned long long epoch, cudaStream_t s) {
  if (Ta == 0) return cudaSuccess;
  const long long vec = x.d_h / 8, n = Ta * vec;
  const uint4 *part =
      reinterpret_cast<const uint4 *>(x.mc_va + x.mpart_off + xfer_slot(epoch) * x.mslot) +
      first * vec;
  reduce_mc_kernel<<<grid_for((n + 3) / 4), 256, 0, s>>>(part, n, reinterpret_cast<uint4 *>(d_out));
  return cudaGetLastError();
}

}  // namespace janus
