// xfer.cu — K6: the attention -> MoE dispatch and MoE -> attention combine
// inside one NVLink/NVSwitch box, as peer-memory kernels.
//
// The reference only prices this exchange (src/comm.cpp; "No bytes move",
// include/moesim/comm.hpp:11-14).  Its semantics are kept:
//   * token ownership on the attention side: even split, remainder to the lowest
//     instance ids (comm.cpp:76-81, janus_shard_tokens);
//   * gating is MoE-side, so every MoE instance receives every token's full
//     activation (comm.hpp:12-14; test_comm.cpp:35-64) — the broadcast
//     transports (P2P, NVLS) — here with its routing (top-k ids) and gate
//     weights, which the scheduler on each MoE GPU needs (it runs replicated on
//     identical inputs);
//   * routed transport (north_star's "permute into per-GPU buffers"): with the
//     routing known on the attention side, each attention GPU runs the same K1
//     over the whole step's routing and sends a row only to the MoE GPUs its
//     slots were scheduled on — the per-destination traffic StepTraffic counts
//     (comm.hpp:20-39) restricted to the instances that need the token, as the
//     one-to-one plan's spread phase does (comm.cpp:155-160).  The layout is
//     the replicated K1/K2 output, so no count exchange;
//   * the MoE side's per-token aggregation "plays the all-reduce role" on the
//     way back (comm.hpp:96-98): each MoE GPU pushes its partial sums for the
//     tokens an attention GPU owns (K5 in push mode, ffn.cu); the owner adds the
//     partials in a fixed instance order.
//
// Transport: every rank allocates one exchange region (identical layout on all
// ranks, CUDA IPC handle exchanged once, or raw pointers in one process); kernels
// store straight into peers' regions over NVLink (P2P), fused with the copy /
// combine math, then publish with a system-scope release store of the step's
// epoch into the receiver's flag.  Receivers wait with acquire loads (bounded:
// a stuck peer sets an error word instead of hanging the GPU, and the step's
// later kernels skip their work).  A failed MoE step (unknown expert) travels
// to the attention ranks in an error slot written before the combine flag.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace janus {
namespace {

constexpr int kMaxPeers = 16;
static_assert(kMaxPeers == kPushMaxPeers, "peer tables");

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

// Grid-wide completion: the last block to finish publishes the flags.
// Every thread fences its own peer stores (system scope) before the block
// counts itself done; the last block fences again (acquire side) before it
// publishes.  Each kernel kind and epoch slot has its own counter, so kernels
// of different kinds (or of two steps in flight) never share one.
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

// Attention rank `a`, broadcast transports: push this shard's rows, routing
// and gate weights into every MoE rank's receive buffers at the shard's token
// offset, then raise flag_dispatch[a] = epoch on each MoE rank.
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

// Routed transport, attention rank `a`: its shard's routing (ids + gate
// weights, 8 B per slot) into every rank of the box — the MoE ranks schedule
// and combine with it, the other attention ranks run the same K1 on it — then
// flag_route[a] = epoch everywhere.
__global__ void route_push_kernel(PeerPtrs peers, int world, int a, const int32_t *__restrict__ ex,
                                  const float *__restrict__ gw, long long first, long long ns,
                                  int k, size_t ex_off, size_t gw_off, XferLayout L,
                                  unsigned long long epoch, unsigned *counter) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ns; i += stride) {
    const int32_t e = __ldg(ex + i);
    const float w = __ldg(gw + i);
    for (int r = 0; r < world; ++r) {
      reinterpret_cast<int32_t *>(peers.base[r] + ex_off)[first * k + i] = e;
      reinterpret_cast<float *>(peers.base[r] + gw_off)[first * k + i] = w;
    }
  }
  if (last_block(counter) && threadIdx.x < world) {
    unsigned long long *flag =
        reinterpret_cast<unsigned long long *>(peers.base[threadIdx.x] + L.flag_route_off) + a;
    st_release_sys(flag, epoch);
  }
}

// Routed transport, attention rank `a`: one warp per owned token t.  Lanes
// j < k read the instance K1 scheduled slot (t, j) on and OR them into t's
// destination mask; the row is loaded once and stored only into those MoE
// ranks' receive buffers (at its token position, so the MoE side's permute
// reads it exactly where a broadcast would have put it).  The mask is kept
// for the combine.  A rejected step (K1 status) sends nothing but still
// publishes, so no MoE rank waits for it.
__global__ void routed_dispatch_kernel(PeerPtrs peers, int M, int moe0, int a,
                                       const uint4 *__restrict__ x,
                                       const int32_t *__restrict__ inst,
                                       const int32_t *__restrict__ status, long long first,
                                       long long Ta, int vec, int k, size_t x_off,
                                       uint32_t *__restrict__ dmask, int *err, XferLayout L,
                                       unsigned long long epoch, unsigned *counter) {
  const int lane = threadIdx.x & 31;
  const long long warp0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const bool ok = status == nullptr || status[0] == JANUS_OK;
  if (!ok && blockIdx.x == 0 && threadIdx.x == 0) {  // this rank's own K1 rejected the step
    if (atomicCAS(err + kErrStatus, 0, status[0]) == 0) err[kErrBad] = status[1];
  }
  constexpr int U = 4;
  for (long long t = warp0; t < Ta; t += nwarps) {
    uint32_t bit = 0;
    for (int j = lane; ok && j < k; j += 32) {
      const int g = __ldg(inst + (first + t) * k + j);
      if (g >= 0 && g < 32) bit |= 1u << g;
    }
    const uint32_t mask = __reduce_or_sync(0xffffffffu, bit);  // 0: nothing sent, zeros back
    if (lane == 0) dmask[t] = mask;
    const uint4 *src = x + t * vec;
    for (int c0 = lane; mask && c0 < vec; c0 += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + 32 * u < vec) v[u] = __ldg(src + c0 + 32 * u);
      for (uint32_t m = mask; m; m &= m - 1) {
        const int g = __ffs(m) - 1;
        uint4 *d = reinterpret_cast<uint4 *>(peers.base[moe0 + g] + x_off) + (first + t) * vec;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + 32 * u < vec) d[c0 + 32 * u] = v[u];
      }
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
// error instead of hanging.  errs (combine waits): the MoE ranks' {status,
// bad} slots of this epoch, read after the acquire of the same rank's flag;
// the first failure is kept (sticky) for janus_xfer_check.  err[kErrSkip]
// tells the step's later kernels whether to skip.
__global__ void wait_flags_kernel(const unsigned long long *flags, int n,
                                  unsigned long long epoch, const int2 *errs, int *err, int kind,
                                  unsigned long long timeout_ns, int skip) {
  const int lane = threadIdx.x;
  const unsigned long long t0 = gtimer();
  bool done = false;
  while (!done) {
    bool mine = true;
    for (int i = lane; i < n; i += 32)
      mine = mine && (i == skip || ld_acquire_sys(flags + i) >= epoch);
    done = __all_sync(0xffffffffu, mine);
    if (!done) {
      if (gtimer() - t0 > timeout_ns) {
        if (lane == 0) {
          atomicExch(err + kErrTimeout, 1);
          if (atomicCAS(err + kErrStatus, 0, JANUS_EPEER) == 0) err[kErrBad] = 0;
          err[kErrSkip + kind] = 1;
        }
        return;
      }
      __nanosleep(200);
    }
  }
  int2 mine_err = make_int2(0, 0);
  if (errs)
    for (int i = lane; i < n; i += 32) {
      const unsigned long long u = *reinterpret_cast<const volatile unsigned long long *>(errs + i);
      const int2 v = make_int2((int)(u & 0xffffffffu), (int)(u >> 32));
      if (v.x != JANUS_OK && mine_err.x == JANUS_OK) mine_err = v;
    }
  const unsigned bad = __ballot_sync(0xffffffffu, mine_err.x != JANUS_OK);
  if (bad && lane == __ffs(bad) - 1) {
    if (atomicCAS(err + kErrStatus, 0, mine_err.x) == 0) err[kErrBad] = mine_err.y;
  }
  if (lane == 0) err[kErrSkip + kind] = bad ? 1 : 0;
}

// MoE rank g: its partial sums of this epoch landed (the K5 push kernel ran
// before on the stream, or wrote its multicast backing); publish the step's
// status into every attention rank's error slot, then flag_combine[g] = epoch
// there.  The release store is cumulative over the preceding kernel's writes
// (stream order), so the owner's reads see them.
__global__ void signal_combine_kernel(PeerPtrs peers, int A, int g, XferLayout L, size_t err_off,
                                      const int32_t *__restrict__ status, int *own_err,
                                      unsigned long long epoch) {
  __threadfence_system();
  const int2 st = status ? make_int2(status[0], status[1]) : make_int2(0, 0);
  if (threadIdx.x == 0 && st.x != JANUS_OK) {  // keep it on this rank too
    if (atomicCAS(own_err + kErrStatus, 0, st.x) == 0) own_err[kErrBad] = st.y;
  }
  if (threadIdx.x < A) {
    *reinterpret_cast<volatile unsigned long long *>(peers.base[threadIdx.x] + err_off +
                                                     8 * (size_t)g) =
        (unsigned long long)(unsigned)st.x | ((unsigned long long)(unsigned)st.y << 32);
    __threadfence_system();
    unsigned long long *flag =
        reinterpret_cast<unsigned long long *>(peers.base[threadIdx.x] + L.flag_combine_off) + g;
    st_release_sys(flag, epoch);
  }
}

// Attention rank: out[t] = sum_g part_recv[g][t] in instance order (fp32).
// Routed: only the instances in t's destination mask pushed a partial.
// A failed step (err[kErrSkip]) yields zeros.
__global__ void reduce_partials_kernel(const __nv_bfloat16 *__restrict__ part, int M,
                                       long long Ta, long long ta_max, int d_h,
                                       const uint32_t *__restrict__ dmask, const int *skip,
                                       __nv_bfloat16 *__restrict__ out) {
  const int vec = d_h / 8;
  const long long n = Ta * vec;
  const bool zero = *skip != 0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    uint32_t mask = zero ? 0u : (dmask ? __ldg(dmask + idx / vec) : (M >= 32 ? ~0u : (1u << M) - 1u));
    for (; mask; mask &= mask - 1) {
      const int g = __ffs(mask) - 1;
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

// Attention rank (multicast path): out[t] = sum over every rank's backing of
// part[first + t], reduced by the NVSwitch (multimem.ld_reduce, fp32
// accumulation, one rounding to bf16).  Ranks that hold no partial for a row
// contribute zeros.
__global__ void reduce_mc_kernel(const uint4 *__restrict__ mc_part, long long n, const int *skip,
                                 uint4 *__restrict__ out) {
  constexpr int U = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const bool zero = *skip != 0;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      v[u] = make_uint4(0, 0, 0, 0);
      if (i < n && !zero)
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

void shard_host(const XferState &x, long long T, long long &first, long long &Ta) {
  const long long base = T / x.A, rem = T % x.A;
  Ta = base + (x.rank < rem ? 1 : 0);
  first = x.rank * base + std::min<long long>(x.rank, rem);
}

unsigned *counter_for(const XferState &x, int kind, unsigned long long epoch) {
  return x.counter + kXferSlots * kind + xfer_slot(epoch);
}

}  // namespace

// Grid of a dispatch-side exchange kernel, which runs beside this GPU's MoE
// kernels in the MoE-only box (the next step's rows move while this step's
// grouped GEMMs run): a third of the SMs.  (The owner's reduce stays on the
// full grid: it is on the step's critical path — capped, the combine went
// from 27 to 197 us.)  Its CTAs co-reside with the GEMM's one
// CTA per SM; on every SM they slowed every tile pair (4-GPU box: 8.2 M ->
// 8.8 M tok/s/GPU with 40-80 dispatch CTAs instead of the full grid, measured).
int side_grid(long long work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // JANUS_DISPATCH_CTAS: tuning override of the measured default (SMs / 3)
  static const int over = getenv("JANUS_DISPATCH_CTAS") ? atoi(getenv("JANUS_DISPATCH_CTAS")) : 0;
  return std::min(grid_for(work), over > 0 ? over : std::max(8, sms / 3));
}


XferLayout xfer_layout(int A, int M, long long T_max, int d_h, int k) {
  XferLayout L{};
  auto up = [](size_t v) { return (v + 255) & ~size_t(255); };
  const long long ta_max = (T_max + A - 1) / A;
  size_t o = 0;
  L.flag_dispatch_off = o;
  o = up(o + 8 * (size_t)A);
  L.flag_combine_off = o;
  o = up(o + 8 * (size_t)M);
  L.flag_route_off = o;
  o = up(o + 8 * (size_t)A);
  const size_t slot0 = o;
  L.x_off = o;
  o = up(o + (size_t)T_max * d_h * 2);
  L.ex_off = o;
  o = up(o + (size_t)T_max * k * 4);
  L.gw_off = o;
  o = up(o + (size_t)T_max * k * 4);
  L.part_off = o;
  o = up(o + (size_t)M * ta_max * d_h * 2);
  L.err_off = o;
  o = up(o + 8 * (size_t)M);
  L.slot_stride = o - slot0;
  L.bytes = o + (kXferSlots - 1) * L.slot_stride;
  L.ta_max = ta_max;
  return L;
}

cudaError_t launch_dispatch(const XferState &x, const void *d_x, const int32_t *d_ex,
                            const float *d_gw, long long T, unsigned long long epoch,
                            cudaStream_t s) {
  long long first = 0, Ta = 0;
  shard_host(x, T, first, Ta);
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
  dispatch_kernel<<<side_grid(std::max<long long>(Ta * x.d_h / 8, 1)), 256, 0, s>>>(
      dst, peer_ptrs(x), x.M, x.moe0, x.rank, reinterpret_cast<const uint4 *>(d_x), d_ex, d_gw,
      first, Ta, vec, x.k, x.L, epoch, counter_for(x, 0, epoch));
  return cudaGetLastError();
}

namespace {
using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WriteValue64Fn write_value64_fn() {
  static WriteValue64Fn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue64Fn>(ptr);
  }
  return fn;
}
}  // namespace

cudaError_t launch_dispatch_ce(const XferState &x, const void *d_x, const int32_t *d_ex,
                               const float *d_gw, long long T, unsigned long long epoch,
                               cudaStream_t s) {
  WriteValue64Fn wv = write_value64_fn();
  if (!wv) return cudaErrorNotSupported;
  long long first = 0, Ta = 0;
  shard_host(x, T, first, Ta);
  const size_t so = xfer_slot(epoch) * x.L.slot_stride;
  const size_t row = (size_t)x.d_h * 2;
  const bool fork = (int)x.ce_streams.size() == x.M && x.M > 1;
  if (fork) {
    cudaError_t e = cudaEventRecord(x.ce_fork, s);
    if (e != cudaSuccess) return e;
  }
  for (int g = 0; g < x.M; ++g) {
    unsigned char *base = static_cast<unsigned char *>(x.peer_base[x.moe0 + g]);
    cudaError_t e = cudaSuccess;
    cudaStream_t sg = s;
    if (fork) {  // rank g's copies on their own stream (their own copy engine)
      sg = x.ce_streams[g];
      e = cudaStreamWaitEvent(sg, x.ce_fork, 0);
      if (e != cudaSuccess) return e;
    }
    if (Ta > 0) {
      e = cudaMemcpyAsync(base + x.L.x_off + so + (size_t)first * row, d_x, (size_t)Ta * row,
                          cudaMemcpyDeviceToDevice, sg);
      if (e == cudaSuccess && d_ex)
        e = cudaMemcpyAsync(base + x.L.ex_off + so + (size_t)first * x.k * 4, d_ex,
                            (size_t)Ta * x.k * 4, cudaMemcpyDeviceToDevice, sg);
      if (e == cudaSuccess && d_gw)
        e = cudaMemcpyAsync(base + x.L.gw_off + so + (size_t)first * x.k * 4, d_gw,
                            (size_t)Ta * x.k * 4, cudaMemcpyDeviceToDevice, sg);
    }
    if (e != cudaSuccess) return e;
    // flag_dispatch[a] = epoch on MoE rank g, after this stream's copies above
    // (default flags: the write is preceded by a memory barrier)
    const CUdeviceptr flag =
        reinterpret_cast<CUdeviceptr>(base + x.L.flag_dispatch_off + 8 * (size_t)x.rank);
    if (wv(reinterpret_cast<CUstream>(sg), flag, (cuuint64_t)epoch, 0) != CUDA_SUCCESS)
      return cudaErrorLaunchFailure;
    if (fork) {
      e = cudaEventRecord(x.ce_done[g], sg);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, x.ce_done[g], 0);  // join
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

cudaError_t launch_route_push(const XferState &x, const int32_t *d_ex, const float *d_gw,
                              long long T, unsigned long long epoch, cudaStream_t s) {
  long long first = 0, Ta = 0;
  shard_host(x, T, first, Ta);
  const size_t so = xfer_slot(epoch) * x.L.slot_stride;
  route_push_kernel<<<side_grid(std::max<long long>(Ta * x.k, 1)), 256, 0, s>>>(
      peer_ptrs(x), x.world, x.rank, d_ex, d_gw, first, Ta * x.k, x.k, x.L.ex_off + so,
      x.L.gw_off + so, x.L, epoch, counter_for(x, 1, epoch));
  return cudaGetLastError();
}

cudaError_t launch_routed_dispatch(const XferState &x, const void *d_x, const int32_t *inst,
                                   const int32_t *status, long long T, unsigned long long epoch,
                                   cudaStream_t s) {
  long long first = 0, Ta = 0;
  shard_host(x, T, first, Ta);
  const size_t so = xfer_slot(epoch) * x.L.slot_stride;
  routed_dispatch_kernel<<<side_grid(std::max<long long>(Ta * 32, 1)), 256, 0, s>>>(
      peer_ptrs(x), x.M, x.moe0, x.rank, reinterpret_cast<const uint4 *>(d_x), inst, status,
      first, Ta, x.d_h / 8, x.k, x.L.x_off + so, x.dmask + xfer_slot(epoch) * x.L.ta_max, x.err,
      x.L, epoch, counter_for(x, 0, epoch));
  return cudaGetLastError();
}

cudaError_t launch_wait(const XferState &x, int kind, unsigned long long epoch, cudaStream_t s,
                        int skip) {
  unsigned char *base = static_cast<unsigned char *>(x.local);
  // kind 3: the combine flags again, for the slot-free wait of a dispatch
  // (its own skip word; errors are the combine's to report)
  const size_t off = kind == 0 ? x.L.flag_dispatch_off
                     : kind == 1 || kind == 3 ? x.L.flag_combine_off
                                              : x.L.flag_route_off;
  const int n = kind == 1 || kind == 3 ? x.M : x.A;
  const int2 *errs =
      kind == 1 ? reinterpret_cast<const int2 *>(base + x.L.err_off + xfer_slot(epoch) * x.L.slot_stride)
                : nullptr;
  wait_flags_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const unsigned long long *>(base + off), n,
                                     epoch, errs, x.err, kind, x.timeout_ns, skip);
  return cudaGetLastError();
}

PushDst push_dst(const XferState &x, unsigned long long epoch) {
  PushDst p{};
  for (int a = 0; a < x.A && a < kPushMaxPeers; ++a)
    p.base[a] = static_cast<unsigned char *>(x.peer_base[a]);
  p.part_off = x.L.part_off + xfer_slot(epoch) * x.L.slot_stride;
  p.ta_max = x.L.ta_max;
  p.A = x.A;
  p.g = x.rank - x.moe0;
  p.skip_empty = x.transport == kXferRouted ? 1 : 0;
  return p;
}

cudaError_t launch_signal_combine(const XferState &x, const int32_t *status,
                                  unsigned long long epoch, cudaStream_t s) {
  signal_combine_kernel<<<1, 32, 0, s>>>(peer_ptrs(x), x.A, x.rank - x.moe0, x.L,
                                         x.L.err_off + xfer_slot(epoch) * x.L.slot_stride, status,
                                         x.err, epoch);
  return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const XferState &x, void *d_out, long long Ta,
                                   unsigned long long epoch, cudaStream_t s) {
  if (Ta == 0) return cudaSuccess;
  const unsigned char *base = static_cast<const unsigned char *>(x.local);
  // JANUS_REDUCE_CTAS: tuning override of the grid (default: the work, <= 8 x SMs)
  static const int over = getenv("JANUS_REDUCE_CTAS") ? atoi(getenv("JANUS_REDUCE_CTAS")) : 0;
  const int grid = over > 0 ? std::min(over, grid_for(Ta * (x.d_h / 8))) : grid_for(Ta * (x.d_h / 8));
  reduce_partials_kernel<<<grid, 256, 0, s>>>(
      reinterpret_cast<const __nv_bfloat16 *>(base + x.L.part_off +
                                               xfer_slot(epoch) * x.L.slot_stride),
      x.M, Ta, x.L.ta_max, x.d_h,
      x.transport == kXferRouted ? x.dmask + xfer_slot(epoch) * x.L.ta_max : nullptr,
      x.err + kErrSkip + 1, reinterpret_cast<__nv_bfloat16 *>(d_out));
  return cudaGetLastError();
}

cudaError_t launch_reduce_mc(const XferState &x, void *d_out, long long first, long long Ta,
                             unsigned long long epoch, cudaStream_t s) {
  if (Ta == 0) return cudaSuccess;
  const long long vec = x.d_h / 8, n = Ta * vec;
  const uint4 *part =
      reinterpret_cast<const uint4 *>(x.mc_va + x.mpart_off + xfer_slot(epoch) * x.mslot) +
      first * vec;
  reduce_mc_kernel<<<grid_for((n + 3) / 4), 256, 0, s>>>(part, n, x.err + kErrSkip + 1,
                                                          reinterpret_cast<uint4 *>(d_out));
  return cudaGetLastError();
}

}  // namespace janus
