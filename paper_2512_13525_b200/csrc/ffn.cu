// ffn.cu — K3 permute and K5 combine (the K4 GEMMs are in gemm.cu).
//   xp[row(s)] = x[s / k]                 (permute, slot-major)
//   out[t] = sum_j w[t,j] y[row(t,j)]    (combine, fixed j order, fp32)
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

namespace janus {
namespace {

// ------------------------------------------------------------ permute -----
// xp[slot_row[t*k+j]] = x[t] for the slots routed to `instance` (all slots
// when instance < 0).  Token-major: one warp task = one 32*U-chunk segment of
// token t's row, loaded once into registers and stored to each of the token's
// k destination rows (x is read once; the k row indices are loaded by lanes
// j < k and broadcast with shuffles).
// (A TMA tile::gather4 fusion of this copy into the GEMM's B loads was
// measured at ~16 cycles per gathered 128-B row per SM — 2x slower at T=4096 —
// and a cp.async gather broke even at best; see profiles/README.md.)
// volatile so the 8 x U loads of a combine group stay ahead of their uses
__device__ __forceinline__ uint4 ld_nc(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

constexpr int kPermU = 4;    // 16-B chunks per lane per task (2 KB segments)
constexpr int kCombU = 2;    // 16-B chunks per lane per task (1 KB segments)
constexpr int kWarpsPerBlock = 4;

__global__ void permute_kernel(const uint4 *__restrict__ x, const int32_t *__restrict__ slot_row,
                               const int32_t *__restrict__ slot_inst, int instance, int T, int k,
                               int vec, uint4 *__restrict__ xp, uint4 *__restrict__ xp_shared,
                               int sh0, int sh1, const int32_t *__restrict__ status) {
  sm100::pdl_trigger();
  sm100::pdl_wait();  // slot_row / slot_inst from K1
  if (status && status[0] != JANUS_OK) return;  // rejected step: no layout
  const int lane = threadIdx.x & 31;
  const int segs = (vec + 32 * kPermU - 1) / (32 * kPermU);
  const int task = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (task >= T * segs) return;
  const int t = task / segs, c0 = (task % segs) * 32 * kPermU + lane;
  const uint4 *src = x + (size_t)t * vec;
  uint4 v[kPermU];
  bool loaded = false;  // x is read only if some slot of t is routed here
  if (xp_shared && t >= sh0 && t < sh1) {  // the shared expert's tokens, in token order
#pragma unroll
    for (int u = 0; u < kPermU; ++u) {
      const int c = c0 + 32 * u;
      if (c < vec) {
        v[u] = __ldg(src + c);
        xp_shared[(size_t)(t - sh0) * vec + c] = v[u];
      }
    }
    loaded = true;
  }
  for (int j0 = 0; j0 < k; j0 += 32) {
    const int j = j0 + lane;
    int row = -1;
    if (j < k) {
      const int s = t * k + j;
      if (instance < 0 || __ldg(slot_inst + s) == instance) row = __ldg(slot_row + s);
    }
    unsigned m = __ballot_sync(0xffffffffu, row >= 0);
    if (m && !loaded) {
#pragma unroll
      for (int u = 0; u < kPermU; ++u) {
        const int c = c0 + 32 * u;
        if (c < vec) v[u] = __ldg(src + c);
      }
      loaded = true;
    }
    for (; m; m &= m - 1) {
      const int r = __shfl_sync(0xffffffffu, row, __ffs(m) - 1);
      uint4 *dst = xp + (size_t)r * vec;
#pragma unroll
      for (int u = 0; u < kPermU; ++u) {
        const int c = c0 + 32 * u;
        if (c < vec) dst[c] = v[u];
      }
    }
  }
}

// ------------------------------------------------------------ combine -----
// out[t] = sum_j w[t,j] * y[slot_row[t,j]] over the slots routed to `instance`
// (all slots when instance < 0), j ascending, fp32, then bf16.  One warp task
// = one 32*U-chunk segment of token t; the row indices / weights are loaded by
// lanes j < k and broadcast; 8 rows x U chunks are in flight per lane.
// G = slots gathered per round (4: measured faster than 8 even with every
// slot local — fewer registers, more warps; with the instance filter about k/M
// of a token's slots are routed here and the ballot compaction keeps the loads
// to the slots that exist).
// Shard rule (comm.cpp:76-81): owner a of token t and the shard's first token.
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

// Push mode (push.A > 0, the box exchange): the partial sum of token t goes
// straight into its owning attention rank's region over NVLink (the combine
// fused with the transfer); skip_empty drops tokens with no slot here.
// One warp task: one 32 * kCombU-chunk segment of token t's output row.
template <int G>
__device__ __forceinline__ void combine_task(int task, int segs, int lane,
                                             const uint4 *__restrict__ y,
                                             const int32_t *__restrict__ slot_row,
                                             const int32_t *__restrict__ slot_inst, int instance,
                                             const float *__restrict__ gw, int T, int k, int vec,
                                             uint4 *__restrict__ out,
                                             const uint4 *__restrict__ y_shared, int sh0, int sh1,
                                             const int32_t *__restrict__ status,
                                             const PushDst &push) {
  const int t = task / segs, c0 = (task % segs) * 32 * kCombU + lane;
  uint4 *orow = out + (size_t)t * vec;
  if (push.A > 0) {
    int a;
    long long first;
    shard_of(T, push.A, t, a, first);
    orow = reinterpret_cast<uint4 *>(push.base[a] + push.part_off) +
           ((long long)push.g * push.ta_max + (t - first)) * vec;
  }
  if (status && status[0] != JANUS_OK) {  // rejected step: no y reads
    if (push.A > 0) return;  // the error slot tells the owner (signal_combine_kernel)
#pragma unroll
    for (int u = 0; u < kCombU; ++u)   // defined zeros
      if (c0 + 32 * u < vec) orow[c0 + 32 * u] = make_uint4(0, 0, 0, 0);
    return;
  }
  bool any = y_shared && t >= sh0 && t < sh1;
  float acc[kCombU][8];
#pragma unroll
  for (int u = 0; u < kCombU; ++u)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
  for (int j0 = 0; j0 < k; j0 += 32) {
    const int j = j0 + lane;
    int row = -1;
    float w = 0.f;
    if (j < k) {
      const int s = t * k + j;
      if (instance < 0 || __ldg(slot_inst + s) == instance) {
        row = __ldg(slot_row + s);
        w = __ldg(gw + s);
      }
    }
    const int n = min(32, k - j0);
    // lanes holding a slot routed here, taken in ascending j, G per round
    unsigned m = __ballot_sync(0xffffffffu, lane < n && row >= 0);
    any = any || m != 0;
    while (m) {
      uint4 v[G][kCombU];
      float wv[G];
      const uint4 *src[G];
      bool ok[G];
#pragma unroll
      for (int b = 0; b < G; ++b) {
        ok[b] = m != 0;
        const int ln = ok[b] ? __ffs(m) - 1 : 0;
        m &= m - 1;
        const int r = __shfl_sync(0xffffffffu, row, ln);
        const float wb = __shfl_sync(0xffffffffu, w, ln);
        wv[b] = ok[b] ? wb : 0.f;
        src[b] = y + (size_t)(ok[b] ? r : 0) * vec;  // clamped; masked below
      }
      // all G x U loads are issued before the first is consumed
#pragma unroll
      for (int b = 0; b < G; ++b)
#pragma unroll
        for (int u = 0; u < kCombU; ++u) {
          const int c = c0 + 32 * u;
          v[b][u] = ld_nc(src[b] + min(c, vec - 1));
        }
#pragma unroll
      for (int b = 0; b < G; ++b)
#pragma unroll
        for (int u = 0; u < kCombU; ++u)
          if (!ok[b] || c0 + 32 * u >= vec) v[b][u] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int b = 0; b < G; ++b)  // fixed j order: bitwise reproducible
#pragma unroll
        for (int u = 0; u < kCombU; ++u) {
          const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v[b][u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            acc[u][2 * e] += wv[b] * f.x;
            acc[u][2 * e + 1] += wv[b] * f.y;
          }
        }
    }
  }
  if (y_shared && t >= sh0 && t < sh1) {  // the shared expert, weight 1, after the routed slots
#pragma unroll
    for (int u = 0; u < kCombU; ++u) {
      const int c = c0 + 32 * u;
      if (c >= vec) continue;
      const uint4 v = __ldg(y_shared + (size_t)(t - sh0) * vec + c);
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        acc[u][2 * e] += f.x;
        acc[u][2 * e + 1] += f.y;
      }
    }
  }
  if (push.skip_empty && !any) return;  // routed: nothing of t was computed here
#pragma unroll
  for (int u = 0; u < kCombU; ++u) {
    const int c = c0 + 32 * u;
    if (c >= vec) continue;
    uint4 o;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(acc[u][2 * e], acc[u][2 * e + 1]);
    orow[c] = o;
  }
}

template <int G>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, 4)
    combine_kernel(const uint4 *__restrict__ y, const int32_t *__restrict__ slot_row,
                   const int32_t *__restrict__ slot_inst, int instance,
                   const float *__restrict__ gw, int T, int k, int vec, uint4 *__restrict__ out,
                   const uint4 *__restrict__ y_shared, int sh0, int sh1,
                   const int32_t *__restrict__ status, const PushDst push) {
  sm100::pdl_trigger();
  sm100::pdl_wait();  // y from the down GEMM
  const int lane = threadIdx.x & 31;
  const int segs = (vec + 32 * kCombU - 1) / (32 * kCombU);
  const int stride = gridDim.x * kWarpsPerBlock;  // a capped grid (push beside the next GEMMs)
  for (int task = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); task < T * segs;
       task += stride)
    combine_task<G>(task, segs, lane, y, slot_row, slot_inst, instance, gw, T, k, vec, out,
                    y_shared, sh0, sh1, status, push);
}

}  // namespace

cudaError_t launch_permute(const void *x, const int32_t *slot_row, const int32_t *slot_instance,
                           int instance, int S, int k, int d_h, void *xp, void *xp_shared,
                           int sh0, int sh1, cudaStream_t s, const int32_t *status) {
  if (S == 0) return cudaSuccess;
  const int T = S / k, vec = d_h / 8;
  const int tasks = T * ((vec + 32 * kPermU - 1) / (32 * kPermU));
  const int blocks = (tasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
  return sm100::launch_pdl(permute_kernel, dim3(blocks), dim3(32 * kWarpsPerBlock), 0, s,
                           reinterpret_cast<const uint4 *>(x), slot_row, slot_instance, instance,
                           T, k, vec, reinterpret_cast<uint4 *>(xp),
                           reinterpret_cast<uint4 *>(xp_shared), sh0, sh1, status);
}

cudaError_t launch_combine(const void *y, const int32_t *slot_row, const int32_t *slot_instance,
                           int instance, const float *gate_w, int T, int k, int d_h, void *out,
                           cudaStream_t s, const void *y_shared, int sh0, int sh1,
                           const int32_t *status, const PushDst *push, int max_blocks) {
  if (T == 0) return cudaSuccess;
  const int vec = d_h / 8;
  const int tasks = T * ((vec + 32 * kCombU - 1) / (32 * kCombU));
  int blocks = (tasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (max_blocks > 0) blocks = std::min(blocks, max_blocks);
  PushDst pd{};
  if (push) pd = *push;
  return sm100::launch_pdl(combine_kernel<4>, dim3(blocks), dim3(32 * kWarpsPerBlock), 0, s,
                           reinterpret_cast<const uint4 *>(y), slot_row, slot_instance, instance,
                           gate_w, T, k, vec, reinterpret_cast<uint4 *>(out),
                           reinterpret_cast<const uint4 *>(y_shared), sh0, sh1, status, pd);
}

}  // namespace janus
