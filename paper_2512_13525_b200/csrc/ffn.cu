// ffn.cu — K3 permute and K5 combine (the K4 GEMMs are in gemm.cu).
//   xp[row(s)] = x[s / k]                 (permute, slot-major)
//   out[t] = sum_j w[t,j] y[row(t,j)]    (combine, fixed j order, fp32)
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"

namespace janus {
namespace {

// ------------------------------------------------------------ permute -----
// xp[slot_row[s]] = x[s / k] for the slots routed to `instance` (all slots
// when instance < 0).  Slot-major: reads of x are sequential and every row
// write is a contiguous burst.  One thread per 16-B chunk; grid-stride.
// (A TMA tile::gather4 fusion of this copy into the GEMM's B loads was
// measured at ~16 cycles per gathered 128-B row per SM — 2x slower at T=4096 —
// see profiles/README.md.)
__global__ void permute_kernel(const uint4 *__restrict__ x, const int32_t *__restrict__ slot_row,
                               const int32_t *__restrict__ slot_inst, int instance, int S, int k,
                               int vec_per_row, uint4 *__restrict__ xp) {
  const long long n = (long long)S * vec_per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / vec_per_row), c = (int)(i % vec_per_row);
    if (instance >= 0 && __ldg(slot_inst + s) != instance) continue;
    xp[(size_t)__ldg(slot_row + s) * vec_per_row + c] = __ldg(x + (size_t)(s / k) * vec_per_row + c);
  }
}

// ------------------------------------------------------------ combine -----
// out[t] = sum_j w[t,j] * y[slot_row[t,j]] over the slots routed to `instance`
// (all slots when instance < 0), j ascending, fp32, then bf16.
__global__ void combine_kernel(const __nv_bfloat16 *__restrict__ y,
                               const int32_t *__restrict__ slot_row,
                               const int32_t *__restrict__ slot_inst, int instance,
                               const float *__restrict__ gw, int T, int k, int d_h,
                               __nv_bfloat16 *__restrict__ out) {
  // One thread per (token, 16-B output chunk); the k row loads of a chunk are
  // issued together (groups of 8) before any is consumed.
  const int vec = d_h / 8;
  const long long n = (long long)T * vec;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(idx / vec), c = (int)(idx % vec);
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int j0 = 0; j0 < k; j0 += 8) {
      uint4 v[8];
      float w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
        w[u] = 0.f;
        v[u] = make_uint4(0, 0, 0, 0);
        if (j < k) {
          const int s = t * k + j;
          if (instance < 0 || __ldg(slot_inst + s) == instance) {
            w[u] = __ldg(gw + s);
            v[u] = __ldg(reinterpret_cast<const uint4 *>(y + (size_t)__ldg(slot_row + s) * d_h) + c);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // fixed j order: bitwise reproducible
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          acc[2 * e] += w[u] * f.x;
          acc[2 * e + 1] += w[u] * f.y;
        }
      }
    }
    uint4 o;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
    reinterpret_cast<uint4 *>(out + (size_t)t * d_h)[c] = o;
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

cudaError_t launch_permute(const void *x, const int32_t *slot_row, const int32_t *slot_instance,
                           int instance, int S, int k, int d_h, void *xp, cudaStream_t s) {
  if (S == 0) return cudaSuccess;
  const long long threads = (long long)S * (d_h / 8);
  const int blocks = (int)std::min<long long>((threads + 255) / 256, sm_count() * 16);
  permute_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint4 *>(x), slot_row,
                                        slot_instance, instance, S, k, d_h / 8,
                                        reinterpret_cast<uint4 *>(xp));
  return cudaGetLastError();
}

cudaError_t launch_combine(const void *y, const int32_t *slot_row, const int32_t *slot_instance,
                           int instance, const float *gate_w, int T, int k, int d_h, void *out,
                           cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const long long threads = (long long)T * (d_h / 8);
  const int blocks = (int)std::min<long long>((threads + 255) / 256, sm_count() * 16);
  combine_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16 *>(y), slot_row,
                                        slot_instance, instance, gate_w, T, k, d_h,
                                        reinterpret_cast<__nv_bfloat16 *>(out));
  return cudaGetLastError();
}

}  // namespace janus
