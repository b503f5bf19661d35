// gate.cu — the MoE-side gating kernel: router GEMM
// logits = x · Wrᵀ on tcgen05, then per-token top-k and the softmax over the
// selected logits, producing the top-k ids (and gate weights) K1 consumes.
// Janus gates on the MoE side; the reference has no gating
// code — it consumes ActivationBatch ids (aebs.hpp:15-24) — so the definition
// is the oracle's or_gate (oracle/oracle.c): ties go to the lower expert id,
// ids are written in rank order, weights are softmax(top-k logits).
//
// One CTA per 128 tokens (UMMA M = 128, cta_group::1), N = E (≤ 256), K = d_h
// in 64-wide k-blocks through a 4-stage TMA ring; fp32 logits in TMEM (one
// token per lane).  Epilogue: each of 128 threads owns one token's logits
// (tcgen05.ld 32x32b), keeps a sorted top-KMAX list in registers while it
// streams the E columns, then writes k ids and k softmax weights.  HBM-bound:
// x is read once (2·d_h bytes per token), Wr (2·E·d_h) from L2.
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace janus {
namespace {

using namespace sm100;

constexpr int kGateM = 128;   // tokens per CTA
constexpr int kGBK = 64;      // K per stage
constexpr int kGStages = 4;
constexpr int kGateThreads = 192;  // warp 0 TMA, warp 1 TMEM + MMA, warps 2-5 epilogue

struct GateParams {
  CUtensorMap tm_x;  // x [T][d_h], box {64, 128}
  CUtensorMap tm_w;  // Wr [E][d_h], box {64, E}
  int T, K, E, k;
  int32_t *experts;  // [T*k]
  float *gw;         // [T*k]
};

__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *tm, uint64_t *bar, int x,
                                         int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// kind::f16 instruction descriptor: D f32, A/B bf16, K-major, M=128, N=n.
__device__ __forceinline__ uint32_t idesc_m128(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <int KMAX>
__global__ void __launch_bounds__(kGateThreads, 1) gate_kernel(const __grid_constant__ GateParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int wbytes = p.E * kGBK * 2;
  const int stage_bytes = kGateM * kGBK * 2 + wbytes;  // multiple of 1024 (E % 16 == 0)
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kGStages * stage_bytes);
  uint64_t *empty = full + kGStages;
  uint64_t *done = empty + kGStages;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * kGateM;
  const int kblocks = p.K / kGBK;
  const uint32_t ncols = p.E <= 32 ? 32 : p.E <= 64 ? 64 : p.E <= 128 ? 128 : 256;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tm_x);
    prefetch_tmap(&p.tm_w);
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {  // TMA producer
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kGStages;
      mbar_wait(&empty[s], ((kb / kGStages) & 1) ^ 1);
      if (elect_one()) {
        unsigned char *st = smem + s * stage_bytes;
        mbar_expect_tx(&full[s], (uint32_t)stage_bytes);
        tma_load(st, &p.tm_x, &full[s], kb * kGBK, t0);
        tma_load(st + kGateM * kGBK * 2, &p.tm_w, &full[s], kb * kGBK, 0);
      }
      __syncwarp();
    }
  } else if (warp == 1) {  // MMA issuer
    const uint32_t idesc = idesc_m128(p.E);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kGStages;
      mbar_wait(&full[s], (kb / kGStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kGateM * kGBK * 2);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kGBK / 16; ++k) umma(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(done);
    __syncwarp();
  } else {  // epilogue: thread = token (TMEM lane)
    const int quad = warp & 3;
    const int row = quad * 32 + lane, t = t0 + row;
    mbar_wait(done, 0);
    tc_fence_after();
    float val[KMAX];
    int idx[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      val[j] = -INFINITY;
      idx[j] = -1;
    }
    for (int e0 = 0; e0 < p.E; e0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + e0, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float x = v[i];
        const int e = e0 + i;
        // insert into the descending list; strict '>' keeps the lower id
        // first among equal logits (ids arrive ascending)
        if (e < p.E && x > val[KMAX - 1]) {
#pragma unroll
          for (int j = KMAX - 1; j > 0; --j) {
            if (x > val[j - 1]) {
              val[j] = val[j - 1];
              idx[j] = idx[j - 1];
            } else if (x > val[j]) {
              val[j] = x;
              idx[j] = e;
            }
          }
          if (x > val[0]) {
            val[0] = x;
            idx[0] = e;
          }
        }
      }
    }
    if (t < p.T) {
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < p.k) sum += expf(val[j] - val[0]);
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < p.k) {
          p.experts[(size_t)t * p.k + j] = idx[j];
          p.gw[(size_t)t * p.k + j] = expf(val[j] - val[0]) / sum;
        }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
  }
}

template <int KMAX>
cudaError_t launch_gate_k(const GateParams &g, size_t smem, cudaStream_t s) {
  static int configured_dev = -1;
  static size_t configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev || smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(gate_kernel<KMAX>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured_dev = dev;
    configured = smem;
  }
  const int blocks = (g.T + kGateM - 1) / kGateM;
  gate_kernel<KMAX><<<blocks, kGateThreads, smem, s>>>(g);
  return cudaGetLastError();
}

}  // namespace

bool gate_shape_ok(int d_h, int E, int k) {
  return d_h > 0 && d_h % kGBK == 0 && E >= 16 && E <= 256 && E % 16 == 0 && k >= 1 && k <= 16 &&
         k <= E;
}

cudaError_t launch_gate(const void *x, const void *wr, int T, int d_h, int E, int k,
                        int32_t *experts, float *gw, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  GateParams g{};
  if (!make_map(&g.tm_x, x, (uint64_t)T, (uint64_t)d_h, kGateM) ||
      !make_map(&g.tm_w, wr, (uint64_t)E, (uint64_t)d_h, (uint32_t)E))
    return cudaErrorInvalidValue;
  g.T = T;
  g.K = d_h;
  g.E = E;
  g.k = k;
  g.experts = experts;
  g.gw = gw;
  const size_t smem =
      (size_t)kGStages * (kGateM * kGBK * 2 + (size_t)E * kGBK * 2) + 1024 + 128;
  if (k <= 4) return launch_gate_k<4>(g, smem, s);
  if (k <= 8) return launch_gate_k<8>(g, smem, s);
  return launch_gate_k<16>(g, smem, s);
}

}  // namespace janus
