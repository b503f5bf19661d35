// gate.cu — the MoE-side gating kernel: router GEMM
// logits = x · Wrᵀ on tcgen05, then per-token top-k and the softmax over the
// selected logits, producing the top-k ids (and gate weights) K1 consumes.
// Janus gates on the MoE side; the reference has no gating
// code — it consumes ActivationBatch ids (aebs.hpp:15-24) — so the definition
// is the oracle's or_gate (oracle/oracle.c): ties go to the lower expert id,
// ids are written in rank order, weights are softmax(top-k logits).
//
// One cluster of S CTAs per 128 tokens (UMMA M = 128, cta_group::1), N = E
// (<= 256), K = d_h split S ways (S = 1, 2, 4 or 8: the largest that keeps
// the grid one wave of resident clusters — at T = 4096 one CTA per token block
// would leave 116 SMs idle and each CTA streaming 1 MB).  Each CTA runs its k-blocks through a TMA ring
// into fp32 TMEM partial logits (one token per lane).  S = 1: each of 128
// epilogue threads keeps a sorted top-KMAX list in registers while it streams
// its token's E logits from TMEM.  S > 1: the partials are staged in smem,
// bulk-stored to a global (L2-resident) exchange slot per CTA, and after a
// cluster barrier the CTA that owns a token (128/S tokens per CTA) sums its S
// partials in split order (deterministic); 2S threads per token each keep a
// top-KMAX of an interleaved column subset, and a shuffle merge yields the
// token's top-k.
// HBM-bound: x is read once (2·d_h bytes per token), Wr (2·E·d_h) from L2.
// Graph replay (c2 shape): 18.6 -> 12.6 -> 10.8 us at T=256, 18.7 -> 14.8 ->
// 12.7 us at T=4096 (one CTA per token block -> split K with a DSMEM exchange
// -> the exchange through L2); the rest is the load -> MMA -> exchange ->
// top-k chain of one token block and the cluster barriers.
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

namespace janus {
namespace {

using namespace sm100;

constexpr int kGateM = 128;   // tokens per CTA
constexpr int kGBK = 64;      // K per stage
constexpr int kGMaxStages = 8;
constexpr int kGRingBytes = 200 * 1024;  // smem ring budget (also the S > 1 receive buffer)
constexpr int kGateThreads = 256;  // warp 0 TMA, warp 1 TMEM + MMA, warps 2-5 TMEM drain; all 8: top-k

struct GateParams {
  CUtensorMap tm_x;  // x [T][d_h], box {64, 128}
  CUtensorMap tm_w;  // Wr [E][d_h], box {64, E}
  int T, K, E, k;
  int splits;        // S: CTAs (cluster) per token block, K split S ways
  int stages;        // ring depth
  int32_t *experts;  // [T*k]
  float *gw;         // [T*k]
  float *xchg;       // S > 1: [chunks][grid][128][ld] partial logits (global, L2-resident)
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

__device__ __forceinline__ void st_shared_v4(uint32_t addr, const float *v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3])
               : "memory");
}
__device__ __forceinline__ float ld_shared_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// global -> own smem bulk copy, completing `bytes` on the mbarrier
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// smem -> global bulk copy (async proxy), tracked by the bulk-group counter
__device__ __forceinline__ void bulk_store(void *dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// (a, ia) ranks before (b, ib): larger logit, ties to the lower id (empty
// entries carry id -1 = the largest unsigned, so they rank last)
__device__ __forceinline__ bool ranks_before(float a, int ia, float b, int ib) {
  return a > b || (a == b && (unsigned)ia < (unsigned)ib);
}

// Insert (x, e) into the descending list val/idx (branch-free: every j uses
// the old list, so the compares run in parallel); strict '>' keeps the lower
// id first among equal logits (callers feed ids in ascending order).
template <int KMAX>
__device__ __forceinline__ void topk_insert(float (&val)[KMAX], int (&idx)[KMAX], float x, int e) {
#pragma unroll
  for (int j = KMAX - 1; j > 0; --j) {
    const bool up = x > val[j - 1], here = x > val[j];
    val[j] = up ? val[j - 1] : here ? x : val[j];
    idx[j] = up ? idx[j - 1] : here ? e : idx[j];
  }
  const bool top = x > val[0];
  val[0] = top ? x : val[0];
  idx[0] = top ? e : idx[0];
}

// Merge the sorted lists of the G consecutive lanes of a token: KMAX rounds
// of a group arg-max over the list heads (xor shuffles, ties to the lower
// id); the lane holding the winner pops it.  Every lane of the group ends
// with the merged list in outv/outi.
template <int KMAX>
__device__ __forceinline__ void merge_group(float (&val)[KMAX], int (&idx)[KMAX], int G,
                                            float (&outv)[KMAX], int (&outi)[KMAX]) {
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    float bv = val[0];
    int bi = idx[0];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      if (off < G) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ranks_before(ov, oi, bv, bi)) {
          bv = ov;
          bi = oi;
        }
      }
    }
    outv[j] = bv;
    outi[j] = bi;
    const bool pop = bi == idx[0];
#pragma unroll
    for (int q = 0; q < KMAX - 1; ++q) {
      val[q] = pop ? val[q + 1] : val[q];
      idx[q] = pop ? idx[q + 1] : idx[q];
    }
    val[KMAX - 1] = pop ? -INFINITY : val[KMAX - 1];
    idx[KMAX - 1] = pop ? -1 : idx[KMAX - 1];
  }
}

template <int KMAX>
__device__ __forceinline__ void write_topk(const GateParams &p, int t, const float (&val)[KMAX],
                                           const int (&idx)[KMAX]) {
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

template <int KMAX>
__global__ void __launch_bounds__(kGateThreads, 1) gate_kernel(const __grid_constant__ GateParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nst = p.stages;
  const int wbytes = p.E * kGBK * 2;
  const int stage_bytes = kGateM * kGBK * 2 + wbytes;  // multiple of 1024 (E % 16 == 0)
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + nst * stage_bytes);
  uint64_t *empty = full + kGMaxStages;
  uint64_t *done = empty + kGMaxStages;
  uint64_t *recv_bar = done + 1;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(recv_bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.splits;
  uint32_t split = 0;
  if (S > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(split));
  const int t0 = (blockIdx.x / S) * kGateM;
  const int kblocks = p.K / kGBK;
  const int kb0 = (int)split * kblocks / S, kb1 = ((int)split + 1) * kblocks / S;
  const uint32_t ncols = p.E <= 32 ? 32 : p.E <= 64 ? 64 : p.E <= 128 ? 128 : 256;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tm_x);
    prefetch_tmap(&p.tm_w);
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(recv_bar, 1);
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
    for (int kb = kb0; kb < kb1; ++kb) {
      const int i = kb - kb0, s = i % nst;
      mbar_wait(&empty[s], ((i / nst) & 1) ^ 1);
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
    for (int kb = kb0; kb < kb1; ++kb) {
      const int i = kb - kb0, s = i % nst;
      mbar_wait(&full[s], (i / nst) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kGateM * kGBK * 2);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kGBK / 16; ++k) umma(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(done);
    __syncwarp();
  } else if (warp < 6) {
    mbar_wait(done, 0);  // the ring is dead and the partial logits are in TMEM
    tc_fence_after();
    if (S == 1) {  // no exchange: thread = token, straight from TMEM
      const int quad = warp & 3, row = quad * 32 + lane;
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
        for (int i = 0; i < 32; ++i)
          if (e0 + i < p.E) topk_insert(val, idx, v[i], e0 + i);
      }
      if (t0 + row < p.T) write_topk(p, t0 + row, val, idx);
    }
  }

  // ---- S > 1: exchange the partial logits, sum in split order, top-k ----
  // The E columns go in chunks of <= 128.  Per chunk: warps 2-5 stage their
  // token rows (thread = TMEM lane) into stg[128][ld] in the dead ring; one
  // thread bulk-stores the whole block to this CTA's slot of the global
  // exchange buffer (L2) and waits for it; after a cluster barrier the owner
  // of tokens [split*R, (split+1)*R) bulk-loads their rows of the S slots of
  // its cluster into recv[S][R][ld] (one L2 round trip), and G = 256/R
  // threads per owned token sum them in split order, inserting columns sub,
  // sub+G, ... into a top-KMAX list; after the last chunk the G lists merge.  (The exchange through DSMEM bulk copies moved
  // ~17-21 B/clk per SM, 1.4-4.7 us per chunk at T = 4096; L2 is several
  // times that.)
  if (S > 1) {
    const int R = kGateM / S;        // tokens owned by this CTA
    const int G = kGateThreads / R;  // threads per token (2S)
    const int nch = (p.E + 127) / 128;
    const int EC = ((p.E + nch - 1) / nch + 15) & ~15;  // chunk width
    const int ld = EC + G;           // row stride (floats)
    const uint32_t stg = smem_u32(smem);
    const uint32_t recv = stg + (uint32_t)(kGateM * ld) * 4u;
    const uint32_t part = (uint32_t)(R * ld) * 4u;  // bytes of one slot's owned rows
    const size_t slot = (size_t)kGateM * ld;  // floats per CTA slot
    const int tok = threadIdx.x / G, sub = threadIdx.x % G;
    const int first = blockIdx.x - (int)split;  // the cluster's first CTA
    float val[KMAX];
    int idx[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      val[j] = -INFINITY;
      idx[j] = -1;
    }
    for (int c = 0; c < nch; ++c) {
      const int c0 = c * EC, c1 = min(p.E, c0 + EC);
      float *xc = p.xchg + (size_t)c * gridDim.x * slot;
      if (c > 0) {  // the previous chunk's bulk store has read stg, every thread recv
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
      }
      if (warp >= 2 && warp < 6) {
        const int quad = warp & 3, row = quad * 32 + lane;
        const uint32_t dst = stg + (uint32_t)(row * ld) * 4u;
        for (int e0 = c0; e0 < c1; e0 += 32) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + e0, v);
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            if (e0 + q < c1) st_shared_v4(dst + (uint32_t)(e0 - c0 + q) * 4u, v + q);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging -> bulk store
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        bulk_store(xc + (size_t)blockIdx.x * slot, stg, (uint32_t)(slot * 4));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // written, not just read
        asm volatile("fence.proxy.async.global;" ::: "memory");    // async writes -> generic reads
      }
      cluster_barrier();  // every CTA's slot of this chunk is in global memory
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // barrier -> async reads
        mbar_expect_tx(recv_bar, (uint32_t)S * part);
        for (int j = 0; j < S; ++j)
          bulk_load(recv + (uint32_t)j * part, xc + (size_t)(first + j) * slot + (size_t)split * R * ld,
                    part, recv_bar);
      }
      mbar_wait(recv_bar, (uint32_t)c & 1);
      // recv[s][tok][e - c0]: split s's partial logit of owned token tok
      const uint32_t base = recv + (uint32_t)(tok * ld) * 4u;
      for (int e = c0 + sub; e < c1; e += G) {
        const uint32_t a = base + (uint32_t)(e - c0) * 4u;
        float x = ld_shared_f32(a);
#pragma unroll
        for (int s = 1; s < 8; ++s)
          if (s < S) x += ld_shared_f32(a + (uint32_t)s * part);
        topk_insert(val, idx, x, e);
      }
    }
    float outv[KMAX];
    int outi[KMAX];
    merge_group(val, idx, G, outv, outi);
    const int t = t0 + (int)split * R + tok;
    if (sub == 0 && t < p.T) write_topk(p, t, outv, outi);
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
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kGateThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // clusters of n CTAs resident at once (GPC-bound: fewer than SMs / n for
  // n = 4, 8), per device and shared-memory size
  static int occ_dev = -1;
  static size_t occ_smem = 0;
  static int occ[4] = {0, 0, 0, 0};  // n = 1, 2, 4, 8
  if (occ_dev != dev || occ_smem != smem) {
    for (int i = 0; i < 4; ++i) {
      attr[0].val.clusterDim.x = 1u << i;
      cfg.gridDim = dim3(1u << i);
      cudaError_t e = cudaOccupancyMaxActiveClusters(&occ[i], gate_kernel<KMAX>, &cfg);
      if (e != cudaSuccess) return e;
    }
    occ_dev = dev;
    occ_smem = smem;
  }
  // split K S ways while every cluster of the grid is resident at once (one
  // wave) and each CTA keeps >= 2 k-blocks
  int S = 1, lg = 0;
  while (S < 8 && blocks <= occ[lg + 1] && g.K / kGBK >= 4 * S) {
    S *= 2;
    ++lg;
  }
  if (S > 1 && !g.xchg) return cudaErrorInvalidValue;
  GateParams gs = g;
  gs.splits = S;
  attr[0].val.clusterDim.x = S;
  cfg.gridDim = dim3(blocks * S);
  return cudaLaunchKernelEx(&cfg, gate_kernel<KMAX>, gs);
}

}  // namespace

bool gate_shape_ok(int d_h, int E, int k) {
  return d_h > 0 && d_h % kGBK == 0 && E >= 16 && E <= 256 && E % 16 == 0 && k >= 1 && k <= 16 &&
         k <= E;
}

size_t gate_xchg_bytes(int sms) {  // S > 1 only while the grid is one wave
  return (size_t)2 * sms * kGateM * (128 + 16) * sizeof(float);
}

cudaError_t launch_gate(const void *x, const void *wr, int T, int d_h, int E, int k,
                        int32_t *experts, float *gw, float *xchg, cudaStream_t s) {
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
  g.xchg = xchg;
  // the K split S is chosen at launch (launch_gate_k: one wave of clusters)
  const int stage_bytes = kGateM * kGBK * 2 + E * kGBK * 2;
  g.stages = std::min(kGMaxStages, kGRingBytes / stage_bytes);
  const size_t smem = (size_t)g.stages * stage_bytes + 1024 + 256;
  if (k <= 4) return launch_gate_k<4>(g, smem, s);
  if (k <= 8) return launch_gate_k<8>(g, smem, s);
  return launch_gate_k<16>(g, smem, s);
}

}  // namespace janus
