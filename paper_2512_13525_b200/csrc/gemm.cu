// gemm.cu — K4: the grouped SwiGLU expert GEMMs on tcgen05 CTA pairs, TMA and
// TMEM.  sm_100a only.
//
// The expert FFN has no reference implementation: the reference models it as
// t_launch + max(A*W_e/beta, 2*b*d_h*d_e/pi) (src/latency.cpp:17-24).  Here it
// is computed for real:
//   h = silu(x Wg^T) * (x Wu^T)          (kernel mode SWIGLU, h kept in bf16)
//   y = h Wd^T                           (kernel mode PLAIN)
//
// Grouped GEMM, swap-AB, on CTA pairs.  The weight rows are the UMMA M side,
// the ragged token rows of one replica group the N side, K the reduction dim.
// A tile is one replica group q x 256 weight rows x <=256 token rows, computed
// by a cluster of 2 CTAs with tcgen05.mma.cta_group::2 (M=256): CTA r holds
// 128 weight rows of A and half of the token rows of B in its own smem, the
// pair's tensor cores share both halves, and CTA r's TMEM accumulates its 128
// rows x N columns.  Per SM and k-block that is 32 KB written by TMA and 32 KB
// read by the MMAs — half the smem traffic of two independent M=128 tiles,
// which capped the single-CTA version at ~58% of the tensor pipe (profiles/).
//   SWIGLU  CTA r's 128 rows = 8 blocks of (8 gate rows, the 8 up rows of the
//           same features), loaded by one 4-D TMA box, so a 16x256b TMEM load
//           hands each epilogue thread gate and up of one feature and h is
//           formed in registers for 64 features per CTA.
//   PLAIN   CTA r's 128 rows = 128 consecutive rows of the down projection.
// Per CTA (352 threads): warp 0 weight (A) producer + tile fetch, warp 1 TMEM
// owner (+ the MMA issuer in the leader CTA), warps 2-9 epilogue (tcgen05.ld ->
// math -> bf16 -> stmatrix.trans -> TMA store), warp 10 token-row (B)
// producer; producer/MMA roles run as whole warps and issue via elect.sync.
// Smem ring of 6 stages (256-row tiles) or 9 (decode, 64-row tiles), TMEM
// double-buffered accumulators of 256 columns.  Persistent: 74 pairs draw
// tiles from a global counter (dynamic scheduling: a pair that drew a cheap
// tile draws the next one sooner) over the tile list that the scheduler
// kernel wrote to device memory (group_off, tile_off) — no host sync; the
// leader publishes each index to both CTAs through a small smem queue.
#include <cuda_bf16.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace janus {
namespace {

using namespace sm100;

constexpr int kBK = 64;                        // K elements per stage (128-B rows, SW128)
constexpr int kATileBytes = 128 * kBK * 2;     // 16 KB: this CTA's 128 weight rows
constexpr int kEpiCols = 32;                   // token columns per epilogue chunk
constexpr int kEpiGroups = 2;                  // epilogue warpgroups (alternate 32-column chunks)
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kWarpStaging = kEpiCols * 32 * 2;  // per epilogue warp: 32 tokens x <=32 features bf16
constexpr int kGemmThreads = 64 + 32 * kEpiWarps + 32;  // + the B-producer warp
constexpr int kTmemCols = 512;                 // 2 accumulators x 256 columns
constexpr int kTQ = 4;                         // tile-queue slots (dynamic tile scheduler)
constexpr int kTQConsumers = 4 + 2 * kEpiWarps;  // leader MMA, peer A producer, 2 B producers, epilogue

// Two shapes of the smem ring, chosen per launch from the expected rows per
// replica group (api.cu): BH = token rows per CTA per tile (pair N = 2*BH).
//   BH=128  6 stages x (16 KB A + 16 KB B): the tensor-bound regime (N=256)
//   BH=32   9 stages x (16 KB A +  4 KB B): decode, 144 KB of weights in flight
template <int BH>
struct Ring {
  static constexpr int kBTileBytes = BH * kBK * 2;
  static constexpr int kStageBytes = kATileBytes + kBTileBytes;
  static constexpr int kStages = BH == 128 ? 6 : 9;
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kEpiWarps * kWarpStaging + 1024 /*align*/ + 512 /*barriers*/;
};

enum Mode { kSwiglu = 0, kPlain = 1 };

struct GemmParams {
  CUtensorMap tm_a;     // weights; SWIGLU: 4-D gate/up interleave map (box = 128 rows), PLAIN: 2-D, box 128 rows
  CUtensorMap tm_b[5];  // activations [S_alloc][K], box rows 8/16/32/64/128 (= N/2)
  CUtensorMap tm_out;   // output [S_alloc][out_ld], no swizzle, box {kF features, 32 rows}
  const int32_t *group_off;
  const int32_t *tile_off;  // n-tiles of tile_n rows per group (prefix)
  unsigned *ctr;            // [2] next-tile counter, finished CTAs (reset by the last CTA)
  int tile_n;     // token rows per tile (= 2*BH)
  int q_begin, q_end;
  int K;          // reduction length
  int m_tiles;    // weight blocks per group (SWIGLU: 128 features, PLAIN: 256)
  int m_per_q;    // weight rows per replica
  int up_off;     // SWIGLU: row offset of the up projection (d_e)
  __nv_bfloat16 *out;
  int out_ld;     // elements per output row
  // tile timeline (JANUS_GEMM_TRACE=1, tools/gemm_timeline.py): per tile
  // [draw, MMA start, accumulator ready, epilogue done, smid | q << 16 |
  // rows << 32 | m << 48, issuer at the tile queue, ns the issuer waited for
  // stages | ns it waited for the queue << 32, issue done] (%globaltimer ns);
  // nullptr = off
  unsigned long long *trace;
};

constexpr int kTW = 16;               // trace words per tile
constexpr int kTraceTiles = 1 << 14;  // per GEMM; the last 512 tiles' words: CTA 0's stage log
constexpr size_t kStageLog = (size_t)(kTraceTiles - 512) * kTW;  // [2048 stages][A, B, full, rows]
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Cluster-window address of the same smem variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// Publish a 16-byte record into a CTA's smem and complete that CTA's mbarrier
// phase with it (arrive + expect 16 bytes, then st.async completing them): no
// release fence, so the issuing thread does not wait for its in-flight TMA.
__device__ __forceinline__ void publish_v4(uint32_t cl_dst, int4 v, uint32_t cl_bar) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], 16;" ::"r"(
                   cl_bar)
               : "memory");
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::
          "r"(cl_dst),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(cl_bar)
      : "memory");
}
__device__ __forceinline__ int4 ld_shared_v4(const void *p) {
  int4 v;
  asm volatile("ld.volatile.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
// Relaxed arrive (consumers of the tile queue: only "read before reuse").
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA 2-D tile load by either CTA of the pair; completion bytes are counted on
// the leader CTA's mbarrier (cluster-window address).
__device__ __forceinline__ void tma_load_pair(void *dst, const CUtensorMap *tm, uint32_t bar_leader,
                                              int x, int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(bar_leader), "l"(policy)
      : "memory");
}
// 4-D variant (the SWIGLU weight map: {k, row in 8, gate/up, 8-row group}).
__device__ __forceinline__ void tma_load_pair_4d(void *dst, const CUtensorMap *tm,
                                                 uint32_t bar_leader, int x0, int x3,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x0), "r"(0), "r"(x3), "r"(bar_leader), "l"(policy)
      : "memory");
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=256 (pair).
__device__ __forceinline__ uint32_t idesc_bf16_m256(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((256u >> 4) << 24);
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// Arrive (once) on the mbarrier at this smem offset in both CTAs of the pair
// when every previously issued MMA of this thread has completed.
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// 16 lanes x 256 bit, 4 repeats along columns: thread t gets, per repeat i,
// lane (t/4) columns 8i + 2(t%4) + {0,1} in r[4i], r[4i+1] and lane (t/4)+8,
// same columns, in r[4i+2], r[4i+3].
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Four 8x8 b16 matrices from mma-fragment registers, stored transposed: lane l
// supplies the smem address of row l%8 of matrix l/8.
__device__ __forceinline__ void stmatrix_x4_trans(uint32_t addr, uint32_t a0, uint32_t a1,
                                                  uint32_t a2, uint32_t a3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr),
               "r"(a0), "r"(a1), "r"(a2), "r"(a3)
               : "memory");
}
// TMA store of one box from smem (bulk async-group of the issuing thread).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *tm, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}

struct TileCoord {
  int q, m, r0, rows;
  int half;     // token rows per CTA of the (first) sub-tile: UMMA N = 2*half
  int half_hi;  // wide tiles: rows per CTA of the second sub-tile (rows tile_n..), else 0
};

__device__ __forceinline__ int rows_per_cta(int rows) { return (((rows + 1) >> 1) + 7) & ~7; }


// Tiles are group-major, n-tiles fastest (consecutive tiles share the weight
// block); the n-tile count per group comes from K2 (tile_off): ceil(r / tile_n),
// or in decode (merge_tail) max(1, r / tile_n) with the last tile also taking
// the remainder — up to 2*tile_n - 1 rows, a "wide" tile of two sub-tiles
// sharing every weight k-block, so a remainder never costs its own pass over
// the weights.
// Token rows one CTA loads per stage for `half` rows: at most two TMA boxes
// (each TMA issue is on the token producer's critical path) — the largest
// power-of-two box <= half, then the remainder rounded up to a power of two.
// Rows past `half` land in smem the MMA never reads.  Box index i = 8 << i rows.
struct BBoxes {
  int i0, i1;  // i1 < 0: one box
  int rows;    // rows loaded (>= half)
};
__device__ __forceinline__ BBoxes b_boxes(int half) {
  BBoxes b;
  const int m8 = half >> 3;
  b.i0 = 31 - __clz(m8);
  const int rem = m8 - (1 << b.i0);
  b.i1 = rem ? 32 - __clz(rem - 1) : -1;  // ceil(log2(rem))
  b.rows = (8 << b.i0) + (rem ? 8 << b.i1 : 0);
  return b;
}

// The tile record the leader's producer publishes through the tile queue:
// {t, q, r0, rows | m << 16}; every other role rebuilds the TileCoord from it
// with a few integer ops instead of a search over tile_off (a chain of
// dependent L2 loads, ~1 us at every tile start in every role).
__device__ __forceinline__ TileCoord coord_of(const GemmParams &p, const int4 rec) {
  TileCoord c;
  c.q = rec.y;
  c.r0 = rec.z;
  c.rows = rec.w & 0xFFFF;
  c.m = rec.w >> 16;
  if (c.rows > p.tile_n) {
    c.half = p.tile_n >> 1;
    c.half_hi = rows_per_cta(c.rows - p.tile_n);
  } else {
    c.half = rows_per_cta(c.rows);
    c.half_hi = 0;
  }
  return c;
}

// Tile t -> its record (warp-cooperative): the group is found by counting the tile_off
// prefix entries <= t with all lanes (one round of independent loads), then
// four lanes load the group's bounds.  Returns the record (all lanes).
__device__ __forceinline__ int4 tile_locate(const GemmParams &p, int t_in, int total, int lane) {
  if (t_in >= total) return make_int4(t_in, 0, 0, 0);
  const int base = p.tile_off[p.q_begin];
  // draws alternate between the front and the back of the list: replica order
  // follows placement order (hot experts first, experts.cpp place_replicas), so
  // tensor-bound hot tiles and weight-streaming cold tiles run side by side
  const int t = (t_in & 1) ? total - 1 - (t_in >> 1) : (t_in >> 1);
  int q = p.q_begin;
  for (int j0 = p.q_begin + 1; j0 < p.q_end; j0 += 128) {
    int v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + 32 * u + lane;
      v[u] = j < p.q_end ? (p.tile_off[j] - base) * p.m_tiles : INT_MAX;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) q += __popc(__ballot_sync(0xffffffffu, v[u] <= t));
  }
  int w = 0;  // lanes 0..3: tile_off[q], tile_off[q+1], group_off[q], group_off[q+1]
  if (lane < 4) w = lane < 2 ? p.tile_off[q + lane] : p.group_off[q + lane - 2];
  const int to0 = __shfl_sync(0xffffffffu, w, 0), to1 = __shfl_sync(0xffffffffu, w, 1);
  const int g0 = __shfl_sync(0xffffffffu, w, 2), g1 = __shfl_sync(0xffffffffu, w, 3);
  const int nt = to1 - to0;
  const int local = t - (to0 - base) * p.m_tiles;
  const int m = local / nt, n = local % nt;
  const int r0 = g0 + n * p.tile_n;
  const int rows = n == nt - 1 ? g1 - r0 : p.tile_n;
  return make_int4(t_in, q, r0, rows | m << 16);
}

template <int MODE, int BH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ GemmParams p) {
  constexpr int kStages = Ring<BH>::kStages;
  constexpr int kStageBytes = Ring<BH>::kStageBytes;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *stage_base = smem;
  unsigned char *epi_base = smem + kStages * kStageBytes;  // per epilogue warp: staging
  uint64_t *bars = reinterpret_cast<uint64_t *>(epi_base + kEpiWarps * kWarpStaging);
  uint64_t *full = bars;                      // [kStages] leader: TMA bytes of both CTAs
  uint64_t *empty = bars + kStages;           // [kStages] both: MMA done with the stage
  uint64_t *tfull = bars + 2 * kStages;       // [2]       both: accumulator ready
  uint64_t *tempty = bars + 2 * kStages + 2;  // [2]       leader: both epilogues drained it
  uint64_t *tq_full = bars + 2 * kStages + 4;  // [kTQ]   both: tile index published
  uint64_t *tq_empty = tq_full + kTQ;          // [kTQ]   leader: every consumer read it
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tq_empty + kTQ);
  int4 *tq = reinterpret_cast<int4 *>(tmem_holder + 4);  // [kTQ] tile records (16-B aligned)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int kblocks = p.K / kBK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tm_a);
    for (int i = 0; i < 5; ++i) prefetch_tmap(&p.tm_b[i]);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * kEpiWarps);  // epilogue warps of both CTAs
    }
    for (int s = 0; s < kTQ; ++s) {
      mbar_init(&tq_full[s], 1);
      mbar_init(&tq_empty[s], kTQConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();
  pdl_wait();  // token rows (K3 / the gate-up GEMM) and the tile list (K1): read below only
  const int total = (p.tile_off[p.q_end] - p.tile_off[p.q_begin]) * p.m_tiles;

  // Dynamic tile scheduler: the leader's producer takes tile indices from a
  // global counter (one tile ahead) and publishes each through a kTQ-slot
  // queue in both CTAs' smem; the other roles of the pair read them from
  // there.  Pairs that draw cheap tiles draw more of them.
  if (warp == 0) {
    // ============ weight (A) producer + tile fetch (both CTAs) ============
    const uint64_t pol_w = policy_evict_first();  // weights: streamed once
    int nst = 0;  // trace: stages so far
    int stage = 0;
    uint32_t phase = 0;
    int slot = 0;
    uint32_t tq_phase = 0;
    int4 rec = make_int4(0, 0, 0, 0);
    if (leader) {
      int t0 = 0;
      if (lane == 0) t0 = (int)atomicAdd(p.ctr, 1u);
      rec = tile_locate(p, __shfl_sync(0xffffffffu, t0, 0), total, lane);
    }
    while (true) {
      if (leader) {
        mbar_wait(&tq_empty[slot], tq_phase ^ 1);
        if (elect_one()) {
          const uint32_t dst = smem_u32(&tq[slot]), bar = smem_u32(&tq_full[slot]);
          publish_v4(mapa(dst, 0), rec, mapa(bar, 0));
          publish_v4(mapa(dst, 1), rec, mapa(bar, 1));
        }
        __syncwarp();
      } else {
        mbar_wait(&tq_full[slot], tq_phase);
        rec = ld_shared_v4(&tq[slot]);
        __syncwarp();
        if (elect_one()) mbar_arrive_cluster_relaxed(mapa(smem_u32(&tq_empty[slot]), 0));
      }
      if (++slot == kTQ) {
        slot = 0;
        tq_phase ^= 1;
      }
      const int t = rec.x;
      if (t >= total) break;
      int t_next = 0;  // drawn one tile ahead; located after this tile's loads
      if (leader && lane == 0) t_next = (int)atomicAdd(p.ctr, 1u);
      const TileCoord c = coord_of(p, rec);
      if (p.trace && leader && lane == 0) {
        p.trace[kTW * t] = gtimer();
        p.trace[kTW * t + 4] = smid() | (unsigned long long)c.q << 16 |
                             (unsigned long long)c.rows << 32 | (unsigned long long)c.m << 48;
      }
      const uint32_t bbytes = 2u * kBK * 2;  // per token row of the pair
      const uint32_t bytes_pair = 2u * kATileBytes + bbytes * b_boxes(c.half).rows;
      const int rowq = (c.q - p.q_begin) * p.m_per_q;
      const unsigned long long a0 = p.trace ? gtimer() : 0;
      unsigned long long a_acq = 0;
      for (int kb = 0; kb < kblocks; ++kb) {
        const unsigned long long w0 = p.trace ? gtimer() : 0;
        mbar_wait(&empty[stage], phase ^ 1);
        if (p.trace) {
          const unsigned long long w1 = gtimer();
          a_acq += w1 - w0;
          if (blockIdx.x == 0 && lane == 0 && nst < 2048) p.trace[kStageLog + 4 * nst] = w1;
          ++nst;
        }
        unsigned char *sa = stage_base + stage * kStageBytes;
        const uint32_t bar = mapa(smem_u32(&full[stage]), 0);
        if (elect_one()) {
          if (leader) mbar_expect_tx(&full[stage], bytes_pair);  // A and B bytes of both CTAs
          if (MODE == kSwiglu) {
            // this CTA's 64 features as 8 blocks of (8 gate rows, 8 up rows)
            const int f0 = c.m * 128 + (int)crank * 64;
            tma_load_pair_4d(sa, &p.tm_a, bar, kb * kBK, (rowq + f0) >> 3, pol_w);
          } else {
            tma_load_pair(sa, &p.tm_a, bar, kb * kBK, rowq + c.m * 256 + (int)crank * 128, pol_w);
          }
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
        if (c.half_hi) {  // wide tile: the next stage carries only the second sub-tile's B
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader && elect_one()) mbar_expect_tx(&full[stage], bbytes * b_boxes(c.half_hi).rows);
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (p.trace && leader && lane == 0) {
        p.trace[kTW * t + 8] = a_acq;
        p.trace[kTW * t + 9] = gtimer() - a0;
      }
      if (leader) rec = tile_locate(p, __shfl_sync(0xffffffffu, t_next, 0), total, lane);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (leader) {
      int stage = 0, nst = 0;
      uint32_t phase = 0;
      uint32_t use = 0;  // accumulator uses so far: buffer use&1, phase (use>>1)&1
      int slot = 0;
      uint32_t tq_phase = 0;
      while (true) {
        const unsigned long long t_q = p.trace ? gtimer() : 0;
        mbar_wait(&tq_full[slot], tq_phase);
        const int4 rec = ld_shared_v4(&tq[slot]);
        const int t = rec.x;
        __syncwarp();
        if (elect_one()) mbar_arrive_cluster_relaxed(mapa(smem_u32(&tq_empty[slot]), 0));
        if (++slot == kTQ) {
          slot = 0;
          tq_phase ^= 1;
        }
        if (t >= total) break;
        unsigned long long t_wait = 0;  // trace: time spent waiting for stages
        const unsigned long long t_read = p.trace ? gtimer() : 0;
        const TileCoord c = coord_of(p, rec);
        const bool wide = c.half_hi != 0;
        const uint32_t idesc = idesc_bf16_m256(2 * c.half);
        const uint32_t idesc_hi = idesc_bf16_m256(wide ? 2 * c.half_hi : 16);
        const uint32_t d = tmem_base + (use & 1) * 256, d_hi = tmem_base + ((use + 1) & 1) * 256;
        mbar_wait(&tempty[use & 1], ((use >> 1) & 1) ^ 1);
        if (wide) mbar_wait(&tempty[(use + 1) & 1], (((use + 1) >> 1) & 1) ^ 1);
        tc_fence_after();
        if (p.trace && lane == 0) {
          p.trace[kTW * t + 1] = gtimer();
          p.trace[kTW * t + 5] = t_q;
        }
        if (!wide) {
          for (int kb = 0; kb < kblocks; ++kb) {
            const unsigned long long w0 = p.trace ? gtimer() : 0;
            mbar_wait(&full[stage], phase);
            if (p.trace) {
              const unsigned long long w1 = gtimer();
              t_wait += w1 - w0;
              if (blockIdx.x == 0 && lane == 0 && nst < 2048) p.trace[kStageLog + 4 * nst + 2] = w1;
              ++nst;
            }
            tc_fence_after();
            const uint32_t sa = smem_u32(stage_base + stage * kStageBytes);
            const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kATileBytes);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                umma_pair(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
              umma_commit_pair(&empty[stage]);
            }
            __syncwarp();
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        } else {
          // wide tile: stage s1 = weights + first sub-tile's rows, s2 = second
          // sub-tile's rows; both sub-tiles reuse the weight k-block of s1
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            const int s1 = stage;
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
            mbar_wait(&full[stage], phase);
            const int s2 = stage;
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
            tc_fence_after();
            const uint32_t sa = smem_u32(stage_base + s1 * kStageBytes);
            const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kATileBytes);
            const uint64_t db2 = sw128_desc(smem_u32(stage_base + s2 * kStageBytes) + kATileBytes);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                umma_pair(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                umma_pair(d_hi, da + 2 * k, db2 + 2 * k, idesc_hi, (kb | k) != 0);
              umma_commit_pair(&empty[s1]);
              umma_commit_pair(&empty[s2]);
            }
            __syncwarp();
          }
        }
        if (elect_one()) {
          umma_commit_pair(&tfull[use & 1]);
          if (wide) umma_commit_pair(&tfull[(use + 1) & 1]);
        }
        __syncwarp();
        if (p.trace && lane == 0) {
          p.trace[kTW * t + 6] = t_wait | (t_read - t_q) << 32;
          p.trace[kTW * t + 7] = gtimer();
        }
        use += wide ? 2 : 1;
      }
    }
  } else if (warp == 2 + kEpiWarps) {
    // ============ token-row (B) producer (both CTAs) ============
    // A separate warp from the weight producer: the per-k-block TMA issue
    // cost of one warp was measurable on the critical path.
    {
      const uint64_t pol_x = policy_evict_last();  // token rows: reused by every m-block
      int stage = 0, nst = 0;
      uint32_t phase = 0;
      int slot = 0;
      uint32_t tq_phase = 0;
      while (true) {
        mbar_wait(&tq_full[slot], tq_phase);
        const int4 rec = ld_shared_v4(&tq[slot]);
        const int t = rec.x;
        __syncwarp();
        if (elect_one()) mbar_arrive_cluster_relaxed(mapa(smem_u32(&tq_empty[slot]), 0));
        if (++slot == kTQ) {
          slot = 0;
          tq_phase ^= 1;
        }
        if (t >= total) break;
        const TileCoord c = coord_of(p, rec);
        const BBoxes bx0 = b_boxes(c.half), bx1 = b_boxes(c.half_hi ? c.half_hi : 8);
        const unsigned long long b0 = p.trace ? gtimer() : 0;
        unsigned long long b_acq = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
          for (int sub = 0; sub < (c.half_hi ? 2 : 1); ++sub) {
            const int half = sub ? c.half_hi : c.half;
            const int brow = c.r0 + sub * p.tile_n + (int)crank * half;
            const unsigned long long w0 = p.trace ? gtimer() : 0;
            mbar_wait(&empty[stage], phase ^ 1);
            if (p.trace) {
              const unsigned long long w1 = gtimer();
              b_acq += w1 - w0;
              if (blockIdx.x == 0 && lane == 0 && nst < 2048) {
                p.trace[kStageLog + 4 * nst + 1] = w1;
                p.trace[kStageLog + 4 * nst + 3] = c.half + c.half_hi;
              }
              ++nst;
            }
            unsigned char *sb = stage_base + stage * kStageBytes + kATileBytes;
            const uint32_t bar = mapa(smem_u32(&full[stage]), 0);
            if (elect_one()) {
              // boxes of 128/64/32/16/8 rows land on 8-row = 1024-B swizzle atoms
              const BBoxes bx = sub ? bx1 : bx0;
              tma_load_pair(sb, &p.tm_b[bx.i0], bar, kb * kBK, brow, pol_x);
              if (bx.i1 >= 0) {
                const int off = 8 << bx.i0;
                tma_load_pair(sb + off * 128, &p.tm_b[bx.i1], bar, kb * kBK, brow + off, pol_x);
              }
            }
            __syncwarp();
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        if (p.trace && leader && lane == 0) {
          p.trace[kTW * t + 10] = b_acq;
          p.trace[kTW * t + 11] = gtimer() - b0;
        }
      }
    }
  } else {
    // ============ epilogue (warps 2.., both CTAs) ============
    // Warp w drains TMEM lanes 32*(w%4).. +31 of the 32-column chunks grp,
    // grp + kEpiGroups, ... of each accumulator (grp = (w-2)/4): two warps per
    // SM sub-partition hide each other's tcgen05.ld / store latency, and each
    // warp transposes through its own smem (no cross-warp barrier).
    const int quad = warp & 3;  // TMEM lane quarter (warp % 4 rule)
    const int grp = (warp - 2) >> 2;
    __nv_bfloat16 *stg = reinterpret_cast<__nv_bfloat16 *>(epi_base + (warp - 2) * kWarpStaging);
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa(smem_u32(&tempty[1]), 0);
    uint32_t use = 0;  // accumulator uses (same sequence as the MMA issuer)
    int slot = 0;
    uint32_t tq_phase = 0;
    while (true) {
      mbar_wait(&tq_full[slot], tq_phase);
      const int4 rec = ld_shared_v4(&tq[slot]);
      const int t = rec.x;
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(mapa(smem_u32(&tq_empty[slot]), 0));
      if (++slot == kTQ) {
        slot = 0;
        tq_phase ^= 1;
      }
      if (t >= total) break;
      const TileCoord c = coord_of(p, rec);
      for (int sub = 0; sub < (c.half_hi ? 2 : 1); ++sub, ++use) {
      const int acc = use & 1;
      mbar_wait(&tfull[acc], (use >> 1) & 1);
      tc_fence_after();
      if (p.trace && leader && warp == 2 && lane == 0 && sub == 0) p.trace[kTW * t + 2] = gtimer();
      const uint32_t d = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * 256;
      // accumulator column j <-> token row sr0 + j (CTA 0 loaded rows [0, half),
      // CTA 1 rows [half, 2*half) of the sub-tile)
      const int sr0 = c.r0 + sub * p.tile_n;
      const int srows = sub ? c.rows - p.tile_n : min(c.rows, p.tile_n);
      for (int c0 = grp * kEpiCols; c0 < srows; c0 += kEpiGroups * kEpiCols) {
        const int rows = min(kEpiCols, srows - c0);
        // Output block of this warp: 32 token rows x kF features (SWIGLU: 16
        // features of h, PLAIN: 32 of y).  The 16x256b TMEM shape hands each
        // thread the mma-fragment layout (feature lane/4 and lane/4+8, token
        // pair 2*(lane%4)), which stmatrix.trans writes into the staging tile
        // as [token][feature] rows; one TMA store then moves the block.
        constexpr int kF = MODE == kSwiglu ? 16 : 32;
        const int f_base = MODE == kSwiglu ? c.m * 128 + (int)crank * 64 + quad * 16
                                           : c.m * 256 + (int)crank * 128 + quad * 32;
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free again
        __syncwarp();
        const uint32_t stg_a = smem_u32(stg);
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // TMEM lanes 16h..16h+15 of this warp's quarter
          uint32_t r[16];
          tmem_ld_16x256b_x4(d + ((uint32_t)(16 * h) << 16) + c0, r);
          uint32_t pk[8];  // pk[2i + j]: feature block j of this 16-lane group, tokens 8i..8i+7
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (MODE == kSwiglu) {
              // lanes 16h..+7 gate, 16h+8..+15 up of features 8h..8h+7
              float hv[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const float g = __uint_as_float(r[4 * i + e]), u = __uint_as_float(r[4 * i + 2 + e]);
                hv[e] = __fdividef(g, 1.0f + __expf(-g)) * u;
              }
              pk[2 * i] = pack_bf16(hv[0], hv[1]);
            } else {
              pk[2 * i] = pack_bf16(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]));
              pk[2 * i + 1] = pack_bf16(__uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
            }
          }
          // 8x8 matrices (feature block fb, token block i) -> staging rows 8i..8i+7
          const int q8 = lane >> 3, rr = lane & 7;
          if (MODE == kSwiglu) {
            // features 8h..8h+7 of this warp's 16: one x4 per (h), token blocks 0..3
            stmatrix_x4_trans(stg_a + ((8 * q8 + rr) * kF + 8 * h) * 2, pk[0], pk[2], pk[4], pk[6]);
          } else {
#pragma unroll
            for (int x = 0; x < 2; ++x) {  // token blocks 2x, 2x+1; feature blocks 2h, 2h+1
              const int fb = 2 * h + (q8 & 1), i = 2 * x + (q8 >> 1);
              stmatrix_x4_trans(stg_a + ((8 * i + rr) * kF + 8 * fb) * 2, pk[4 * x], pk[4 * x + 1],
                                pk[4 * x + 2], pk[4 * x + 3]);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging -> TMA (async proxy)
        __syncwarp();
        if (rows == kEpiCols) {
          if (elect_one()) {
            tma_store_2d(&p.tm_out, stg_a, f_base, sr0 + c0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          __syncwarp();
        } else {  // ragged tail of the sub-tile: 16-B stores
          __nv_bfloat16 *obase = p.out + (size_t)(sr0 + c0) * p.out_ld + f_base;
          constexpr int kV = kF / 8;  // 16-B pieces per row
          for (int i = lane; i < rows * kV; i += 32) {
            const int rw = i / kV, ch = i % kV;
            *reinterpret_cast<uint4 *>(obase + (size_t)rw * p.out_ld + ch * 8) =
                *reinterpret_cast<const uint4 *>(stg + rw * kF + ch * 8);
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      __syncwarp();
      // relaxed: only the TMEM reads (complete: tcgen05.wait::ld, fenced
      // above) must precede the MMA's reuse of the accumulator; a release
      // arrive would also wait for this warp's global stores to be acked
      if (lane == 0) mbar_arrive_cluster_relaxed(acc ? tempty_leader1 : tempty_leader0);
      if (p.trace && lane == 0) atomicMax(&p.trace[kTW * t + 3], gtimer());  // last warp of the pair
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // epilogue TMA stores done
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x == 0) {  // the last CTA to finish resets the tile counter for the next launch
    __threadfence();
    if (atomicAdd(p.ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(p.ctr, 0u);
      atomicExch(p.ctr + 1, 0u);
    }
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
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




// Epilogue output map: bf16 [rows][cols], no swizzle, box {box_cols, 32 rows}.
bool make_out_map(CUtensorMap *tm, const void *base, uint64_t rows, uint64_t cols,
                  uint32_t box_cols) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, 32};
  cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The gate/up weight store [Q][gate d_e | up d_e][d_h] as a 4-D map {k, row in
// an 8-row block, gate/up (+d_e rows), 8-row block}: one box {64, 8, 2, 8}
// lands as 8 x (8 gate rows, the 8 up rows of the same features) — the row
// order the SwiGLU epilogue's 16x256b TMEM loads pair up.
bool make_w13_map(CUtensorMap *tm, const void *base, uint64_t Q, uint64_t d_e, uint64_t d_h) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {d_h, 8, 2, (Q * 2 * d_e - d_e) / 8};
  cuuint64_t strides[3] = {d_h * 2, d_e * d_h * 2, 8 * d_h * 2};
  cuuint32_t box[4] = {64, 8, 2, 8};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

namespace {
unsigned long long *g_trace = nullptr;
}  // namespace

cudaError_t build_ffn_tensor_maps(FfnPlan &p) {
  // the tile-timeline buffer (debug), allocated here: never during a capture
  static const bool trace = getenv("JANUS_GEMM_TRACE") && atoi(getenv("JANUS_GEMM_TRACE"));
  if (trace && !g_trace &&
      cudaMalloc(&g_trace, 2ull * kTraceTiles * kTW * sizeof(unsigned long long)) != cudaSuccess)
    return cudaErrorMemoryAllocation;
  const int Q = p.q_end - p.q_begin;
  bool ok = make_w13_map(&p.tm_w13, p.w13, Q, p.d_e, p.d_h) &&
            make_map(&p.tm_w2, p.w2, (uint64_t)Q * p.d_h, p.d_e, 128);
  for (int i = 0; i < 5 && ok; ++i) {
    ok = make_map(&p.tm_xp[i], p.xp, p.S_alloc, p.d_h, 8u << i) &&
         make_map(&p.tm_h[i], p.h, p.S_alloc, p.d_e, 8u << i);
  }
  if (ok) {
    ok = make_out_map(&p.tm_h_out, p.h, p.S_alloc, p.d_e, 16) &&
         make_out_map(&p.tm_y_out, p.y, p.S_alloc, p.d_h, 32) &&
         (!p.y2 || make_out_map(&p.tm_y_out2, p.y2, p.S_alloc, p.d_h, 32));
  }
  p.maps_ready = ok;
  return ok ? cudaSuccess : cudaErrorInvalidValue;
}

namespace {

template <int MODE, int BH>
cudaError_t launch_gemm(const GemmParams &g, cudaStream_t s) {
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(grouped_gemm_kernel<MODE, BH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Ring<BH>::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured_dev = dev;
  }
  const int grid = sm_count() & ~1;  // CTA pairs
  return launch_pdl(grouped_gemm_kernel<MODE, BH>, dim3(grid), dim3(kGemmThreads),
                    Ring<BH>::kSmemBytes, s, g);
}

}  // namespace

cudaError_t launch_ffn(const FfnPlan &p, const int32_t *group_off, const int32_t *tile_off,
                       cudaStream_t s, int *launches, int ybuf) {
  GemmParams g{};
  g.trace = g_trace;
  g.group_off = group_off;
  g.tile_off = tile_off;
  g.tile_n = p.tile_n;
  g.ctr = p.tile_ctr;
  g.q_begin = p.q_begin;
  g.q_end = p.q_end;
  const bool decode = p.tile_n <= 64;

  // gate + up -> h: per replica A rows [gate d_e | up d_e]; 128 features per tile
  g.tm_a = p.tm_w13;
  for (int i = 0; i < 5; ++i) g.tm_b[i] = p.tm_xp[i];
  g.tm_out = p.tm_h_out;
  g.K = p.d_h;
  g.m_tiles = p.d_e / 128;
  g.m_per_q = 2 * p.d_e;
  g.up_off = p.d_e;
  g.out = reinterpret_cast<__nv_bfloat16 *>(p.h);
  g.out_ld = p.d_e;
  cudaError_t err = decode ? launch_gemm<kSwiglu, 32>(g, s) : launch_gemm<kSwiglu, 128>(g, s);
  if (err != cudaSuccess) return err;

  // down: y = h Wd^T, 256 output features per tile
  g.tm_a = p.tm_w2;
  for (int i = 0; i < 5; ++i) g.tm_b[i] = p.tm_h[i];
  const bool alt = ybuf && p.y2;
  g.tm_out = alt ? p.tm_y_out2 : p.tm_y_out;
  g.ctr = p.tile_ctr + 2;
  g.K = p.d_e;
  g.m_tiles = p.d_h / 256;
  g.m_per_q = p.d_h;
  g.up_off = 0;
  g.out = reinterpret_cast<__nv_bfloat16 *>(alt ? p.y2 : p.y);
  g.out_ld = p.d_h;
  if (g.trace) g.trace += (size_t)kTraceTiles * kTW;
  err = decode ? launch_gemm<kPlain, 32>(g, s) : launch_gemm<kPlain, 128>(g, s);
  if (launches) *launches += 2;
  return err;
}

}  // namespace janus

// Debug: copy the traced FFN tile timeline ([2 GEMMs][16384 tiles][16] u64) to
// host and clear it; JANUS_ESTATE when JANUS_GEMM_TRACE was not set.
extern "C" int janus_debug_ffn_trace(unsigned long long *host, int cap_words) {
  if (!janus::g_trace) return 4;
  const size_t n = std::min((size_t)cap_words, (size_t)2 * janus::kTraceTiles * janus::kTW);
  if (cudaMemcpy(host, janus::g_trace, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 3;
  // cleared after the read: the next read holds only tiles drawn after this one
  return cudaMemset(janus::g_trace, 0, 2ull * janus::kTraceTiles * janus::kTW * 8) == cudaSuccess ? 0 : 3;
}
