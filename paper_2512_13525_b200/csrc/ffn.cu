// ffn.cu — K3 permute, K4 grouped SwiGLU expert GEMMs (tcgen05 + TMA + TMEM),
// K5 combine.  sm_100a only.
//
// The expert FFN has no reference implementation: the reference models it as
// t_launch + max(A*W_e/beta, 2*b*d_h*d_e/pi) (src/latency.cpp:17-24).  Here it
// is computed for real:
//   h = silu(x Wg^T) * (x Wu^T)          (kernel mode SWIGLU, h kept in bf16)
//   y = h Wd^T                           (kernel mode PLAIN)
//   out[t] = sum_j w[t,j] y[row(t,j)]    (combine, fixed j order, fp32)
//
// Grouped GEMM, swap-AB: the weight rows are the UMMA M side (128 per
// instruction), the ragged token rows of one replica group are the N side
// (16..128, one of four TMA boxes), K is the reduction dim.  A tile is one
// replica group q, one 2x128-row weight block, one <=128-row token block:
//   A0, A1  two 128x64 bf16 weight tiles per k-block (gate+up, or two halves of
//           the down projection), SWIZZLE_128B, TMA
//   B       the token tile, shared by both MMAs
//   D0, D1  two fp32 accumulators in TMEM (128 lanes x N columns each),
//           double-buffered across tiles (4 x 128 of the 512 columns)
// Warp roles (192 threads, one CTA per SM, persistent over the tile list):
//   warp 0  TMA producer      warp 1  TMEM owner + single-thread MMA issuer
//   warps 2-5 epilogue: tcgen05.ld -> SwiGLU / bf16 pack -> smem -> 16B stores
// The tile list (groups x n-blocks x m-blocks) is read from device memory
// (group_off / tile_off written by the scheduler kernel): no host sync.
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"

namespace janus {
namespace {

constexpr int kBK = 64;              // K elements per stage (128 B rows, SW128)
constexpr int kStages = 4;
constexpr int kATileBytes = 128 * kBK * 2;    // 16 KB
constexpr int kBTileBytes = kTileN * kBK * 2; // 16 KB (max box)
constexpr int kStageBytes = 2 * kATileBytes + kBTileBytes;
constexpr int kEpiRows = 32;                  // token rows per epilogue chunk
constexpr int kStagingBytes = kEpiRows * 256 * 2;  // 32 rows x 256 bf16
constexpr int kGemmThreads = 192;
constexpr int kTmemCols = 512;
constexpr int kSmemBytes = kStages * kStageBytes + kStagingBytes + 1024 /*align*/ + 256;

enum Mode { kSwiglu = 0, kPlain = 1 };

struct GemmParams {
  CUtensorMap tm_a;     // weights [Q*M_per_q][K]
  CUtensorMap tm_b[4];  // activations [S_alloc][K], box rows 16/32/64/128
  const int32_t *group_off;
  const int32_t *tile_off;
  int q_begin, q_end;
  int K;          // reduction length
  int m_tiles;    // weight blocks per group
  int m_per_q;    // weight rows per replica
  int a1_off;     // row offset of A1 inside a block pair (SWIGLU: d_e; PLAIN: 128)
  int a_blk;      // row stride between m-blocks (SWIGLU: 128; PLAIN: 256)
  __nv_bfloat16 *out;
  int out_ld;     // elements per output row
  int out_blk;    // output features per tile (SWIGLU 128, PLAIN 256)
};

// ---------------------------------------------------------------- PTX -----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, uint64_t *bar,
                                            int x, int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// SW128 K-major smem matrix descriptor (cute::UMMA::SmemDescriptor layout):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major), SBO>>4
// [32,46) = 1024 B between 8-row groups, version 1 [46,48), layout 2 = 128B
// swizzle [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128.
__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
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
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct TileCoord {
  int q, m, r0, rows;
};

// Tile t (relative to the first tile of q_begin) -> (group, m-block, rows).
__device__ __forceinline__ TileCoord tile_coord(const GemmParams &p, int t) {
  const int base = p.tile_off[p.q_begin];
  int lo = p.q_begin, hi = p.q_end;  // find q: (tile_off[q]-base)*m <= t < (tile_off[q+1]-base)*m
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((p.tile_off[mid] - base) * p.m_tiles <= t) lo = mid;
    else hi = mid;
  }
  const int q = lo;
  const int nt = p.tile_off[q + 1] - p.tile_off[q];
  const int local = t - (p.tile_off[q] - base) * p.m_tiles;
  TileCoord c;
  c.q = q;
  c.m = local / nt;
  const int n = local % nt;
  c.r0 = p.group_off[q] + n * kTileN;
  c.rows = min(kTileN, p.group_off[q + 1] - c.r0);
  return c;
}

__device__ __forceinline__ int box_index(int rows) {
  return rows <= 16 ? 0 : rows <= 32 ? 1 : rows <= 64 ? 2 : 3;
}

template <int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *stage_base = smem;
  __nv_bfloat16 *staging = reinterpret_cast<__nv_bfloat16 *>(smem + kStages * kStageBytes);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes + kStagingBytes);
  uint64_t *full = bars;                  // [kStages]
  uint64_t *empty = bars + kStages;       // [kStages]
  uint64_t *tfull = bars + 2 * kStages;   // [2]
  uint64_t *tempty = bars + 2 * kStages + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * kStages + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = (p.tile_off[p.q_end] - p.tile_off[p.q_begin]) * p.m_tiles;
  const int kblocks = p.K / kBK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tm_a);
    for (int i = 0; i < 4; ++i) prefetch_tmap(&p.tm_b[i]);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once
      const uint64_t pol_x = policy_evict_last();   // token rows: reused by every m-block
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TileCoord c = tile_coord(p, t);
        const int bi = box_index(c.rows);
        const uint32_t bbytes = (16u << bi) * kBK * 2;
        const int arow = (c.q - p.q_begin) * p.m_per_q + c.m * p.a_blk;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char *sa = stage_base + stage * kStageBytes;
          mbar_expect_tx(&full[stage], 2 * kATileBytes + bbytes);
          tma_load_2d(sa, &p.tm_a, &full[stage], kb * kBK, arow, pol_w);
          tma_load_2d(sa + kATileBytes, &p.tm_a, &full[stage], kb * kBK, arow + p.a1_off, pol_w);
          tma_load_2d(sa + 2 * kATileBytes, &p.tm_b[bi], &full[stage], kb * kBK, c.r0, pol_x);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TileCoord c = tile_coord(p, t);
        const int n = 16 << box_index(c.rows);
        const uint32_t idesc = idesc_bf16(n);
        const uint32_t d0 = tmem_base + acc * 256, d1 = d0 + 128;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(stage_base + stage * kStageBytes);
          const uint64_t da0 = sw128_desc(sa), da1 = sw128_desc(sa + kATileBytes),
                         db = sw128_desc(sa + 2 * kATileBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint32_t accum = (kb | k) != 0;
            umma_bf16(d0, da0 + 2 * k, db + 2 * k, idesc, accum);
            umma_bf16(d1, da1 + 2 * k, db + 2 * k, idesc, accum);
          }
          umma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int quad = warp & 3;  // TMEM lanes quad*32 .. +31
    const int feat = quad * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..127
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const TileCoord c = tile_coord(p, t);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t d0 = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * 256;
      const uint32_t d1 = d0 + 128;
      const int out_w = p.out_blk;  // features per output row in this tile
      __nv_bfloat16 *obase = p.out + (size_t)c.r0 * p.out_ld + (size_t)c.m * p.out_blk;
      for (int c0 = 0; c0 < c.rows; c0 += kEpiRows) {
        float v0[32], v1[32];
        tmem_ld32(d0 + c0, v0);
        tmem_ld32(d1 + c0, v1);
        if (MODE == kSwiglu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float g = v0[j];
            const float h = g / (1.0f + __expf(-g)) * v1[j];
            staging[j * 128 + feat] = __float2bfloat16_rn(h);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            staging[j * 256 + feat] = __float2bfloat16_rn(v0[j]);
            staging[j * 256 + 128 + feat] = __float2bfloat16_rn(v1[j]);
          }
        }
        named_bar(1, 128);
        // cooperative 16 B stores of up to 32 rows x out_w features
        const int rows = min(kEpiRows, c.rows - c0);
        const int chunks_per_row = out_w / 8;
        for (int i = et; i < rows * chunks_per_row; i += 128) {
          const int r = i / chunks_per_row, ch = i % chunks_per_row;
          const uint4 v = *reinterpret_cast<const uint4 *>(staging + r * out_w + ch * 8);
          *reinterpret_cast<uint4 *>(obase + (size_t)(c0 + r) * p.out_ld + ch * 8) = v;
        }
        named_bar(1, 128);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

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

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  }
  return fn;
}

// 2-D bf16 row-major [rows][cols] tensor map, box {64, box_rows}, 128B swizzle.
bool make_map(CUtensorMap *tm, const void *base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t build_ffn_tensor_maps(FfnPlan &p) {
  const int Q = p.q_end - p.q_begin;
  bool ok = make_map(&p.tm_w13, p.w13, (uint64_t)Q * 2 * p.d_e, p.d_h, 128) &&
            make_map(&p.tm_w2, p.w2, (uint64_t)Q * p.d_h, p.d_e, 128);
  for (int i = 0; i < 4 && ok; ++i) {
    ok = make_map(&p.tm_xp[i], p.xp, p.S_alloc, p.d_h, 16u << i) &&
         make_map(&p.tm_h[i], p.h, p.S_alloc, p.d_e, 16u << i);
  }
  p.maps_ready = ok;
  return ok ? cudaSuccess : cudaErrorInvalidValue;
}

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

cudaError_t launch_ffn(const FfnPlan &p, const int32_t *group_off, const int32_t *tile_off,
                       cudaStream_t s, int *launches) {
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    cudaError_t e1 = cudaFuncSetAttribute(grouped_gemm_kernel<kSwiglu>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    cudaError_t e2 = cudaFuncSetAttribute(grouped_gemm_kernel<kPlain>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e1 != cudaSuccess) return e1;
    if (e2 != cudaSuccess) return e2;
    configured_dev = dev;
  }
  const int grid = sm_count();
  GemmParams g{};
  g.group_off = group_off;
  g.tile_off = tile_off;
  g.q_begin = p.q_begin;
  g.q_end = p.q_end;

  // gate + up -> h  (A rows: [gate d_e | up d_e] per replica)
  g.tm_a = p.tm_w13;
  for (int i = 0; i < 4; ++i) g.tm_b[i] = p.tm_xp[i];
  g.K = p.d_h;
  g.m_tiles = p.d_e / 128;
  g.m_per_q = 2 * p.d_e;
  g.a1_off = p.d_e;
  g.a_blk = 128;
  g.out = reinterpret_cast<__nv_bfloat16 *>(p.h);
  g.out_ld = p.d_e;
  g.out_blk = 128;
  grouped_gemm_kernel<kSwiglu><<<grid, kGemmThreads, kSmemBytes, s>>>(g);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;

  // down: y = h Wd^T (A rows: d_h per replica, 256-row blocks as two halves)
  g.tm_a = p.tm_w2;
  for (int i = 0; i < 4; ++i) g.tm_b[i] = p.tm_h[i];
  g.K = p.d_e;
  g.m_tiles = p.d_h / 256;
  g.m_per_q = p.d_h;
  g.a1_off = 128;
  g.a_blk = 256;
  g.out = reinterpret_cast<__nv_bfloat16 *>(p.y);
  g.out_ld = p.d_h;
  g.out_blk = 256;
  grouped_gemm_kernel<kPlain><<<grid, kGemmThreads, kSmemBytes, s>>>(g);
  if (launches) *launches += 2;
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
