// aebs.cu — K1+K2: the activation-balanced expert scheduler and the dispatch
// layout as ONE sm_100a kernel (one thread-block cluster of 1..8 CTAs).
//
// Replaces moesim::schedule (src/aebs.cpp:172-197: collect_activated :126-168,
// greedy :178-194, finish_assignment :89-122) and schedule_random (:250-262),
// bit-exact with schedule_reference (:199-248).
//
// The batch's T*k slots are cut into contiguous ranges: one per CTA of the
// cluster, then one per warp (32 warps per CTA), so every per-expert count is
// warp-private and the slot order is (CTA, warp, window, lane):
//   load    every warp issues all of its slot loads at once into registers
//           (MAXIT windows per lane) while the CTA stages the map tables in smem
//           — one memory latency for the batch instead of one per window.
//   pass 1  warp histogram: equal expert ids of a 32-slot window are grouped by
//           a peer mask built from log2(E) independent __ballot_sync (one per
//           id bit; MATCH.ANY serialises over distinct values and was ~1 µs per
//           window); the lowest peer adds __popc(peers) to the warp's row.
//   scan    per expert, exclusive prefix over the 32 warp rows -> this CTA's
//           total; ONE cluster barrier, then every CTA reads every CTA's totals
//           through DSMEM: global tot[e] and this CTA's starting rank.
//   decide  replicated in every CTA (identical inputs -> identical results, no
//           second exchange): pin single-replica experts; the order-dependent
//           greedy over multi-replica experts in ascending id (warp 0); the
//           finish pass (replica id, replica-order index q, routed tokens) and
//           block scans -> group_off[q] and the n-tile prefix for the GEMM.
//   pass 2  the same windows again (registers): row = group_off[q(e)] + CTA base
//           + warp base + rank in window -> slot_row (+ optional row_slot), and
//           the Assignment's per-slot instance / replica.
//
// The greedy (aebs.cpp:186-194: least-loaded host, ties to the lowest id) is a
// chain of dependent argmins, one warp-wide __reduce_min_sync per activated
// multi-replica expert (~40 cycles each).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>

#include "internal.h"

namespace cg = cooperative_groups;

namespace janus {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxCluster = 16;  // non-portable above 8 (one GPC holds 16+ SMs on B200)

__device__ __forceinline__ uint64_t splitmix64(uint64_t &s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// include/moesim/rng.hpp:53-61
__device__ __forceinline__ uint64_t next_below(uint64_t &s, uint64_t n) {
  uint64_t threshold = (0 - n) % n;
  for (;;) {
    uint64_t r = splitmix64(s);
    if (r >= threshold) return r % n;
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes of `valid` holding the same id as this lane: one ballot per id bit.
__device__ __forceinline__ unsigned peers_of(unsigned valid, int id, int nbits) {
  unsigned peers = valid;
#pragma unroll 4
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (id >> b) & 1;
    const unsigned m = __ballot_sync(kFull, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Exclusive scan of two int arrays of n entries in place (1024 threads).
__device__ void block_exscan2(int32_t *a, int32_t *b, int n, int32_t *scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + kSchedThreads - 1) / kSchedThreads;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int sa = 0, sb = 0;
  for (int i = lo; i < hi; ++i) {
    sa += a[i];
    sb += b[i];
  }
  int ia = sa, ib = sb;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int ta = __shfl_up_sync(kFull, ia, d), tb = __shfl_up_sync(kFull, ib, d);
    if (lane >= d) {
      ia += ta;
      ib += tb;
    }
  }
  if (lane == 31) {
    scratch[warp] = ia;
    scratch[32 + warp] = ib;
  }
  __syncthreads();
  if (warp == 0) {
    int wa = scratch[lane], wb = scratch[32 + lane];
    int xa = wa, xb = wb;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int ta = __shfl_up_sync(kFull, xa, d), tb = __shfl_up_sync(kFull, xb, d);
      if (lane >= d) {
        xa += ta;
        xb += tb;
      }
    }
    scratch[lane] = xa - wa;
    scratch[32 + lane] = xb - wb;
  }
  __syncthreads();
  int ra = scratch[warp] + ia - sa, rb = scratch[32 + warp] + ib - sb;
  for (int i = lo; i < hi; ++i) {
    int va = a[i], vb = b[i];
    a[i] = ra;
    b[i] = rb;
    ra += va;
    rb += vb;
  }
  __syncthreads();
}

// Greedy over multi-replica activated experts, N <= 32 instances (warp 0),
// aebs.cpp:186-194.  Lane g keeps key_g = load[g] << 5 | g in a register, so
// one step is: mask the expert's hosts (the mask is loaded ahead, off the
// dependency chain) -> __reduce_min_sync -> bump the winner's key.  The
// minimum key is the least load with ties to the lowest instance id.
__device__ void greedy_warp(int E, int N, const int32_t *tot, const int32_t *off,
                            const uint32_t *hm_tab, int32_t *load, int32_t *chg) {
  const int lane = threadIdx.x & 31;
  uint32_t key = lane < N ? ((uint32_t)load[lane] << 5) | (uint32_t)lane : 0xffffffffu;
  for (int cb = 0; cb < E; cb += 32) {
    const int e = cb + lane;
    const bool multi = e < E && tot[e] > 0 && off[e + 1] - off[e] > 1;
    unsigned mm = __ballot_sync(kFull, multi);
    const uint32_t myhm = multi ? hm_tab[e] : 0u;
    while (mm) {
      const int b = __ffs(mm) - 1;
      mm &= mm - 1;
      const uint32_t drop = ((__shfl_sync(kFull, myhm, b) >> lane) & 1u) ? 0u : 0xffffffffu;
      const uint32_t win = __reduce_min_sync(kFull, key | drop);
      key += (key == win) ? 32u : 0u;
      if (lane == b) chg[e] = (int)(win & 31u);
    }
  }
  if (lane < N) load[lane] = (int)(key >> 5);
}

// Slot source: MAXIT > 0 keeps this warp's ids in registers (window i at
// v[i]); MAXIT == 0 streams them from global memory (very large batches).
template <int MAXIT>
struct Slots {
  int v[MAXIT];
  __device__ __forceinline__ void load(const int32_t *__restrict__ ex, int beg, int end, int lane,
                                       int nit) {
#pragma unroll
    for (int i = 0; i < MAXIT; ++i) {
      const int s = beg + i * 32 + lane;
      v[i] = (i < nit && s < end) ? __ldg(ex + s) : 0;
    }
  }
  __device__ __forceinline__ int get(const int32_t *__restrict__, int i, int) const { return v[i]; }
};
template <>
struct Slots<0> {
  __device__ __forceinline__ void load(const int32_t *, int, int, int, int) {}
  __device__ __forceinline__ int get(const int32_t *__restrict__ ex, int, int s) const {
    return __ldg(ex + s);
  }
};

// A rejected step (unknown expert, or the exchange aborted it) still leaves a
// layout the layer's later kernels can run on safely: no replica groups, no
// GEMM tiles, every slot unrouted.  K3 / K5 also check status[0] and skip.
// Called by every thread of one CTA.
__device__ void write_error_layout(const SchedArgs &a, int status, int bad) {
  const int R = a.map.R;
  for (int q = threadIdx.x; q <= R; q += kSchedThreads) {
    if (a.out.group_off) a.out.group_off[q] = 0;
    if (a.tile_off) a.tile_off[q] = 0;
  }
  if (a.shared_off && threadIdx.x < 4) a.shared_off[threadIdx.x] = 0;
  for (int s = threadIdx.x; s < a.S; s += kSchedThreads) a.out.instance[s] = -1;
  if (threadIdx.x == 0) {
    a.out.status[0] = status;
    a.out.status[1] = bad;
  }
}

template <int MAXIT>
__global__ void __launch_bounds__(kSchedThreads, 1) aebs_schedule_kernel(SchedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  // the layer's next kernel (K3, launched with PDL) may become resident now;
  // it waits for this grid's completion before reading the layout
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank(), csize = (int)cluster.num_blocks();
  const int E = a.map.E, N = a.map.N, R = a.map.R, S = a.S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool leader = crank == 0;  // writes the per-expert / per-instance outputs
  uint64_t *trace = leader ? a.trace : nullptr;
  if (trace && tid == 0) trace[0] = globaltimer();
  // the box exchange aborted this step (a peer never published its rows)
  if (a.abort_flag && *a.abort_flag) {
    if (leader) write_error_layout(a, JANUS_EPEER, 0);
    return;  // before any cluster barrier: every CTA reads the same flag
  }

  // routed counts fit 32 bits (S < 2^31): 32-bit shared atomics are native.
  unsigned *routed = reinterpret_cast<unsigned *>(smem);        // [N]
  int32_t *cnt = reinterpret_cast<int32_t *>(routed + N);       // [32][E]
  int32_t *tot = cnt + 32 * E;                                  // [E] cluster totals
  int32_t *ltot = tot + E;                                      // [E] this CTA's totals
  int32_t *xbase = ltot + E;                                    // [E] ranks before this CTA
  int32_t *chg = xbase + E;                                     // [E]
  int32_t *qof = chg + E;                                       // [E]
  int32_t *ridof = qof + E;                                     // [E]
  int32_t *load = ridof + E;                                    // [N]
  int32_t *qcnt = load + N;                                     // [R+1]
  int32_t *tcnt = qcnt + R + 1;                                 // [R+1]
  int32_t *s_off = tcnt + R + 1;                                // [E+1]
  int32_t *s_hosts = s_off + E + 1;                             // [R]
  int32_t *s_rid = s_hosts + R;                                 // [R]
  int32_t *s_qidx = s_rid + R;                                  // [R]
  uint32_t *s_hm = reinterpret_cast<uint32_t *>(s_qidx + R);    // [E]
  __shared__ int32_t s_bad;
  __shared__ int32_t s_scan[64];

  // ---- slot ranges: CTA, then warp; issue every slot load at once ----------
  const int windows = (S + 31) / 32;
  const int cwin = (windows + csize - 1) / csize;
  const int cbeg = min(S, crank * cwin * 32), cend = min(S, cbeg + cwin * 32);
  const int nit = (cwin + 31) / 32;  // windows per warp
  const int beg = min(cend, cbeg + warp * nit * 32), end = min(cend, beg + nit * 32);
  Slots<MAXIT> sl;
  sl.load(a.experts, beg, end, lane, nit);
  for (int i = tid; i <= E; i += kSchedThreads) s_off[i] = a.map.off[i];
  for (int i = tid; i < R; i += kSchedThreads) {
    s_hosts[i] = a.map.hosts[i];
    s_rid[i] = a.map.rid[i];
    s_qidx[i] = a.map.qidx[i];
  }
  for (int e = tid; e < E; e += kSchedThreads) {
    s_hm[e] = a.map.hmask[e];
    chg[e] = -1;
  }
  for (int i = tid; i < 32 * E; i += kSchedThreads) cnt[i] = 0;
  for (int g = tid; g < N; g += kSchedThreads) {
    load[g] = 0;
    routed[g] = 0;
  }
  for (int q = tid; q <= R; q += kSchedThreads) {
    qcnt[q] = 0;
    tcnt[q] = 0;
  }
  if (tid == 0) s_bad = INT_MAX;
  __syncthreads();
  if (trace && tid == 0) trace[1] = globaltimer();

  // ---- pass 1: warp-private histogram ---------------------------------------
  int32_t *mycnt = cnt + warp * E;
#pragma unroll
  for (int i = 0; i < (MAXIT > 0 ? MAXIT : nit); ++i) {
    if (i >= nit) break;
    const int s = beg + i * 32 + lane;
    const bool in = s < end;
    const int e = in ? sl.get(a.experts, i, s) : 0;
    const bool valid = in && e >= 0 && e < E;
    if (in && !valid) atomicMin(&s_bad, e);
    const unsigned vm = __ballot_sync(kFull, valid);
    const unsigned peers = peers_of(vm, e, a.id_bits);
    if (valid && lane == __ffs(peers) - 1) mycnt[e] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int e = tid; e < E; e += kSchedThreads) {
    int run = 0;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) {
      const int c = cnt[w * E + e];
      cnt[w * E + e] = run;
      run += c;
    }
    ltot[e] = run;
  }
  if (trace && tid == 0) trace[2] = globaltimer();

  // ---- the one cluster exchange: totals and bad ids via DSMEM ---------------
  int bad = INT_MAX;
  if (csize == 1) {  // no peers: local smem only
    __syncthreads();
    bad = s_bad;
    for (int e = tid; e < E; e += kSchedThreads) {
      xbase[e] = 0;
      tot[e] = ltot[e];
    }
  } else {
    cluster.sync();
    for (int c = 0; c < csize; ++c) bad = min(bad, *cluster.map_shared_rank(&s_bad, c));
    for (int e = tid; e < E; e += kSchedThreads) {
      int before = 0, all = 0;
      for (int c = 0; c < csize; ++c) {
        const int v = *cluster.map_shared_rank(ltot + e, c);
        before += c < crank ? v : 0;
        all += v;
      }
      xbase[e] = before;
      tot[e] = all;
    }
  }
  cluster_arrive();  // our reads of remote smem are done (wait before exit)
  if (bad != INT_MAX) {
    if (leader) write_error_layout(a, JANUS_EUNKNOWN_EXPERT, bad);
    cluster_wait();
    return;
  }
  __syncthreads();

  // ---- pins (aebs.cpp:180-185) ------------------------------------------------
  for (int e = tid; e < E; e += kSchedThreads) {
    const int r = s_off[e + 1] - s_off[e];
    // a validated map gives every expert a replica; the reference's second
    // check (:164-166) is kept for completeness
    if (tot[e] > 0 && r == 0) atomicMin(&s_bad, e);
    if (tot[e] > 0 && r == 1) {
      const int g = s_hosts[s_off[e]];
      chg[e] = g;
      atomicAdd(&load[g], 1);
    }
  }
  __syncthreads();
  if (s_bad != INT_MAX) {
    if (leader) write_error_layout(a, JANUS_EUNKNOWN_EXPERT, s_bad);
    cluster_wait();
    return;
  }
  if (trace && tid == 0) trace[3] = globaltimer();

  // ---- sequential phase, warp 0 --------------------------------------------
  if (warp == 0) {
    if (a.policy == JANUS_POLICY_AEBS) {
      if (N <= 32) {
        greedy_warp(E, N, tot, s_off, s_hm, load, chg);
      } else {
        for (int e = 0; e < E; ++e) {
          const int r = s_off[e + 1] - s_off[e];
          if (tot[e] == 0 || r <= 1) continue;
          uint32_t best = 0xffffffffu;
          for (int i = lane; i < r; i += 32)
            best = min(best, ((uint32_t)load[s_hosts[s_off[e] + i]] << 11) | (uint32_t)i);
          best = __reduce_min_sync(kFull, best);
          const int g = s_hosts[s_off[e] + (int)(best & 2047u)];
          if (lane == 0) {
            load[g] += 1;
            chg[e] = g;
          }
          __syncwarp();
        }
      }
    } else if (lane == 0) {  // schedule_random, aebs.cpp:250-262
      uint64_t st = a.rng_state;
      for (int e = 0; e < E; ++e) {
        const int r = s_off[e + 1] - s_off[e];
        if (tot[e] == 0 || r <= 1) continue;
        const int g = s_hosts[s_off[e] + (int)next_below(st, (uint64_t)r)];
        chg[e] = g;
        load[g] += 1;
      }
    }
  }
  __syncthreads();
  if (trace && tid == 0) trace[4] = globaltimer();

  // ---- finish_assignment per expert (aebs.cpp:94-108) ---------------------
  for (int e = tid; e < E; e += kSchedThreads) {
    const int g = chg[e];
    if (g >= 0) {
      int p = s_off[e];
      if (N <= 32) {
        p += __popc(s_hm[e] & ((1u << g) - 1u));
      } else {
        while (s_hosts[p] != g) ++p;
      }
      ridof[e] = s_rid[p];
      const int q = s_qidx[p];
      qof[e] = q;
      qcnt[q] = tot[e];
      // tiles of tile_n rows; the last one also takes the remainder (gemm.cu)
      tcnt[q] = a.merge_tail ? (tot[e] > 0 ? max(1, tot[e] / a.tile_n) : 0)
                             : (tot[e] + a.tile_n - 1) / a.tile_n;
      atomicAdd(&routed[g], (unsigned)tot[e]);
    }
    if (leader) {
      a.out.expert_instance[e] = g;
      if (a.out.expert_tokens) a.out.expert_tokens[e] = tot[e];
    }
  }
  __syncthreads();
  block_exscan2(qcnt, tcnt, R + 1, s_scan);
  if (leader) {
    if (a.out.group_off)
      for (int q = tid; q <= R; q += kSchedThreads) a.out.group_off[q] = qcnt[q];
    if (a.tile_off)
      for (int q = tid; q <= R; q += kSchedThreads) a.tile_off[q] = tcnt[q];
    if (a.shared_off && tid == 0) {  // one group of this instance's shared tokens
      const int rows = a.shared_rows;
      a.shared_off[0] = 0;
      a.shared_off[1] = rows;
      a.shared_off[2] = 0;
      a.shared_off[3] = rows > 0 ? (rows + a.shared_tile_n - 1) / a.shared_tile_n : 0;
    }
    for (int g = tid; g < N; g += kSchedThreads) {
      a.out.load[g] = load[g];
      a.out.routed_tokens[g] = (int64_t)routed[g];
    }
  }
  if (trace && tid == 0) trace[5] = globaltimer();

  // ---- pass 2: remap slots and lay out rows --------------------------------
  {
    int32_t *__restrict__ o_inst = a.out.instance;
    int32_t *__restrict__ o_repl = a.out.replica;
    int32_t *__restrict__ o_srow = a.out.slot_row;
    int32_t *__restrict__ o_rslot = a.out.row_slot;
#pragma unroll
    for (int i = 0; i < (MAXIT > 0 ? MAXIT : nit); ++i) {
      if (i >= nit) break;
      const int s = beg + i * 32 + lane;
      const bool in = s < end;
      const int e = in ? sl.get(a.experts, i, s) : 0;
      const unsigned vm = __ballot_sync(kFull, in);
      const unsigned peers = peers_of(vm, e, a.id_bits);
      if (in) {
        const int rank = __popc(peers & lanemask_lt());
        const int cbase = mycnt[e];
        const int row = qcnt[qof[e]] + xbase[e] + cbase + rank;
        __syncwarp(vm);
        if (lane == __ffs(peers) - 1) mycnt[e] = cbase + __popc(peers);
        o_inst[s] = chg[e];
        o_repl[s] = ridof[e];
        if (o_srow) o_srow[s] = row;
        if (o_rslot) o_rslot[row] = s;
      }
      __syncwarp();
    }
  }
  if (leader && tid == 0) {
    a.out.status[0] = JANUS_OK;
    a.out.status[1] = 0;
  }
  if (trace) {
    __syncthreads();
    if (tid == 0) trace[6] = globaltimer();
  }
  cluster_wait();
}

template <int MAXIT>
cudaError_t launch_variant(const SchedArgs &a, size_t smem, int csize, cudaStream_t stream) {
  // The opt-in smem limit is per device and per function; raise it when a
  // larger map needs more (227 KB minus the static shared memory at most).
  static int configured_dev = -1;
  static size_t configured_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev || smem > configured_smem) {
    const size_t want = smem > 48 * 1024 ? smem : 48 * 1024;
    cudaError_t err = cudaFuncSetAttribute(aebs_schedule_kernel<MAXIT>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(aebs_schedule_kernel<MAXIT>,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
    configured_dev = dev;
    configured_smem = want;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(kSchedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, aebs_schedule_kernel<MAXIT>, a);
}

}  // namespace

size_t schedule_smem_bytes(int E, int N, int R) {
  return (size_t)N * 4 + (size_t)32 * E * 4 + (size_t)6 * E * 4 + (size_t)N * 4 +
         (size_t)2 * (R + 1) * 4 + (size_t)(E + 1) * 4 + (size_t)3 * R * 4 + (size_t)E * 4;
}

int schedule_cluster_size(int S) {
  // ~1024 slots per CTA, and at least 4 CTAs once there are 512 per CTA; the
  // per-phase cost is mostly barrier latency, so small steps gain from more
  // CTAs only up to a point (graph-replayed µs, tools/sched_sweep.py, c2 map:
  // 2048 slots 9.3 / 8.4 / 8.0 / 8.1 µs on 1 / 2 / 4 / 8 CTAs; 6144 slots
  // 9.8 / 8.9 / 9.4 / 9.9 on 3 / 6 / 12 / 16).  Above 16 K slots (the box
  // path's MoE GPUs scheduling every attention shard) the cluster is 16.
  const int c = std::max((S + 1023) / 1024, std::min(4, (S + 511) / 512));
  return c < 1 ? 1 : (c > kMaxCluster ? kMaxCluster : c);
}

cudaError_t launch_schedule(const SchedArgs &a, cudaStream_t stream) {
  const size_t smem = schedule_smem_bytes(a.map.E, a.map.N, a.map.R);
  const int csize = schedule_cluster_size(a.S);
  const int windows = (a.S + 31) / 32;
  const int nit = ((windows + csize - 1) / csize + 31) / 32;
  if (nit <= 1) return launch_variant<1>(a, smem, csize, stream);
  if (nit <= 2) return launch_variant<2>(a, smem, csize, stream);
  if (nit <= 4) return launch_variant<4>(a, smem, csize, stream);
  if (nit <= 8) return launch_variant<8>(a, smem, csize, stream);
  if (nit <= 16) return launch_variant<16>(a, smem, csize, stream);
  return launch_variant<0>(a, smem, csize, stream);
}

}  // namespace janus
