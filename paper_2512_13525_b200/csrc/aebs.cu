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
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

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

// Exclusive scan of two int arrays of n entries in place (NT threads).
template <int NT = kSchedThreads>
__device__ void block_exscan2(int32_t *a, int32_t *b, int n, int32_t *scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + NT - 1) / NT;
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
    int wa = lane < NT / 32 ? scratch[lane] : 0, wb = lane < NT / 32 ? scratch[32 + lane] : 0;
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
  for (int q = threadIdx.x; q <= R; q += blockDim.x) {
    if (a.out.group_off) a.out.group_off[q] = 0;
    if (a.tile_off) a.tile_off[q] = 0;
  }
  if (a.shared_off && threadIdx.x < 4) a.shared_off[threadIdx.x] = 0;
  for (int s = threadIdx.x; s < a.S; s += blockDim.x) a.out.instance[s] = -1;
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
  // the one-lane pairs greedy's records and list (N <= 8, DevMap::pair_info)
  const bool pairs = a.map.pair_info != nullptr;
  const int E4 = (E + 3) & ~3;
  uint4 *s_pinfo = reinterpret_cast<uint4 *>(
      (reinterpret_cast<uintptr_t>(s_hm + E) + 15) & ~uintptr_t(15));  // [E]
  uint4 *s_plist = s_pinfo + E;                                       // [E+4]
  uint32_t *s_pbhi = reinterpret_cast<uint32_t *>(s_plist + E + 4);   // [E4]
  uint32_t *s_pbh_list = s_pbhi + E4;                                 // [E4+4]
  int32_t *s_elist = reinterpret_cast<int32_t *>(s_pbh_list + E4 + 4);  // [E4]
  int32_t *s_res = s_elist + E4;                                      // [E4+4]
  __shared__ int32_t s_bad;
  __shared__ int32_t s_scan[64];

  // ---- slot ranges: CTA, then warp; issue every slot load at once ----------
  const int windows = (S + 31) / 32;
  const int cwin = (windows + csize - 1) / csize;
  const int cbeg = min(S, crank * cwin * 32), cend = min(S, cbeg + cwin * 32);
  const int nit = (cwin + 31) / 32;  // windows per warp
  const int beg = min(cend, cbeg + warp * nit * 32), end = min(cend, beg + nit * 32);
  Slots<MAXIT> sl;
  {
    // the first element per thread of every map table: all loads go out
    // before any smem store (in order, a load -> store pair per table would
    // cost one L2 round trip each)
    int r_off = 0, r_h = 0, r_r = 0, r_q = 0;
    uint32_t r_hm = 0, r_pb = 0;
    uint4 r_pi = make_uint4(0, 0, 0, 0);
    if (tid <= E) r_off = __ldg(a.map.off + tid);
    if (tid < R) {
      r_h = __ldg(a.map.hosts + tid);
      r_r = __ldg(a.map.rid + tid);
      r_q = __ldg(a.map.qidx + tid);
    }
    if (tid < E) {
      r_hm = __ldg(a.map.hmask + tid);
      if (pairs) {
        r_pi = __ldg(a.map.pair_info + tid);
        r_pb = __ldg(a.map.pair_bhi + tid);
      }
    }
    for (int i = tid; i < 32 * E; i += kSchedThreads) cnt[i] = 0;
    if (tid <= E) s_off[tid] = r_off;
    if (tid < R) {
      s_hosts[tid] = r_h;
      s_rid[tid] = r_r;
      s_qidx[tid] = r_q;
    }
    if (tid < E) {
      s_hm[tid] = r_hm;
      chg[tid] = -1;
      if (pairs) {
        s_pinfo[tid] = r_pi;
        s_pbhi[tid] = r_pb;
      }
    }
  }
  for (int i = tid + kSchedThreads; i <= E; i += kSchedThreads) s_off[i] = a.map.off[i];
  for (int i = tid + kSchedThreads; i < R; i += kSchedThreads) {
    s_hosts[i] = a.map.hosts[i];
    s_rid[i] = a.map.rid[i];
    s_qidx[i] = a.map.qidx[i];
  }
  for (int e = tid + kSchedThreads; e < E; e += kSchedThreads) {
    s_hm[e] = a.map.hmask[e];
    chg[e] = -1;
    if (pairs) {
      s_pinfo[e] = __ldg(a.map.pair_info + e);
      s_pbhi[e] = __ldg(a.map.pair_bhi + e);
    }
  }
  // the map is constant across steps: staged above before the dependency wait
  // (overlaps the previous kernel under programmatic dependent launch); the
  // routing, the abort word and every output belong to the predecessors
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the box exchange aborted this step (a peer never published its rows)
  if (a.abort_flag && *a.abort_flag) {
    if (leader) write_error_layout(a, JANUS_EPEER, 0);
    return;  // before any cluster barrier: every CTA reads the same flag
  }
  sl.load(a.experts, beg, end, lane, nit);
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
  for (int e0 = warp * 32; e0 < E; e0 += kSchedThreads) {  // warp-uniform trip count
    const int e = e0 + lane;
    const int r = e < E ? s_off[e + 1] - s_off[e] : 0;
    const bool act = e < E && tot[e] > 0;
    // a validated map gives every expert a replica; the reference's second
    // check (:164-166) is kept for completeness
    if (act && r == 0) atomicMin(&s_bad, e);
    const bool pin = act && r == 1;
    const int g = pin ? s_hosts[s_off[e]] : -1;
    if (pin) chg[e] = g;
    if (N <= 32) {  // count the pins per instance with one vote per instance, not per expert
      const unsigned pm = __ballot_sync(kFull, pin);
      if (pm) {
        const unsigned my = __match_any_sync(kFull, g);
        if (pin && lane == __ffs(my & pm) - 1) atomicAdd(&load[g], __popc(my & pm));
      }
    } else if (pin) {
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
      if (pairs) {
        greedy_pairs(
            lane, (E + 31) / 32, N, a.map.pairs_only != 0,
            [&](int w) {
              const int e = w * 32 + lane;
              return __ballot_sync(kFull, e < E && tot[e] > 0 && s_off[e + 1] - s_off[e] > 1);
            },
            [&](int e) { return s_hm[e]; }, load, s_pinfo, s_pbhi, s_plist, s_pbh_list, s_elist,
            s_res, chg, load);
      } else if (N <= 32) {
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

// ---------------------------------------------------------------------------
// The decode-size scheduler: S <= kSmallMaxSlots slots, N <= 32 instances,
// R <= kSmallMaxReplicas — one CTA of 16 warps, no cluster, no DSMEM, the map
// read as compact tables (DevMap::ex_info / rep_info / multi_mask / pin_mask,
// ~8 B per expert and replica) in the same round trip as the batch.  The
// order-dependent greedy (aebs.cpp:186-194) starts right after the histogram
// pass: it needs only the activated set (a bitmask built in pass 1) and the
// single-replica pins per instance (popc of activated & pin_mask[g]), so warp
// 0 runs it while the other 15 warps scan the per-warp counts (token totals
// and each warp's starting rank per expert).  Same outputs, bit for bit, as
// aebs_schedule_kernel.
constexpr int kSmallThreads = 512, kSmallWarps = kSmallThreads / 32, kSmallMaxIt = 4;
constexpr int kSmallMaxSlots = kSmallWarps * kSmallMaxIt * 32;  // 2048
constexpr int kSmallMaxReplicas = 2048;

__host__ __device__ inline size_t small_absent_off(int E, int N, int R) {
  const int W = (E + 31) / 32;
  const size_t b = (size_t)16 * E + (size_t)8 * R + (size_t)4 * kSmallWarps * E + (size_t)16 * E +
                   (size_t)8 * (R + 1) + (size_t)4 * (2 * W + 2 * N * W) + (size_t)4 * (N + 1);
  return (b + 15) & ~(size_t)15;
}

// finish_assignment (aebs.cpp:94-108) for one expert placed on instance g.
__device__ __forceinline__ void finish_multi(const SchedArgs &a, int e, int g, int4 x,
                                             const int2 *rep, const int32_t *tot, int32_t *chg,
                                             int32_t *ridof, int32_t *qof, int32_t *qcnt,
                                             int32_t *tcnt) {
  const int t = tot[e];
  const int p = x.x + __popc((uint32_t)x.z & ((1u << g) - 1u));
  const int2 rq = rep[p];
  chg[e] = g;
  ridof[e] = rq.x;
  qof[e] = rq.y;
  qcnt[rq.y] = t;
  tcnt[rq.y] = a.merge_tail ? max(1, t / a.tile_n) : (t + a.tile_n - 1) / a.tile_n;
  a.out.expert_instance[e] = g;
  if (a.out.expert_tokens) a.out.expert_tokens[e] = t;
}

// The one-lane greedy for N <= 8 instances with loads < 256 (DevMap::pair_info),
// run by one warp.  The loads live as bytes of two registers (lo: instances
// 0-3, hi: 4-7).  The activated multi-replica experts are first listed in
// ascending order with their precomputed records (warp-cooperative, one
// 32-expert word per round), padded with no-op records to a multiple of 4.
// One lane then walks the list four records per load round.  For a two-replica
// expert (hosts a < b) two PRMTs build words equal but for their top byte,
// load[a] resp. load[b], so one unsigned <= picks a on ties
// (aebs.cpp:186-194: least-loaded host, ties to the lowest id); the winner's
// byte gets + 1: a 4-deep dependent chain per expert.  Three or more
// replicas: a scan of the host bytes (strict <, ascending ids).
// act_multi(w): word w of the activated multi-replica experts; hmask_of(e):
// host bitmask; init_load: the pins' loads; results in chg[] and load_out[].
template <class ActMulti, class HostMask>
__device__ void greedy_pairs(int lane, int W, int N, bool pairs_only, ActMulti act_multi,
                             HostMask hmask_of, const int32_t *init_load, const uint4 *pinfo,
                             const uint32_t *pinfo_bhi, uint4 *plist, uint32_t *pb_hi,
                             int32_t *elist, int32_t *res, int32_t *chg, int32_t *load_out) {
  int total = 0;
  for (int w = 0; w < W; ++w) {
    const unsigned m = act_multi(w);
    if ((m >> lane) & 1u) {
      const int pos = total + __popc(m & lanemask_lt());
      const int e = w * 32 + lane;
      const uint4 r = pinfo[e];
      plist[pos] = make_uint4(r.x, r.y, r.z, r.w);
      pb_hi[pos] = pinfo_bhi[e];  // read back as uint4 per group of 4
      elist[pos] = e;
    }
    total += __popc(m);
  }
  const int padded = (total + 3) & ~3;
  if (total + lane < padded) {  // no-op records: nothing moves
    plist[total + lane] = make_uint4(0, 0, 0, 0);
    pb_hi[total + lane] = 0;
  }
  uint32_t lo = 0, hi = 0;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const uint32_t v = (uint32_t)(g < N ? init_load[g] : 0) & 0xffu;
    if (g < 4)
      lo |= v << (8 * g);
    else
      hi |= v << (8 * (g - 4));
  }
  __syncwarp();
  if (lane == 0) {
    if (pairs_only) {
      // every multi-replica expert has exactly two hosts: no branch per step
      for (int i = 0; i < padded; i += 4) {
        uint4 r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r[u] = plist[i + u];
        const uint4 bh = *reinterpret_cast<const uint4 *>(pb_hi + i);  // one vector load
        const uint32_t bhs[4] = {bh.x, bh.y, bh.z, bh.w};
        int4 out;
        int *o = reinterpret_cast<int *>(&out);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t da, db;
          asm("prmt.b32 %0, %1, %2, %3;" : "=r"(da) : "r"(lo), "r"(hi), "r"(r[u].x));
          asm("prmt.b32 %0, %1, %2, %3;" : "=r"(db) : "r"(lo), "r"(hi), "r"(r[u].x >> 16));
          // both successors formed beside the PRMTs: the chain per expert is
          // PRMT -> compare -> select (unconditional uses: no sunk loads)
          uint32_t la, lb, ha, hb;  // (asm: kept apart from the select, not re-associated)
          asm("add.u32 %0, %1, %2;" : "=r"(la) : "r"(lo), "r"(r[u].y));
          asm("add.u32 %0, %1, %2;" : "=r"(lb) : "r"(lo), "r"(r[u].w));
          asm("add.u32 %0, %1, %2;" : "=r"(ha) : "r"(hi), "r"(r[u].z));
          asm("add.u32 %0, %1, %2;" : "=r"(hb) : "r"(hi), "r"(bhs[u]));
          const bool ka = da <= db;
          lo = ka ? la : lb;
          hi = ka ? ha : hb;
          o[u] = (int)ka;
        }
        *reinterpret_cast<int4 *>(res + i) = out;
      }
    } else {
      for (int i = 0; i < padded; ++i) {
        const uint4 r = plist[i];
        int ca;
        if (r.x != 0xffffffffu) {
          uint32_t da, db;
          asm("prmt.b32 %0, %1, %2, %3;" : "=r"(da) : "r"(lo), "r"(hi), "r"(r.x));
          asm("prmt.b32 %0, %1, %2, %3;" : "=r"(db) : "r"(lo), "r"(hi), "r"(r.x >> 16));
          ca = da <= db;
          lo += ca ? r.y : r.w;
          hi += ca ? r.z : pb_hi[i];
        } else {  // >= 3 replicas: r.y = host bitmask; ca = the winner
          uint32_t best = 0xffffffffu;
          ca = 0;
          for (uint32_t hm = r.y; hm; hm &= hm - 1) {
            const int h = __ffs(hm) - 1;
            uint32_t l;
            asm("prmt.b32 %0, %1, %2, %3;" : "=r"(l) : "r"(lo), "r"(hi), "r"(h));
            l &= 0xffu;
            if (l < best) {
              best = l;
              ca = h;
            }
          }
          const uint32_t inc = 1u << (8 * (ca & 3));
          lo += ca < 4 ? inc : 0u;
          hi += ca < 4 ? 0u : inc;
        }
        res[i] = ca;
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g)
      if (g < N) {
        uint32_t l;
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(l) : "r"(lo), "r"(hi), "r"(g));
        load_out[g] = (int)(l & 0xffu);
      }
  }
  __syncwarp();
  for (int i = lane; i < total; i += 32) {  // results -> finish, in parallel
    const int e = elist[i];
    const uint32_t hm = hmask_of(e);
    const int rr = res[i];
    // two replicas: rr = 1 -> the lower host (a), 0 -> b; else rr = the host
    chg[e] = __popc(hm) == 2 ? (rr ? __ffs(hm) - 1 : 31 - __clz(hm)) : rr;
  }
}

// Peers with a compile-time id width (fully unrolled; NB == 0: runtime width).
template <int NB>
__device__ __forceinline__ unsigned peers_nb(unsigned valid, int id, int nbits) {
  if (NB == 0) return peers_of(valid, id, nbits);
  unsigned peers = valid;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const bool bit = (id >> b) & 1;
    const unsigned m = __ballot_sync(kFull, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

template <int NB>
__global__ void __launch_bounds__(kSmallThreads, 1) aebs_small_kernel(SchedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int E = a.map.E, N = a.map.N, R = a.map.R, S = a.S, W = (E + 31) / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long c0 = 0;
  if (a.trace && tid == 0) {
    a.trace[0] = globaltimer();
    c0 = clock64();
  }
  int4 *exi = reinterpret_cast<int4 *>(smem);                   // [E]
  int2 *rep = reinterpret_cast<int2 *>(exi + E);                // [R]
  int32_t *cnt = reinterpret_cast<int32_t *>(rep + R);          // [16][E]
  int32_t *tot = cnt + kSmallWarps * E;                         // [E]
  int32_t *chg = tot + E;                                       // [E]
  int32_t *qof = chg + E;                                       // [E]
  int32_t *ridof = qof + E;                                     // [E]
  int32_t *qcnt = ridof + E;                                    // [R+1]
  int32_t *tcnt = qcnt + R + 1;                                 // [R+1]
  uint32_t *act = reinterpret_cast<uint32_t *>(tcnt + R + 1);   // [W]
  uint32_t *multi = act + W;                                    // [W]
  uint32_t *pin = multi + W;                                    // [N][W]
  uint32_t *hmk = pin + N * W;                                  // [N][W]
  int32_t *qb = reinterpret_cast<int32_t *>(hmk + N * W);       // [N+1]
  // pair-record list of the one-lane greedy: [E+1] records, [E] expert ids, and
  // the per-expert records staged from DevMap::pair_info
  uint4 *pinfo = reinterpret_cast<uint4 *>(smem + small_absent_off(E, N, R));  // [E]
  uint4 *plist = pinfo + E;                                     // [E+4]
  uint32_t *pinfo_bhi = reinterpret_cast<uint32_t *>(plist + E + 4);  // [E]
  uint32_t *pb_hi = pinfo_bhi + ((E + 3) & ~3);                 // [E+4], 16-B aligned
  int32_t *elist = reinterpret_cast<int32_t *>(pb_hi + ((E + 3) & ~3) + 4);  // [E]
  int32_t *res = elist + ((E + 3) & ~3);                        // [E+4], 16-B aligned
  unsigned char *seen = reinterpret_cast<unsigned char *>(res + E + 4);  // [E]
  __shared__ int32_t s_load[32];
  __shared__ int32_t s_bad;

  // ---- the compact map tables (constant across steps: staged before the
  // dependency wait, so under programmatic dependent launch this overlaps the
  // previous kernel), then this warp's slots ---------------------------------
  const int per = ((S + kSmallWarps - 1) / kSmallWarps + 31) / 32 * 32;
  const int beg = min(S, warp * per), end = min(S, beg + per);
  const int nit = (end - beg + 31) / 32;
  // Every global load of the first element per thread goes out before any
  // smem store: an in-order warp would otherwise stall on each load -> store
  // pair in turn (one L2 round trip per table instead of one in all).
  const bool pairs = a.map.pair_info != nullptr;
  int4 r_exi = make_int4(0, 0, 0, 0);
  int2 r_rep = make_int2(0, 0);
  uint4 r_pi = make_uint4(0, 0, 0, 0);
  uint32_t r_pbh = 0, r_multi = 0, r_pin = 0, r_hmk = 0;
  int r_qb = 0;
  if (tid < E) r_exi = __ldg(a.map.ex_info + tid);
  if (tid < R) r_rep = __ldg(a.map.rep_info + tid);
  if (pairs && tid < E) {
    r_pi = __ldg(a.map.pair_info + tid);
    r_pbh = __ldg(a.map.pair_bhi + tid);
  }
  if (tid < W) r_multi = __ldg(a.map.multi_mask + tid);
  if (tid < N * W) {
    r_pin = __ldg(a.map.pin_mask + tid);
    r_hmk = __ldg(a.map.host_mask + tid);
  }
  if (tid <= N) r_qb = __ldg(a.map.qbase + tid);
  // zeroing meanwhile
  for (int i = tid; i < kSmallWarps * E; i += kSmallThreads) cnt[i] = 0;
  for (int e = tid; e < E; e += kSmallThreads) seen[e] = 0;
  for (int q = tid; q <= R; q += kSmallThreads) {
    qcnt[q] = 0;
    tcnt[q] = 0;
  }
  if (tid < E) exi[tid] = r_exi;
  if (tid < R) rep[tid] = r_rep;
  if (pairs && tid < E) {
    pinfo[tid] = r_pi;
    pinfo_bhi[tid] = r_pbh;
  }
  if (tid < W) multi[tid] = r_multi;
  if (tid < N * W) {
    pin[tid] = r_pin;
    hmk[tid] = r_hmk;
  }
  if (tid <= N) qb[tid] = r_qb;
  // tables longer than one element per thread (E or R above 512, N*W above 512)
  for (int e = tid + kSmallThreads; e < E; e += kSmallThreads) {
    exi[e] = __ldg(a.map.ex_info + e);
    if (pairs) {
      pinfo[e] = __ldg(a.map.pair_info + e);
      pinfo_bhi[e] = __ldg(a.map.pair_bhi + e);
    }
  }
  for (int p = tid + kSmallThreads; p < R; p += kSmallThreads) rep[p] = __ldg(a.map.rep_info + p);
  for (int i = tid + kSmallThreads; i < N * W; i += kSmallThreads) {
    pin[i] = __ldg(a.map.pin_mask + i);
    hmk[i] = __ldg(a.map.host_mask + i);
  }
  // the step's inputs (routing, the exchange's abort word) and every output
  // buffer belong to the predecessor kernels until they complete
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.abort_flag && *a.abort_flag) {  // the box exchange aborted this step
    write_error_layout(a, JANUS_EPEER, 0);
    return;
  }
  int v[kSmallMaxIt];
#pragma unroll
  for (int i = 0; i < kSmallMaxIt; ++i) {
    const int sl = beg + i * 32 + lane;
    v[i] = (i < nit && sl < end) ? __ldg(a.experts + sl) : 0;
  }
  if (tid < 32) s_load[tid] = 0;
  if (tid == 0) s_bad = INT_MAX;
  __syncthreads();
  if (a.trace && tid == 0) a.trace[1] = globaltimer();

  // ---- pass 1: warp histogram + the activated set --------------------------
  __shared__ int32_t s_scan[64];
  int32_t *mycnt = cnt + warp * E;
#pragma unroll
  for (int i = 0; i < kSmallMaxIt; ++i) {
    if (i >= nit) break;
    const int sl = beg + i * 32 + lane;
    const bool in = sl < end;
    const int e = in ? v[i] : 0;
    const bool valid = in && e >= 0 && e < E;
    if (in && !valid) atomicMin(&s_bad, e);
    const unsigned vm = __ballot_sync(kFull, valid);
    const unsigned peers = peers_nb<NB>(vm, e, a.id_bits);
    if (valid && lane == __ffs(peers) - 1) {
      seen[e] = 1;  // plain byte stores: warp 0 ballots them into the activated set
      mycnt[e] += __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  if (s_bad != INT_MAX) {
    write_error_layout(a, JANUS_EUNKNOWN_EXPERT, s_bad);
    return;
  }
  if (a.trace && tid == 0) a.trace[2] = globaltimer();

  if (warp == 0) {
    // ---- the activated set, pins, the sequential greedy (aebs.cpp:180-194) --
    for (int w = 0; w < W; ++w) {
      const unsigned b = __ballot_sync(kFull, w * 32 + lane < E && seen[w * 32 + lane]);
      if (lane == 0) act[w] = b;
    }
    __syncwarp();
    int pins = 0;
    if (lane < N)
      for (int w = 0; w < W; ++w) pins += __popc(act[w] & pin[lane * W + w]);
    if (a.policy == JANUS_POLICY_AEBS && pairs) {
      if (lane < N) s_load[lane] = pins;
      __syncwarp();
      greedy_pairs(
          lane, W, N, a.map.pairs_only != 0, [&](int w) { return act[w] & multi[w]; },
          [&](int e) { return (uint32_t)exi[e].z; }, s_load, pinfo, pinfo_bhi, plist, pb_hi,
          elist, res, chg, s_load);
    } else if (a.policy == JANUS_POLICY_AEBS) {
      // 9..32 instances: lane g keeps key_g = load << 5 | g; the candidate
      // test reads lane g's own bitmask of the multi-replica experts it hosts
      uint32_t key = lane < N ? ((uint32_t)pins << 5) | (uint32_t)lane : 0xffffffffu;
      for (int w = 0; w < W; ++w) {
        unsigned mm = act[w] & multi[w];
        const uint32_t mine = lane < N ? hmk[lane * W + w] : 0u;
        while (mm) {
          const int b = __ffs(mm) - 1;
          mm &= mm - 1;
          const uint32_t drop = ((mine >> b) & 1u) ? 0u : 0xffffffffu;
          const uint32_t win = __reduce_min_sync(kFull, key | drop);
          key += (key == win) ? 32u : 0u;
          if (lane == 0) chg[w * 32 + b] = (int)(win & 31u);
        }
      }
      if (lane < N) s_load[lane] = (int)(key >> 5);
    } else {  // schedule_random, aebs.cpp:250-262: ascending e, one lane
      if (lane < N) s_load[lane] = pins;
      __syncwarp();
      if (lane == 0) {
        uint64_t st = a.rng_state;
        for (int w = 0; w < W; ++w)
          for (unsigned mm = act[w] & multi[w]; mm; mm &= mm - 1) {
            const int e = w * 32 + __ffs(mm) - 1;
            const int4 x = exi[e];
            const int pick = (int)next_below(st, (uint64_t)x.y);
            // the pick-th set bit of the host mask
            uint32_t hm = (uint32_t)x.z;
            for (int i = 0; i < pick; ++i) hm &= hm - 1;
            const int g = __ffs(hm) - 1;
            chg[e] = g;
            s_load[g] += 1;
          }
      }
    }
  } else {
    // ---- meanwhile: per-expert totals and each warp's starting rank ---------
    for (int e = tid - 32; e < E; e += kSmallThreads - 32) {
      int run = 0;
#pragma unroll
      for (int w = 0; w < kSmallWarps; ++w) {
        const int c = cnt[w * E + e];
        cnt[w * E + e] = run;
        run += c;
      }
      tot[e] = run;
      const int4 x = exi[e];
      // finish_assignment (aebs.cpp:94-108) for every expert whose instance is
      // known now: inactive, or pinned (one replica); warp 0 finishes the
      // multi-replica ones after its greedy
      if (run == 0) {
        chg[e] = -1;
      } else if (x.y == 1) {
        chg[e] = x.w;
        const int2 rq = rep[x.x];
        ridof[e] = rq.x;
        qof[e] = rq.y;
        qcnt[rq.y] = run;
        tcnt[rq.y] = a.merge_tail ? max(1, run / a.tile_n) : (run + a.tile_n - 1) / a.tile_n;
      }
      if (run == 0 || x.y == 1) {
        a.out.expert_instance[e] = run == 0 ? -1 : x.w;
        if (a.out.expert_tokens) a.out.expert_tokens[e] = run;
      }
    }
  }
  __syncthreads();
  if (a.trace && tid == 0) a.trace[4] = globaltimer();

  // ---- finish the multi-replica experts the greedy placed (the others were
  // finished during the greedy), then the group offsets ----------------------
  for (int e = tid; e < E; e += kSmallThreads)
    if (((act[e >> 5] & multi[e >> 5]) >> (e & 31)) & 1u)
      finish_multi(a, e, chg[e], exi[e], rep, tot, chg, ridof, qof, qcnt, tcnt);
  __syncthreads();
  block_exscan2<kSmallThreads>(qcnt, tcnt, R + 1, s_scan);
  if (a.out.group_off)
    for (int q = tid; q <= R; q += kSmallThreads) a.out.group_off[q] = qcnt[q];
  if (a.tile_off)
    for (int q = tid; q <= R; q += kSmallThreads) a.tile_off[q] = tcnt[q];
  if (a.shared_off && tid == 0) {
    const int rows = a.shared_rows;
    a.shared_off[0] = 0;
    a.shared_off[1] = rows;
    a.shared_off[2] = 0;
    a.shared_off[3] = rows > 0 ? (rows + a.shared_tile_n - 1) / a.shared_tile_n : 0;
  }
  if (tid < N) {  // an instance's groups are contiguous in replica order
    a.out.load[tid] = s_load[tid];
    a.out.routed_tokens[tid] = (int64_t)(qcnt[qb[tid + 1]] - qcnt[qb[tid]]);
  }
  if (a.trace && tid == 0) a.trace[5] = globaltimer();

  // ---- pass 2: remap slots and lay out rows --------------------------------
#pragma unroll
  for (int i = 0; i < kSmallMaxIt; ++i) {
    if (i >= nit) break;
    const int sl = beg + i * 32 + lane;
    const bool in = sl < end;
    const int e = in ? v[i] : 0;
    const unsigned vm = __ballot_sync(kFull, in);
    const unsigned peers = peers_nb<NB>(vm, e, a.id_bits);
    if (in) {
      const int rank = __popc(peers & lanemask_lt());
      const int cbase = mycnt[e];
      const int row = qcnt[qof[e]] + cbase + rank;
      __syncwarp(vm);
      if (lane == __ffs(peers) - 1) mycnt[e] = cbase + __popc(peers);
      a.out.instance[sl] = chg[e];
      a.out.replica[sl] = ridof[e];
      if (a.out.slot_row) a.out.slot_row[sl] = row;
      if (a.out.row_slot) a.out.row_slot[row] = sl;
    }
    __syncwarp();
  }
  if (tid == 0) {
    a.out.status[0] = JANUS_OK;
    a.out.status[1] = 0;
  }
  if (a.trace) {
    __syncthreads();
    if (tid == 0) {
      a.trace[3] = a.trace[2];  // no separate pin phase
      a.trace[6] = globaltimer();
      a.trace[7] = (uint64_t)(clock64() - c0);  // SM cycles over the kernel (clock rate)
    }
  }
}

size_t small_smem_bytes(int E, int N, int R) {
  return small_absent_off(E, N, R) + (size_t)16 * (2 * E + 4) + (size_t)4 * (4 * E + 24) +
         (size_t)E;
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
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = sm100::pdl_enabled && !a.trace ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, aebs_schedule_kernel<MAXIT>, a);
}

__global__ void abort_gate_kernel(SchedArgs a) {
  if (*a.abort_flag) write_error_layout(a, JANUS_EPEER, 0);
}

}  // namespace

cudaError_t launch_abort_gate(const SchedArgs &a, cudaStream_t stream) {
  abort_gate_kernel<<<1, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

size_t schedule_smem_bytes(int E, int N, int R) {
  const size_t base = (size_t)N * 4 + (size_t)32 * E * 4 + (size_t)6 * E * 4 + (size_t)N * 4 +
                      (size_t)2 * (R + 1) * 4 + (size_t)(E + 1) * 4 + (size_t)3 * R * 4 +
                      (size_t)E * 4;
  if (N > 8) return base;
  const size_t E4 = (E + 3) & ~3;  // + the pairs greedy's records and list
  return base + 16 + (size_t)16 * (2 * E + 4) + (size_t)4 * (4 * E4 + 8);
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
  // JANUS_SCHED_CLUSTER=1 forces the cluster kernel at every size (A/B runs)
  static const bool force_cluster = std::getenv("JANUS_SCHED_CLUSTER") != nullptr;
  if (a.S <= kSmallMaxSlots && a.map.N <= 32 && a.map.R <= kSmallMaxReplicas && a.map.host_mask &&
      !force_cluster) {
    const size_t smem = small_smem_bytes(a.map.E, a.map.N, a.map.R);
    if (smem <= 200 * 1024) {
      static int configured_dev = -1;
      static size_t configured_smem = 0;
      int dev = 0;
      cudaGetDevice(&dev);
      if (configured_dev != dev || smem > configured_smem) {
        const size_t want = smem > 48 * 1024 ? smem : 48 * 1024;
        for (auto k : {aebs_small_kernel<0>, aebs_small_kernel<6>, aebs_small_kernel<7>,
                       aebs_small_kernel<8>}) {
          cudaError_t err =
              cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
          if (err != cudaSuccess) return err;
        }
        configured_dev = dev;
        configured_smem = want;
      }
      // the id width the BASELINE configs use (E = 64 / 128 / 256) unrolled
      auto k = a.id_bits == 6   ? aebs_small_kernel<6>
               : a.id_bits == 7 ? aebs_small_kernel<7>
               : a.id_bits == 8 ? aebs_small_kernel<8>
                                : aebs_small_kernel<0>;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(1);
      cfg.blockDim = dim3(kSmallThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = sm100::pdl_enabled && !a.trace ? 1 : 0;
      return cudaLaunchKernelEx(&cfg, k, a);
    }
  }
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
