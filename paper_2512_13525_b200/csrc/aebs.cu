// aebs.cu — K1+K2: the activation-balanced expert scheduler and the dispatch
// layout as ONE single-CTA sm_100a kernel.
//
// Replaces moesim::schedule (src/aebs.cpp:172-197: collect_activated :126-168,
// greedy :178-194, finish_assignment :89-122) and schedule_random (:250-262),
// bit-exact with schedule_reference (:199-248).
//
// One CTA of 32 warps.  The batch is cut into 32 contiguous slot ranges, one per
// warp, so every per-expert count is warp-private (no atomics):
//   pass 1  warp-aggregated histogram: __match_any_sync groups equal expert ids
//           in a 32-slot window; the lowest peer adds __popc(peers) to the
//           warp's smem row cnt[w][e].
//   scan    per expert, exclusive prefix over the 32 warp rows -> tot[e] and
//           each warp's starting rank for that expert (stable counting sort).
//   pin     single-replica activated experts, in parallel (order-free counts).
//   greedy  warp 0, multi-replica activated experts in ascending id: lane g
//           holds load[g] in a register; key = load<<5 | g for the expert's
//           hosts (bitmask), __reduce_min_sync picks the least-loaded host with
//           ties to the lowest instance id — exactly aebs.cpp:186-194.
//   finish  per expert: replica id, replica-order index q, routed tokens;
//           block scans give group_off[q] (rows per replica group) and the
//           n-tile prefix the grouped GEMM walks.
//   pass 2  the same windows again: row = group_off[q(e)] + warp base + rank
//           among equal ids in the window -> slot_row / row_slot, and the
//           Assignment's per-slot instance / replica.
#include <climits>

#include "internal.h"

namespace janus {
namespace {

constexpr unsigned kFull = 0xffffffffu;

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

__global__ void __launch_bounds__(kSchedThreads, 1) aebs_schedule_kernel(SchedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int E = a.map.E, N = a.map.N, R = a.map.R, S = a.S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t *__restrict__ off = a.map.off;
  const int32_t *__restrict__ hosts = a.map.hosts;
  const uint32_t *__restrict__ hmask = a.map.hmask;

  unsigned long long *routed = reinterpret_cast<unsigned long long *>(smem);  // [N]
  int32_t *cnt = reinterpret_cast<int32_t *>(routed + N);                   // [32][E]
  int32_t *tot = cnt + 32 * E;                                              // [E]
  int32_t *chg = tot + E;                                                   // [E]
  int32_t *qof = chg + E;                                                   // [E]
  int32_t *ridof = qof + E;                                                 // [E]
  int32_t *load = ridof + E;                                                // [N]
  int32_t *qcnt = load + N;                                                 // [R+1]
  int32_t *tcnt = qcnt + R + 1;                                             // [R+1]
  __shared__ int32_t s_bad;
  __shared__ int32_t s_scan[64];

  for (int i = tid; i < 32 * E; i += kSchedThreads) cnt[i] = 0;
  for (int e = tid; e < E; e += kSchedThreads) chg[e] = -1;
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

  // ---- pass 1: warp-private histogram over this warp's slot range --------
  const int per = ((S + 31) / 32 + 31) & ~31;
  const int beg = min(S, warp * per), end = min(S, beg + per);
  int32_t *mycnt = cnt + warp * E;
  {
    int nxt = beg + lane < end ? __ldg(a.experts + beg + lane) : 0;
    for (int base = beg; base < end; base += 32) {
      const int s = base + lane;
      const int e = nxt;
      nxt = s + 32 < end ? __ldg(a.experts + s + 32) : 0;  // prefetch next window
      const bool in = s < end;
      const bool valid = in && e >= 0 && e < E;
      if (in && !valid) atomicMin(&s_bad, e);
      const unsigned vm = __ballot_sync(kFull, valid);
      if (valid) {
        const unsigned peers = __match_any_sync(vm, e);
        if (lane == __ffs(peers) - 1) mycnt[e] += __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (s_bad != INT_MAX) {
    if (tid == 0) {
      a.out.status[0] = JANUS_EUNKNOWN_EXPERT;
      a.out.status[1] = s_bad;
    }
    return;
  }

  // ---- per-expert prefix over warps ---------------------------------------
  for (int e = tid; e < E; e += kSchedThreads) {
    int run = 0;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) {
      const int c = cnt[w * E + e];
      cnt[w * E + e] = run;
      run += c;
    }
    tot[e] = run;
    // A validated map gives every expert a replica; keep the reference's
    // second check (aebs.cpp:164-166) for completeness.
    if (run > 0 && off[e + 1] == off[e]) atomicMin(&s_bad, e);
  }
  __syncthreads();
  if (s_bad != INT_MAX) {
    if (tid == 0) {
      a.out.status[0] = JANUS_EUNKNOWN_EXPERT;
      a.out.status[1] = s_bad;
    }
    return;
  }

  // ---- pin single-replica experts (aebs.cpp:180-185) ----------------------
  for (int e = tid; e < E; e += kSchedThreads)
    if (tot[e] > 0 && off[e + 1] - off[e] == 1) {
      const int g = hosts[off[e]];
      chg[e] = g;
      atomicAdd(&load[g], 1);
    }
  __syncthreads();

  // ---- sequential phase, warp 0 --------------------------------------------
  if (warp == 0) {
    if (a.policy == JANUS_POLICY_AEBS) {
      if (N <= 32) {
        int my = lane < N ? load[lane] : 0;
        for (int cb = 0; cb < E; cb += 32) {
          const int e = cb + lane;
          const bool multi = e < E && tot[e] > 0 && off[e + 1] - off[e] > 1;
          unsigned mm = __ballot_sync(kFull, multi);
          const uint32_t myhm = multi ? hmask[e] : 0u;
          while (mm) {
            const int b = __ffs(mm) - 1;
            mm &= mm - 1;
            const uint32_t hm = __shfl_sync(kFull, myhm, b);
            const uint32_t key = ((hm >> lane) & 1u) ? ((uint32_t)my << 5) | (uint32_t)lane
                                                     : 0xffffffffu;
            const int g = (int)(__reduce_min_sync(kFull, key) & 31u);
            my += (lane == g);
            if (lane == b) chg[e] = g;
          }
        }
        if (lane < N) load[lane] = my;
      } else {
        for (int e = 0; e < E; ++e) {
          const int r = off[e + 1] - off[e];
          if (tot[e] == 0 || r <= 1) continue;
          uint32_t best = 0xffffffffu;
          for (int i = lane; i < r; i += 32)
            best = min(best, ((uint32_t)load[hosts[off[e] + i]] << 11) | (uint32_t)i);
          best = __reduce_min_sync(kFull, best);
          const int g = hosts[off[e] + (int)(best & 2047u)];
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
        const int r = off[e + 1] - off[e];
        if (tot[e] == 0 || r <= 1) continue;
        const int g = hosts[off[e] + (int)next_below(st, (uint64_t)r)];
        chg[e] = g;
        load[g] += 1;
      }
    }
  }
  __syncthreads();

  // ---- finish_assignment per expert (aebs.cpp:94-108) ---------------------
  for (int e = tid; e < E; e += kSchedThreads) {
    const int g = chg[e];
    if (g >= 0) {
      int p = off[e];
      if (N <= 32) {
        p += __popc(hmask[e] & ((1u << g) - 1u));
      } else {
        while (hosts[p] != g) ++p;
      }
      ridof[e] = a.map.rid[p];
      const int q = a.map.qidx[p];
      qof[e] = q;
      qcnt[q] = tot[e];
      tcnt[q] = (tot[e] + kTileN - 1) / kTileN;
      atomicAdd(&routed[g], (unsigned long long)tot[e]);
    }
    a.out.expert_instance[e] = g;
    if (a.out.expert_tokens) a.out.expert_tokens[e] = tot[e];
  }
  __syncthreads();
  block_exscan2(qcnt, tcnt, R + 1, s_scan);
  if (a.out.group_off)
    for (int q = tid; q <= R; q += kSchedThreads) a.out.group_off[q] = qcnt[q];
  if (a.tile_off)
    for (int q = tid; q <= R; q += kSchedThreads) a.tile_off[q] = tcnt[q];
  for (int g = tid; g < N; g += kSchedThreads) {
    a.out.load[g] = load[g];
    a.out.routed_tokens[g] = (int64_t)routed[g];
  }

  // ---- pass 2: remap slots and lay out rows --------------------------------
  {
    int32_t *__restrict__ o_inst = a.out.instance;
    int32_t *__restrict__ o_repl = a.out.replica;
    int32_t *__restrict__ o_srow = a.out.slot_row;
    int32_t *__restrict__ o_rslot = a.out.row_slot;
    int nxt = beg + lane < end ? __ldg(a.experts + beg + lane) : 0;
    for (int base = beg; base < end; base += 32) {
      const int s = base + lane;
      const int e = nxt;
      nxt = s + 32 < end ? __ldg(a.experts + s + 32) : 0;
      const bool in = s < end;
      const unsigned vm = __ballot_sync(kFull, in);
      if (in) {
        const unsigned peers = __match_any_sync(vm, e);
        const int rank = __popc(peers & lanemask_lt());
        const int cbase = mycnt[e];
        const int row = qcnt[qof[e]] + cbase + rank;
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
  if (tid == 0) {
    a.out.status[0] = JANUS_OK;
    a.out.status[1] = 0;
  }
}

}  // namespace

size_t schedule_smem_bytes(int E, int N, int R) {
  return (size_t)N * 8 + (size_t)32 * E * 4 + (size_t)4 * E * 4 + (size_t)N * 4 +
         (size_t)2 * (R + 1) * 4;
}

cudaError_t launch_schedule(const SchedArgs &a, cudaStream_t stream) {
  const size_t smem = schedule_smem_bytes(a.map.E, a.map.N, a.map.R);
  // The opt-in limit is per device and per function; raise it when a larger
  // map needs more (227 KB minus the kernel's static shared memory at most).
  static int configured_dev = -1;
  static size_t configured_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev || smem > configured_smem) {
    const size_t want = smem > 48 * 1024 ? smem : 48 * 1024;
    cudaError_t err = cudaFuncSetAttribute(aebs_schedule_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    if (err != cudaSuccess) return err;
    configured_dev = dev;
    configured_smem = want;
  }
  aebs_schedule_kernel<<<1, kSchedThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace janus
