// stats.cu — GPU activation statistics: the reference's
// ActivationStats::record_step (experts.cpp:30-57) — per-expert activation
// counts and the E x E co-activation matrix over a sliding window of steps —
// kept on the device and updated from a step's routing without a host round
// trip.  Bit-exact with the reference (tests/test_gpu_stats.py).
//
// State: counts[E] and coact[E*E] (int64), a ring of the last W activated
// sets as bitmasks (W x ceil(E/32) words), the device step counter and an
// error word.  One record = three stream-ordered kernels:
//   stats_mask_kernel    one CTA: the step's activated bitmask from the
//                        top-k ids (smem atomicOr), the minimum out-of-range
//                        id if any (the reference rejects the step: no change)
//   stats_update_kernel  one CTA per row i: coact[i][j] += new_i·new_j −
//                        old_i·old_j (j ≠ i), counts[i] += new_i − old_i, where
//                        old = the set retiring from the window (step >= W)
//   stats_commit_kernel  ring slot <- new set, step += 1
// Rows with neither bit set are skipped, so the update costs O(A·E), not E².
#include <climits>

#include "internal.h"

namespace janus {
namespace {

constexpr int kStatsThreads = 1024;

__global__ void stats_mask_kernel(const int32_t *__restrict__ experts, long long S, int E,
                                  int words, uint32_t *__restrict__ mask, int *__restrict__ bad) {
  extern __shared__ uint32_t sm[];
  __shared__ int s_bad;
  for (int w = threadIdx.x; w < words; w += blockDim.x) sm[w] = 0;
  if (threadIdx.x == 0) s_bad = INT_MAX;
  __syncthreads();
  for (long long s = threadIdx.x; s < S; s += blockDim.x) {
    const int e = __ldg(experts + s);
    if (e < 0 || e >= E)
      atomicMin(&s_bad, e);
    else
      atomicOr(&sm[e >> 5], 1u << (e & 31));
  }
  __syncthreads();
  for (int w = threadIdx.x; w < words; w += blockDim.x) mask[w] = sm[w];
  if (threadIdx.x == 0) *bad = s_bad;
}

__global__ void stats_update_kernel(const uint32_t *__restrict__ mask, const uint32_t *ring,
                                    const long long *step_p, const int *bad, int E, int W,
                                    int words, long long *__restrict__ counts,
                                    long long *__restrict__ coact) {
  if (*bad != INT_MAX) return;  // rejected step: the window is unchanged
  const long long step = *step_p;
  const uint32_t *old = step >= W ? ring + (size_t)(step % W) * words : nullptr;
  const int i = blockIdx.x;
  const int ni = (mask[i >> 5] >> (i & 31)) & 1;
  const int oi = old ? (old[i >> 5] >> (i & 31)) & 1 : 0;
  if (!ni && !oi) return;
  if (threadIdx.x == 0) counts[i] += ni - oi;
  long long *row = coact + (size_t)i * E;
  for (int j = threadIdx.x; j < E; j += blockDim.x) {
    if (j == i) continue;
    const int nj = (mask[j >> 5] >> (j & 31)) & 1;
    const int oj = old ? (old[j >> 5] >> (j & 31)) & 1 : 0;
    const int d = (ni & nj) - (oi & oj);
    if (d) row[j] += d;
  }
}

__global__ void stats_commit_kernel(const uint32_t *__restrict__ mask, uint32_t *ring,
                                    long long *step_p, const int *bad, int W, int words) {
  if (*bad != INT_MAX) return;
  const long long step = *step_p;
  uint32_t *slot = ring + (size_t)(step % W) * words;
  for (int w = threadIdx.x; w < words; w += blockDim.x) slot[w] = mask[w];
  __syncthreads();
  if (threadIdx.x == 0) *step_p = step + 1;
}

}  // namespace

cudaError_t launch_stats_record(const StatsState &st, const int32_t *experts, long long S,
                                cudaStream_t s) {
  const int words = (st.E + 31) / 32;
  stats_mask_kernel<<<1, kStatsThreads, words * sizeof(uint32_t), s>>>(experts, S, st.E, words,
                                                                       st.mask, st.bad);
  stats_update_kernel<<<st.E, 256, 0, s>>>(st.mask, st.ring, st.step, st.bad, st.E, st.W, words,
                                           st.counts, st.coact);
  stats_commit_kernel<<<1, 256, 0, s>>>(st.mask, st.ring, st.step, st.bad, st.W, words);
  return cudaGetLastError();
}

}  // namespace janus
