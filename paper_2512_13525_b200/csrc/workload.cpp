// workload.cpp — synthetic routing for benches and examples: moesim::gen_batch
// (src/workload.cpp:56-130) over a RoutingPattern cdf (:11-54), bit-exact.
// Host-side input generation, outside every timed region.
#include <algorithm>
#include <cstdint>

#include "janus_b200.h"

namespace {

uint64_t splitmix64(uint64_t &s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double next_double(uint64_t &s) { return static_cast<double>(splitmix64(s) >> 11) * 0x1.0p-53; }

int sample(const double *cdf, int E, double u) {
  const double *it = std::lower_bound(cdf, cdf + E, u);
  if (it == cdf + E) --it;
  return static_cast<int>(it - cdf);
}

}  // namespace

extern "C" janus_status janus_gen_batch(const double *cdf, int E, int T, int k, uint64_t seed,
                                        uint64_t step, int32_t *out) {
  if (T < 0 || k < 1 || k > E) return JANUS_EINVAL;
  const uint64_t step_seed = janus_derive_seed(seed, "workload/step", step);
#pragma omp parallel for schedule(static) if (T >= 256)
  for (int i = 0; i < T; ++i) {
    uint64_t st = janus_derive_seed(step_seed, "token", static_cast<uint64_t>(i));
    int32_t *row = out + static_cast<size_t>(i) * k;
    int chosen = 0;
    while (chosen < k) {
      int e = -1;
      for (int attempt = 0; attempt < 64; ++attempt) {
        const int cand = sample(cdf, E, next_double(st));
        if (std::find(row, row + chosen, cand) == row + chosen) {
          e = cand;
          break;
        }
      }
      if (e < 0) {
        const int cand = sample(cdf, E, next_double(st));
        for (int o = 0; o < E; ++o) {
          const int c = (cand + o) % E;
          if (std::find(row, row + chosen, c) == row + chosen) {
            e = c;
            break;
          }
        }
      }
      row[chosen++] = e;
    }
    std::sort(row, row + k);
  }
  return JANUS_OK;
}
