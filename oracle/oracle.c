/*
 * oracle.c — CPU restatement of the reference (moesim, arXiv 2512.13525
 * "Janus") MoE-side hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2512_13525_b200/) never links or calls
 * it.
 *
 * Parity is pinned two ways (see tests/test_oracle_golden.py):
 *   - against the reference's own golden vectors (test_rng.cpp:17-18 SplitMix64
 *     values, test_aebs.cpp:83-114 worked examples, acceptance.cpp:84 C02
 *     frozen gap histogram {496,4,0}, configs/sample-* fixture);
 *   - against the reference itself compiled here from /root/reference sources
 *     into oracle/_ref/libmoesim_ref.so (oracle/Makefile), on random cases.
 *
 * Reference paths are relative to /root/reference/proj.
 *
 * Rows A9 (dispatch layout), A13 (SwiGLU expert FFN) and A14 (combine) have no
 * reference implementation; they are defined here and in
 * DESIGN.md, and are "parity unpinned" beyond their definition.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL 1
#define OR_EUNKNOWN_EXPERT 2
#define OR_EINFEASIBLE 3

/* ---------------------------------------------------------------- rng ---- */

/* include/moesim/rng.hpp:13-19 */
uint64_t or_splitmix64(uint64_t *state) {
  *state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* include/moesim/rng.hpp:22-29 (FNV-1a) */
uint64_t or_hash_label(const char *label) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const unsigned char *p = (const unsigned char *)label; *p; ++p) {
    h ^= *p;
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* include/moesim/rng.hpp:34-44 */
uint64_t or_derive_seed(uint64_t root, const char *label, uint64_t extra) {
  uint64_t s = root;
  or_splitmix64(&s);
  s ^= or_hash_label(label);
  or_splitmix64(&s);
  uint64_t e = extra;
  s ^= or_splitmix64(&e);
  return or_splitmix64(&s);
}

/* include/moesim/rng.hpp:53-61 (Rng::next_below, rejection) */
uint64_t or_next_below(uint64_t *state, uint64_t n) {
  if (n == 0) return 0;
  uint64_t threshold = (0 - n) % n;
  for (;;) {
    uint64_t r = or_splitmix64(state);
    if (r >= threshold) return r % n;
  }
}

/* include/moesim/rng.hpp:63 */
double or_next_double(uint64_t *state) {
  return (double)(or_splitmix64(state) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------ routing ---- */

/* src/workload.cpp:11-30 RoutingPattern::from_pmf.  Writes pmf and cdf (E
 * doubles each).  Returns OR_EINVAL on the reference's ValidationError cases. */
int or_pattern_from_pmf(const double *w, int E, double *pmf, double *cdf) {
  if (E <= 0) return OR_EINVAL;
  double sum = 0;
  for (int i = 0; i < E; ++i) {
    if (!(w[i] >= 0)) return OR_EINVAL;
    sum += w[i];
  }
  if (sum <= 0) return OR_EINVAL;
  double acc = 0;
  for (int i = 0; i < E; ++i) {
    pmf[i] = w[i] / sum;
    acc += pmf[i];
    cdf[i] = acc;
  }
  cdf[E - 1] = 1.0;
  return OR_OK;
}

/* src/workload.cpp:32-35 */
int or_pattern_uniform(int E, double *pmf, double *cdf) {
  if (E < 1) return OR_EINVAL;
  double *w = (double *)malloc(sizeof(double) * E);
  for (int i = 0; i < E; ++i) w[i] = 1.0;
  int rc = or_pattern_from_pmf(w, E, pmf, cdf);
  free(w);
  return rc;
}

/* src/workload.cpp:37-48 */
int or_pattern_gaussian(int E, double sigma, double *pmf, double *cdf) {
  if (E < 1 || !(sigma > 0)) return OR_EINVAL;
  double center = E / 2.0;
  double denom = 2.0 * (sigma * E) * (sigma * E);
  double *w = (double *)malloc(sizeof(double) * E);
  for (int e = 0; e < E; ++e) {
    double d = e - center;
    w[e] = exp(-d * d / denom);
  }
  int rc = or_pattern_from_pmf(w, E, pmf, cdf);
  free(w);
  return rc;
}

/* src/workload.cpp:50-54: smallest id with cdf >= u (std::lower_bound). */
int or_pattern_sample(const double *cdf, int E, double u) {
  int lo = 0, hi = E;
  while (lo < hi) {
    int mid = lo + (hi - lo) / 2;
    if (cdf[mid] < u) lo = mid + 1;
    else hi = mid;
  }
  if (lo == E) --lo;
  return lo;
}

static int row_has(const int32_t *row, int n, int32_t v) {
  for (int i = 0; i < n; ++i)
    if (row[i] == v) return 1;
  return 0;
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* src/workload.cpp:56-130 gen_batch.  out: T*k int32, token-major, each row
 * sorted ascending (:98).  cover_all restated from :101-126. */
int or_gen_batch(const double *cdf, int E, int T, int k, uint64_t seed, uint64_t step,
                 int cover_all, int32_t *out) {
  if (T < 0) return OR_EINVAL;
  if (k < 1 || k > E) return OR_EINVAL;
  uint64_t step_seed = or_derive_seed(seed, "workload/step", step);
#pragma omp parallel for schedule(static) if (T >= 256)
  for (int i = 0; i < T; ++i) {
    uint64_t st = or_derive_seed(step_seed, "token", (uint64_t)i);
    int32_t *row = out + (size_t)i * k;
    int chosen = 0;
    while (chosen < k) {
      int e = -1;
      for (int attempt = 0; attempt < 64; ++attempt) {
        int cand = or_pattern_sample(cdf, E, or_next_double(&st));
        if (!row_has(row, chosen, cand)) {
          e = cand;
          break;
        }
      }
      if (e < 0) {
        int cand = or_pattern_sample(cdf, E, or_next_double(&st));
        for (int off = 0; off < E; ++off) {
          int c = (cand + off) % E;
          if (!row_has(row, chosen, c)) {
            e = c;
            break;
          }
        }
      }
      row[chosen++] = e;
    }
    qsort(row, k, sizeof(int32_t), cmp_i32);
  }
  if (cover_all && T > 0) {
    if ((long long)T * k < E) return OR_EINFEASIBLE;
    int *counts = (int *)calloc(E, sizeof(int));
    for (long long s = 0; s < (long long)T * k; ++s) ++counts[out[s]];
    size_t cursor = 0, total = (size_t)T * k;
    for (int miss = 0; miss < E; ++miss) {
      if (counts[miss] > 0) continue;
      int placed = 0;
      for (size_t tries = 0; tries < total && !placed; ++tries, ++cursor) {
        size_t s = cursor % total;
        size_t tok = s / k;
        int old = out[s];
        if (counts[old] < 2) continue;
        int32_t *row = out + tok * k;
        if (row_has(row, k, miss)) continue;
        --counts[old];
        out[s] = miss;
        counts[miss] = 1;
        qsort(row, k, sizeof(int32_t), cmp_i32);
        placed = 1;
      }
      if (!placed) {
        free(counts);
        return OR_EINFEASIBLE;
      }
    }
    free(counts);
  }
  return OR_OK;
}

/* ---------------------------------------------------------- scheduler ---- */

/* The replica map in CSR form: hosts[off[e]..off[e+1]) strictly ascending,
 * rid[] parallel (include/moesim/aebs.hpp:29-38). */
typedef struct {
  int E, N, C;
  const int32_t *off, *hosts, *rid;
} or_map;

/* src/aebs.cpp:49-77 ReplicaMap::validate. */
int or_map_validate(int E, int N, int C, const int32_t *off, const int32_t *hosts) {
  if (E <= 0 || N <= 0 || C <= 0) return OR_EINVAL;
  if (off[0] != 0) return OR_EINVAL;
  int *used = (int *)calloc(N, sizeof(int));
  int rc = OR_OK;
  for (int e = 0; e < E && rc == OR_OK; ++e) {
    if (off[e + 1] <= off[e]) rc = OR_EINVAL; /* "has no replica" */
    for (int i = off[e]; i < off[e + 1] && rc == OR_OK; ++i) {
      int g = hosts[i];
      if (g < 0 || g >= N) rc = OR_EINVAL;
      else if (i > off[e] && hosts[i - 1] >= g) rc = OR_EINVAL;
      else ++used[g];
    }
  }
  for (int g = 0; g < N && rc == OR_OK; ++g)
    if (used[g] > C) rc = OR_EINVAL;
  free(used);
  return rc;
}

/* Policies. */
#define OR_POLICY_AEBS 0       /* schedule() / schedule_reference() */
#define OR_POLICY_RANDOM 1     /* schedule_random() */
#define OR_POLICY_BRUTE 2      /* brute_force_schedule() */

/* src/aebs.cpp:89-122 finish_assignment: given choice_pos[e] (-1 inactive),
 * fill per-slot and per-instance tables. */
static void finish(const int32_t *experts, long long S, const or_map *m, const int32_t *choice,
                   const long long *etok, int32_t *instance, int32_t *replica,
                   int32_t *expert_instance, int32_t *load, long long *routed) {
  int32_t *slot_of = (int32_t *)malloc(sizeof(int32_t) * m->E);
  for (int g = 0; g < m->N; ++g) {
    load[g] = 0;
    routed[g] = 0;
  }
  for (int e = 0; e < m->E; ++e) {
    expert_instance[e] = -1;
    slot_of[e] = -1;
    if (choice[e] < 0) continue;
    int g = m->hosts[m->off[e] + choice[e]];
    expert_instance[e] = g;
    slot_of[e] = m->rid[m->off[e] + choice[e]];
    load[g] += 1;
    routed[g] += etok[e];
  }
  for (long long s = 0; s < S; ++s) {
    instance[s] = expert_instance[experts[s]];
    replica[s] = slot_of[experts[s]];
  }
  free(slot_of);
}

/* src/aebs.cpp:126-168 collect_activated.  Returns OR_EUNKNOWN_EXPERT with
 * *bad = the MINIMUM out-of-range id (schedule()'s convention, :137-162). */
static int collect(const int32_t *experts, long long S, const or_map *m, long long *etok,
                   int32_t *bad) {
  int32_t mn = INT32_MAX;
  for (int e = 0; e < m->E; ++e) etok[e] = 0;
  for (long long s = 0; s < S; ++s) {
    int32_t e = experts[s];
    if (e < 0 || e >= m->E) {
      if (e < mn) mn = e;
    } else {
      ++etok[e];
    }
  }
  if (mn != INT32_MAX) {
    *bad = mn;
    return OR_EUNKNOWN_EXPERT;
  }
  for (int e = 0; e < m->E; ++e)
    if (etok[e] > 0 && m->off[e + 1] == m->off[e]) {
      *bad = e;
      return OR_EUNKNOWN_EXPERT;
    }
  return OR_OK;
}

/* Exhaustive oracle, src/aebs.cpp:264-321: minimum max-load, lexicographically
 * smallest choice vector over ascending expert ids.  Guard: <= 20 activated,
 * <= 1e6 combinations, else OR_EINVAL. */
static int brute_choice(const or_map *m, const long long *etok, int32_t *choice) {
  int A = 0;
  double combos = 1;
  int *multi = (int *)malloc(sizeof(int) * m->E);
  int nm = 0;
  int32_t *base = (int32_t *)calloc(m->N, sizeof(int32_t));
  for (int e = 0; e < m->E; ++e) {
    choice[e] = -1;
    if (etok[e] == 0) continue;
    ++A;
  }
  int rc = OR_OK;
  if (A > 20) rc = OR_EINVAL;
  for (int e = 0; e < m->E && rc == OR_OK; ++e) {
    if (etok[e] == 0) continue;
    int r = m->off[e + 1] - m->off[e];
    combos *= (double)r;
    if (combos > 1e6) rc = OR_EINVAL;
  }
  if (rc != OR_OK) {
    free(multi);
    free(base);
    return rc;
  }
  for (int e = 0; e < m->E; ++e) {
    if (etok[e] == 0) continue;
    int r = m->off[e + 1] - m->off[e];
    if (r == 1) {
      ++base[m->hosts[m->off[e]]];
      choice[e] = 0;
    } else {
      multi[nm++] = e;
    }
  }
  int32_t *pos = (int32_t *)calloc(nm > 0 ? nm : 1, sizeof(int32_t));
  int32_t *best_pos = (int32_t *)calloc(nm > 0 ? nm : 1, sizeof(int32_t));
  int32_t *load = (int32_t *)malloc(sizeof(int32_t) * m->N);
  int best = INT32_MAX;
  for (;;) {
    memcpy(load, base, sizeof(int32_t) * m->N);
    for (int i = 0; i < nm; ++i) ++load[m->hosts[m->off[multi[i]] + pos[i]]];
    int peak = 0;
    for (int g = 0; g < m->N; ++g)
      if (load[g] > peak) peak = load[g];
    if (peak < best) {
      best = peak;
      memcpy(best_pos, pos, sizeof(int32_t) * (nm > 0 ? nm : 1));
    }
    int i = nm;
    int done = 1;
    while (i > 0) {
      --i;
      if (++pos[i] < m->off[multi[i] + 1] - m->off[multi[i]]) {
        done = 0;
        break;
      }
      pos[i] = 0;
    }
    if (done) break;
  }
  for (int i = 0; i < nm; ++i) choice[multi[i]] = best_pos[i];
  free(pos);
  free(best_pos);
  free(load);
  free(multi);
  free(base);
  return OR_OK;
}

/* The scheduling pass.
 *   AEBS   — src/aebs.cpp:199-248 schedule_reference (identical outputs to
 *            schedule(), :172-197): pin single-replica experts (:213-221),
 *            then multi-replica experts ascending to the least-loaded host,
 *            ties to the lowest instance id (:222-229).
 *   RANDOM — src/aebs.cpp:250-262 schedule_random: Rng(derive_seed(seed,
 *            "sched/random")), one next_below(R) per activated multi-replica
 *            expert in ascending id order.
 *   BRUTE  — src/aebs.cpp:264-321.
 * bad_mode 0: *bad = min bad id (schedule(), aebs.cpp:137-162);
 * bad_mode 1: *bad = first bad id in slot order (schedule_reference, :206). */
int or_schedule(int policy, int bad_mode, uint64_t seed, const int32_t *experts, int T, int k,
                int E, int N, int C, const int32_t *off, const int32_t *hosts,
                const int32_t *rid, int32_t *instance, int32_t *replica,
                int32_t *expert_instance, int32_t *load, long long *routed,
                long long *expert_tokens, int32_t *bad) {
  or_map m = {E, N, C, off, hosts, rid};
  long long S = (long long)T * k;
  if (bad_mode == 1) {
    for (long long s = 0; s < S; ++s)
      if (experts[s] < 0 || experts[s] >= E) {
        *bad = experts[s];
        return OR_EUNKNOWN_EXPERT;
      }
  }
  long long *etok = (long long *)malloc(sizeof(long long) * (E > 0 ? E : 1));
  int rc = collect(experts, S, &m, etok, bad);
  if (rc != OR_OK) {
    free(etok);
    return rc;
  }
  int32_t *choice = (int32_t *)malloc(sizeof(int32_t) * E);
  if (policy == OR_POLICY_AEBS) {
    int32_t *ld = (int32_t *)calloc(N, sizeof(int32_t));
    for (int e = 0; e < E; ++e) {
      choice[e] = -1;
      if (etok[e] == 0) continue;
      if (off[e + 1] - off[e] == 1) {
        choice[e] = 0;
        ++ld[hosts[off[e]]];
      }
    }
    for (int e = 0; e < E; ++e) {
      if (etok[e] == 0 || off[e + 1] - off[e] <= 1) continue;
      int best = 0;
      for (int i = 1; i < off[e + 1] - off[e]; ++i)
        if (ld[hosts[off[e] + i]] < ld[hosts[off[e] + best]]) best = i;
      choice[e] = best;
      ++ld[hosts[off[e] + best]];
    }
    free(ld);
  } else if (policy == OR_POLICY_RANDOM) {
    uint64_t st = or_derive_seed(seed, "sched/random", 0);
    for (int e = 0; e < E; ++e) {
      choice[e] = -1;
      if (etok[e] == 0) continue;
      uint64_t r = (uint64_t)(off[e + 1] - off[e]);
      choice[e] = r == 1 ? 0 : (int32_t)or_next_below(&st, r);
    }
  } else if (policy == OR_POLICY_BRUTE) {
    rc = brute_choice(&m, etok, choice);
    if (rc != OR_OK) {
      free(choice);
      free(etok);
      return rc;
    }
  } else {
    free(choice);
    free(etok);
    return OR_EINVAL;
  }
  finish(experts, S, &m, choice, etok, instance, replica, expert_instance, load, routed);
  if (expert_tokens)
    for (int e = 0; e < E; ++e) expert_tokens[e] = etok[e];
  free(choice);
  free(etok);
  return OR_OK;
}

/* ---------------------------------------------- dispatch layout (A9) ---- */

/* Per-instance replica order: the replicas hosted on
 * instance g, sorted by (replica id, expert id).  Flat index
 * q = qbase[g] + rank.  qidx[off[e]+p] receives q of (e, p); qexpert[q] the
 * expert held at q; qbase has N+1 entries. */
int or_replica_order(int E, int N, const int32_t *off, const int32_t *hosts, const int32_t *rid,
                     int32_t *qidx, int32_t *qexpert, int32_t *qbase) {
  int R = off[E];
  for (int g = 0; g <= N; ++g) qbase[g] = 0;
  for (int i = 0; i < R; ++i) qbase[hosts[i] + 1]++;
  for (int g = 0; g < N; ++g) qbase[g + 1] += qbase[g];
  for (int e = 0; e < E; ++e)
    for (int p = off[e]; p < off[e + 1]; ++p) {
      int g = hosts[p];
      int rank = 0;
      for (int e2 = 0; e2 < E; ++e2)
        for (int p2 = off[e2]; p2 < off[e2 + 1]; ++p2) {
          if (hosts[p2] != g) continue;
          if (rid[p2] < rid[p] || (rid[p2] == rid[p] && e2 < e)) ++rank;
        }
      qidx[p] = qbase[g] + rank;
      qexpert[qbase[g] + rank] = e;
    }
  return OR_OK;
}

/* Dispatch layout of one step: rows grouped by q (instance-major, replica
 * order within an instance), slots of one expert in ascending slot order.
 * group_off: R+1 entries; slot_row: S; row_slot: S. */
int or_dispatch_layout(const int32_t *experts, int T, int k, int E, const int32_t *off,
                       const int32_t *hosts, const int32_t *qidx, const int32_t *expert_instance,
                       int32_t *group_off, int32_t *slot_row, int32_t *row_slot) {
  long long S = (long long)T * k;
  int R = off[E];
  int32_t *qof = (int32_t *)malloc(sizeof(int32_t) * E);
  int32_t *cnt = (int32_t *)calloc(R + 1, sizeof(int32_t));
  for (int e = 0; e < E; ++e) {
    qof[e] = -1;
    if (expert_instance[e] < 0) continue;
    for (int p = off[e]; p < off[e + 1]; ++p)
      if (hosts[p] == expert_instance[e]) qof[e] = qidx[p];
  }
  for (long long s = 0; s < S; ++s) cnt[qof[experts[s]]]++;
  group_off[0] = 0;
  for (int q = 0; q < R; ++q) group_off[q + 1] = group_off[q] + cnt[q];
  for (int q = 0; q < R; ++q) cnt[q] = 0;
  for (long long s = 0; s < S; ++s) {
    int q = qof[experts[s]];
    int r = group_off[q] + cnt[q]++;
    slot_row[s] = r;
    row_slot[r] = (int32_t)s;
  }
  free(qof);
  free(cnt);
  return OR_OK;
}

/* ------------------------------------------------ latency model (A12) ---- */

/* src/latency.cpp:17-24 moe_instance_latency (2 weight matrices, 2 FLOP per
 * (token, d_h*d_e) — the reference's accounting, kept as is). */
double or_moe_instance_latency(int activated, long long routed, int d_h, int d_e, int bpp,
                               double peak_flops, double hbm_bw, double t_launch) {
  if (activated <= 0) return 0;
  double wbytes = 2.0 * d_h * d_e * bpp;
  double mem = activated * wbytes / hbm_bw;
  double comp = 2.0 * (double)routed * d_h * d_e / peak_flops;
  return t_launch + (mem > comp ? mem : comp);
}

/* src/latency.cpp:26-32 */
double or_moe_layer_latency(int N, const int32_t *load, const long long *routed, int d_h,
                            int d_e, int bpp, double peak_flops, double hbm_bw,
                            double t_launch) {
  double worst = 0;
  for (int g = 0; g < N; ++g) {
    double t = or_moe_instance_latency(load[g], routed[g], d_h, d_e, bpp, peak_flops, hbm_bw,
                                       t_launch);
    if (t > worst) worst = t;
  }
  return worst;
}

/* ------------------------------------------- expert FFN + combine (A13/A14) */

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40); /* NaN */
  u += 0x7fffu + ((u >> 16) & 1u);                                           /* RNE */
  return (uint16_t)(u >> 16);
}

void or_f32_to_bf16(const float *in, uint16_t *out, long long n) {
  for (long long i = 0; i < n; ++i) out[i] = f32_to_bf16(in[i]);
}

void or_bf16_to_f32(const uint16_t *in, float *out, long long n) {
  for (long long i = 0; i < n; ++i) out[i] = bf16_to_f32(in[i]);
}

/* SwiGLU expert over a set of token rows (A13):
 *   g = x·Wgᵀ, u = x·Wuᵀ (fp32 accumulate over bf16 inputs)
 *   h = silu(g)·u, optionally rounded to bf16 (round_h: the device keeps h in
 *       bf16 between its two GEMMs)
 *   y = h·Wdᵀ (fp32)
 * x: [n, d_h] bf16; wg, wu: [d_e, d_h] bf16; wd: [d_h, d_e] bf16; y: [n, d_h]
 * fp32.  Threaded over rows with OpenMP when nthreads > 1. */
void or_expert_swiglu(const uint16_t *x, int n, const uint16_t *wg, const uint16_t *wu,
                      const uint16_t *wd, int d_h, int d_e, int round_h, int nthreads,
                      float *y) {
  float *wgf = (float *)malloc(sizeof(float) * (size_t)d_e * d_h);
  float *wuf = (float *)malloc(sizeof(float) * (size_t)d_e * d_h);
  float *wdf = (float *)malloc(sizeof(float) * (size_t)d_h * d_e);
  const long long nw = (long long)d_e * d_h;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
  for (long long i = 0; i < nw; ++i) {
    wgf[i] = bf16_to_f32(wg[i]);
    wuf[i] = bf16_to_f32(wu[i]);
    wdf[i] = bf16_to_f32(wd[i]);
  }
#pragma omp parallel for schedule(dynamic) num_threads(nthreads > 0 ? nthreads : 1)
  for (int r = 0; r < n; ++r) {
    float *xf = (float *)malloc(sizeof(float) * d_h);
    float *h = (float *)malloc(sizeof(float) * d_e);
    for (int i = 0; i < d_h; ++i) xf[i] = bf16_to_f32(x[(size_t)r * d_h + i]);
    for (int f = 0; f < d_e; ++f) {
      const float *a = wgf + (size_t)f * d_h;
      const float *b = wuf + (size_t)f * d_h;
      float g = 0, u = 0;
      for (int i = 0; i < d_h; ++i) {
        g += a[i] * xf[i];
        u += b[i] * xf[i];
      }
      float v = g / (1.0f + expf(-g)) * u;
      h[f] = round_h ? bf16_to_f32(f32_to_bf16(v)) : v;
    }
    for (int o = 0; o < d_h; ++o) {
      const float *c = wdf + (size_t)o * d_e;
      float acc = 0;
      for (int f = 0; f < d_e; ++f) acc += c[f] * h[f];
      y[(size_t)r * d_h + o] = acc;
    }
    free(xf);
    free(h);
  }
  free(wgf);
  free(wuf);
  free(wdf);
}

/* Combine (A14): out[t] = Σ_j w[t*k+j] · y[row(t,j)], j ascending, fp32.
 * y: [rows, d_h] fp32; out: [T, d_h] fp32. */
void or_combine(const float *y, const int32_t *slot_row, const float *w, int T, int k, int d_h,
                float *out) {
  for (int t = 0; t < T; ++t) {
    float *o = out + (size_t)t * d_h;
    for (int i = 0; i < d_h; ++i) o[i] = 0;
    for (int j = 0; j < k; ++j) {
      int r = slot_row[(size_t)t * k + j];
      float wj = w[(size_t)t * k + j];
      const float *yr = y + (size_t)r * d_h;
      for (int i = 0; i < d_h; ++i) o[i] += wj * yr[i];
    }
  }
}

/* MoE-side gating (no reference implementation — Janus gates
 * on the MoE side, the reference only consumes top-k ids):
 *   logits[t][e] = x[t]·Wr[e] (bf16 inputs, accumulated in double here),
 *   top-k by logit descending, ties to the lower expert id (out order = rank),
 *   gate weights = softmax over the k selected logits (Qwen3-MoE's
 *   norm_topk_prob form).
 * x: [T, d_h] bf16; wr: [E, d_h] bf16; experts/gw: [T*k]; logits_out
 * (optional) [T, E] as double. */
void or_gate(const uint16_t *x, const uint16_t *wr, int T, int d_h, int E, int k,
             int32_t *experts, float *gw, double *logits_out) {
  double *lg = (double *)malloc(sizeof(double) * (E > 0 ? E : 1));
  double *wf = (double *)malloc(sizeof(double) * (size_t)E * d_h);
  for (long long i = 0; i < (long long)E * d_h; ++i) wf[i] = bf16_to_f32(wr[i]);
  double *xf = (double *)malloc(sizeof(double) * (d_h > 0 ? d_h : 1));
  for (int t = 0; t < T; ++t) {
    for (int i = 0; i < d_h; ++i) xf[i] = bf16_to_f32(x[(size_t)t * d_h + i]);
    for (int e = 0; e < E; ++e) {
      const double *w = wf + (size_t)e * d_h;
      double acc = 0;
      for (int i = 0; i < d_h; ++i) acc += w[i] * xf[i];
      lg[e] = acc;
      if (logits_out) logits_out[(size_t)t * E + e] = acc;
    }
    int32_t *ex = experts + (size_t)t * k;
    for (int j = 0; j < k; ++j) {  /* selection: largest remaining, lowest id on ties */
      int best = -1;
      for (int e = 0; e < E; ++e) {
        int taken = 0;
        for (int q = 0; q < j; ++q) taken |= ex[q] == e;
        if (!taken && (best < 0 || lg[e] > lg[best])) best = e;
      }
      ex[j] = best;
    }
    double m = lg[ex[0]], sum = 0;
    for (int j = 0; j < k; ++j) sum += exp(lg[ex[j]] - m);
    for (int j = 0; j < k; ++j) gw[(size_t)t * k + j] = (float)(exp(lg[ex[j]] - m) / sum);
  }
  free(lg);
  free(wf);
  free(xf);
}

/* ActivationStats::record_step (experts.cpp:30-57), restated over a ring of
 * the last `window` activated sets kept as bitmasks (the device layout):
 * counts[e] = #steps in the window with e activated, coact[i][j] (i != j) =
 * #steps with both.  `ring` holds window * words uint32 (words = ceil(E/32)),
 * `step` the number of steps recorded before this one.  Returns 0, or 1 + the
 * first bad index if the set is not ascending/distinct/in range (the
 * reference's ValidationError cases). */
int or_stats_record(int E, int window, long long step, uint32_t *ring, long long *counts,
                    long long *coact, const int32_t *activated, int n) {
  const int words = (E + 31) / 32;
  for (int i = 0; i < n; ++i)
    if (activated[i] < 0 || activated[i] >= E || (i > 0 && activated[i - 1] >= activated[i]))
      return 1 + i;
  uint32_t *slot = ring + (size_t)(step % window) * words;
  if (step >= window) { /* retire the oldest step, which lives in this slot */
    for (int i = 0; i < E; ++i) {
      if (!((slot[i >> 5] >> (i & 31)) & 1u)) continue;
      --counts[i];
      for (int j = 0; j < E; ++j)
        if (j != i && ((slot[j >> 5] >> (j & 31)) & 1u)) --coact[(size_t)i * E + j];
    }
  }
  memset(slot, 0, sizeof(uint32_t) * words);
  for (int i = 0; i < n; ++i) slot[activated[i] >> 5] |= 1u << (activated[i] & 31);
  for (int i = 0; i < n; ++i) {
    ++counts[activated[i]];
    for (int j = 0; j < n; ++j)
      if (j != i) ++coact[(size_t)activated[i] * E + activated[j]];
  }
  return 0;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
