// ref_shim.cpp — extern "C" wrapper over the UNMODIFIED reference library
// (moesim, /root/reference/proj/src/{aebs,workload,experts,latency,config}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libmoesim_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin oracle/oracle.c against the
// reference itself, by oracle/make_maps.py to run the reference placement
// pipeline, and by bench.py's CPU-baseline / --impl reference leg to time the
// reference's own schedule() on the host cores.  Never linked by the product.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "moesim/aebs.hpp"
#include "moesim/experts.hpp"
#include "moesim/latency.hpp"
#include "moesim/rng.hpp"
#include "moesim/workload.hpp"

using namespace moesim;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

RoutingPattern make_pattern(int kind, int E, double sigma, const double* w) {
  if (kind == 0) return RoutingPattern::uniform(E);
  if (kind == 1) return RoutingPattern::gaussian(E, sigma);
  return RoutingPattern::from_pmf(std::vector<double>(w, w + E));
}

ReplicaMap make_map(int E, int N, int C, const int32_t* off, const int32_t* hosts,
                    const int32_t* rid) {
  ReplicaMap m;
  m.num_experts = E;
  m.num_instances = N;
  m.slots_per_instance = C;
  m.hosts.resize(E);
  m.replica_ids.resize(E);
  for (int e = 0; e < E; ++e) {
    m.hosts[e].assign(hosts + off[e], hosts + off[e + 1]);
    m.replica_ids[e].assign(rid + off[e], rid + off[e + 1]);
  }
  return m;
}

ActivationBatch make_batch(const int32_t* experts, int T, int k) {
  ActivationBatch b;
  b.num_tokens = T;
  b.top_k = k;
  b.experts.assign(experts, experts + static_cast<size_t>(T) * k);
  return b;
}

Assignment run(int policy, const ActivationBatch& b, const ReplicaMap& m, uint64_t seed) {
  switch (policy) {
    case 0: return schedule(b, m);
    case 1: return schedule_reference(b, m);
    case 2: return schedule_random(b, m, seed);
    default: return brute_force_schedule(b, m);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_splitmix64(uint64_t* state) { return splitmix64(*state); }

uint64_t ref_derive_seed(uint64_t root, const char* label, uint64_t extra) {
  return derive_seed(root, label, extra);
}

// kind: 0 uniform, 1 gaussian(sigma), 2 from_pmf(w)
int ref_pattern(int kind, int E, double sigma, const double* w, double* pmf, double* cdf) {
  try {
    RoutingPattern p = make_pattern(kind, E, sigma, w);
    std::copy(p.pmf.begin(), p.pmf.end(), pmf);
    std::copy(p.cdf.begin(), p.cdf.end(), cdf);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_gen_batch(int kind, int E, double sigma, const double* w, int T, int k, uint64_t seed,
                  uint64_t step, int cover_all, int32_t* out) {
  try {
    ActivationBatch b = gen_batch(make_pattern(kind, E, sigma, w), T, k, seed, step, cover_all);
    std::copy(b.experts.begin(), b.experts.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// policy: 0 schedule, 1 schedule_reference, 2 schedule_random(seed), 3 brute force.
// Returns 0, 1 (ValidationError: message via ref_last_error), 2 (other).
int ref_schedule(int policy, uint64_t seed, const int32_t* experts, int T, int k, int E, int N,
                 int C, const int32_t* off, const int32_t* hosts, const int32_t* rid,
                 int32_t* instance, int32_t* replica, int32_t* expert_instance, int32_t* load,
                 long long* routed) {
  try {
    ReplicaMap m = make_map(E, N, C, off, hosts, rid);
    ActivationBatch b = make_batch(experts, T, k);
    Assignment a = run(policy, b, m, seed);
    std::copy(a.instance.begin(), a.instance.end(), instance);
    std::copy(a.replica.begin(), a.replica.end(), replica);
    std::copy(a.expert_instance.begin(), a.expert_instance.end(), expert_instance);
    std::copy(a.load.begin(), a.load.end(), load);
    std::copy(a.routed_tokens.begin(), a.routed_tokens.end(), routed);
    return 0;
  } catch (const ValidationError& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

int ref_map_validate(int E, int N, int C, const int32_t* off, const int32_t* hosts,
                     const int32_t* rid) {
  try {
    make_map(E, N, C, off, hosts, rid).validate();
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// Median wall time (µs, std::chrono::steady_clock) of `reps` calls, following
// tools/bench_schedule.cpp:41-51.  The batches rotate through `nb` inputs.
double ref_time_schedule(int policy, uint64_t seed, const int32_t* experts, int nb, int T, int k,
                         int E, int N, int C, const int32_t* off, const int32_t* hosts,
                         const int32_t* rid, int reps, int warmup, long long* sink_out) {
  ReplicaMap m = make_map(E, N, C, off, hosts, rid);
  std::vector<ActivationBatch> bs;
  for (int i = 0; i < nb; ++i)
    bs.push_back(make_batch(experts + static_cast<size_t>(i) * T * k, T, k));
  long long sink = 0;
  for (int i = 0; i < warmup; ++i) sink += run(policy, bs[i % nb], m, seed).max_load();
  std::vector<double> t(reps);
  for (int i = 0; i < reps; ++i) {
    auto a = std::chrono::steady_clock::now();
    sink += run(policy, bs[i % nb], m, seed).max_load();
    t[i] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
  }
  std::nth_element(t.begin(), t.begin() + reps / 2, t.end());
  if (sink_out) *sink_out = sink;
  return t[reps / 2];
}

// The DecodeEngine::rebuild_placement recipe (src/sim.cpp:107-122,134-148):
// warm ActivationStats over `steps` gen_batch steps, allocate_replicas ->
// cap_allocation -> place_replicas -> to_replica_map.  Output CSR: off[E+1],
// hosts/rid with capacity N*C.
int ref_placement(int kind, int E, double sigma, const double* w, int k, int N, int C,
                  int warm_steps, int warm_tokens, uint64_t seed, int32_t* off, int32_t* hosts,
                  int32_t* rid) {
  try {
    RoutingPattern pat = make_pattern(kind, E, sigma, w);
    ActivationStats stats(E, 256);
    std::vector<char> seen(E);
    std::vector<int32_t> activated;
    for (int s = 0; s < warm_steps; ++s) {
      ActivationBatch b = gen_batch(pat, warm_tokens, k, seed, derive_seed(seed, "warmup", s));
      std::fill(seen.begin(), seen.end(), 0);
      for (int32_t e : b.experts) seen[e] = 1;
      activated.clear();
      for (int e = 0; e < E; ++e)
        if (seen[e]) activated.push_back(e);
      stats.record_step(activated);
    }
    std::vector<long long> counts = stats.counts();
    bool any = false;
    for (long long c : counts) any = any || c > 0;
    if (!any) counts.assign(E, 1);
    long long budget = std::min(static_cast<long long>(N) * C, static_cast<long long>(N) * E);
    Allocation alloc = cap_allocation(allocate_replicas(counts, static_cast<int>(budget)), counts, N);
    Placement place = place_replicas(alloc, stats, N, C);
    ReplicaMap m = to_replica_map(place);
    off[0] = 0;
    for (int e = 0; e < E; ++e) {
      off[e + 1] = off[e] + static_cast<int32_t>(m.hosts[e].size());
      std::copy(m.hosts[e].begin(), m.hosts[e].end(), hosts + off[e]);
      std::copy(m.replica_ids[e].begin(), m.replica_ids[e].end(), rid + off[e]);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

double ref_moe_layer_latency(int N, const int32_t* load, const long long* routed, int d_h,
                             int d_e, int bpp, double peak_flops, double hbm_bw,
                             double t_launch) {
  ModelSpec m;
  m.hidden_dim = d_h;
  m.expert_dim = d_e;
  m.bytes_per_param = bpp;
  HardwareSpec h;
  h.peak_flops = peak_flops;
  h.hbm_bandwidth = hbm_bw;
  h.kernel_launch_overhead = t_launch;
  std::vector<InstanceLoad> loads(N);
  for (int g = 0; g < N; ++g) loads[g] = {load[g], routed[g]};
  return moe_layer_latency(loads, m, h);
}

// Text formats (src/aebs.cpp:338-479).  Results are written into caller
// buffers; *_len receives the needed size.
int ref_load_replica_map_text(const char* text, int* E, int* N, int* C, int32_t* off,
                              int32_t* hosts, int32_t* rid, int cap) {
  try {
    std::istringstream in(text);
    ReplicaMap m = load_replica_map(in);
    *E = m.num_experts;
    *N = m.num_instances;
    *C = m.slots_per_instance;
    int o = 0;
    off[0] = 0;
    for (int e = 0; e < m.num_experts; ++e) {
      for (size_t i = 0; i < m.hosts[e].size(); ++i) {
        if (o >= cap) return 3;
        hosts[o] = m.hosts[e][i];
        rid[o] = m.replica_ids[e][i];
        ++o;
      }
      off[e + 1] = o;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_load_batch_text(const char* text, int* T, int* k, int32_t* experts, int cap) {
  try {
    std::istringstream in(text);
    ActivationBatch b = load_batch(in);
    *T = b.num_tokens;
    *k = b.top_k;
    if (static_cast<int>(b.experts.size()) > cap) return 3;
    std::copy(b.experts.begin(), b.experts.end(), experts);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_dump_assignment(const int32_t* experts, int T, int k, int N, const int32_t* replica,
                        const int32_t* load, const long long* routed, char* buf, int cap,
                        int* len) {
  ActivationBatch b = make_batch(experts, T, k);
  Assignment a;
  a.replica.assign(replica, replica + static_cast<size_t>(T) * k);
  a.load.assign(load, load + N);
  a.routed_tokens.assign(routed, routed + N);
  std::ostringstream os;
  dump_assignment(os, a, b);
  std::string s = os.str();
  *len = static_cast<int>(s.size());
  if (*len + 1 > cap) return 3;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

// ActivationStats (experts.cpp:11-62): windowed per-expert counts and the
// co-activation matrix.  Opaque handle; status 1 = ValidationError (message
// in ref_last_error).
void* ref_stats_new(int E, int window) {
  try {
    return new ActivationStats(E, window);
  } catch (const std::exception& e) {
    fail(e, 1);
    return nullptr;
  }
}
void ref_stats_free(void* h) { delete static_cast<ActivationStats*>(h); }
int ref_stats_record(void* h, const int32_t* activated, int n) {
  try {
    static_cast<ActivationStats*>(h)->record_step(std::vector<int32_t>(activated, activated + n));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}
void ref_stats_read(void* h, long long* counts, long long* coact) {
  auto* s = static_cast<ActivationStats*>(h);
  const int E = s->num_experts();
  for (int i = 0; i < E; ++i) {
    counts[i] = s->count(i);
    for (int j = 0; j < E; ++j) coact[static_cast<size_t>(i) * E + j] = s->coactivation(i, j);
  }
}

}  // extern "C"
