// Drop-in check on the REFERENCE's own types: include/janus_moesim_compat.hpp
// with JANUS_USE_REFERENCE_TYPES, compiled against /root/reference/proj/include
// and linked with the reference library (oracle/_ref/libmoesim_ref.so) and
// libjanus_b200.so.  janus::schedule / schedule_random must equal
// moesim::schedule / schedule_reference / schedule_random field by field, and
// dump_assignment strings must be identical (acceptance.cpp C11 style), on the
// reference's own generators (gen_batch, placement pipeline).  Built where
// /root/reference exists; the binary travels to the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>

#include "moesim/aebs.hpp"
#include "moesim/experts.hpp"
#include "moesim/latency.hpp"
#include "moesim/workload.hpp"
#define JANUS_USE_REFERENCE_TYPES
#include "janus_moesim_compat.hpp"

using namespace moesim;

static int failures = 0, checks = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    ++checks;                                                     \
    if (!(cond)) {                                                \
      ++failures;                                                 \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

static bool same(const Assignment& a, const Assignment& b) {
  return a.instance == b.instance && a.replica == b.replica &&
         a.expert_instance == b.expert_instance && a.load == b.load &&
         a.routed_tokens == b.routed_tokens;
}

static std::string dump(const Assignment& a, const ActivationBatch& b) {
  std::ostringstream os;
  dump_assignment(os, a, b);
  return os.str();
}

// DecodeEngine::rebuild_placement recipe (src/sim.cpp:134-148)
static ReplicaMap placed_map(const RoutingPattern& pat, int E, int k, int N, int C, uint64_t seed) {
  ActivationStats stats(E, 256);
  std::vector<char> seen(E);
  for (int s = 0; s < 32; ++s) {
    ActivationBatch b = gen_batch(pat, 256, k, seed, derive_seed(seed, "warmup", s));
    std::fill(seen.begin(), seen.end(), 0);
    for (int32_t e : b.experts) seen[e] = 1;
    std::vector<int32_t> act;
    for (int e = 0; e < E; ++e)
      if (seen[e]) act.push_back(e);
    stats.record_step(act);
  }
  long long budget = std::min<long long>(static_cast<long long>(N) * C,
                                         static_cast<long long>(N) * E);
  Allocation alloc = cap_allocation(allocate_replicas(stats.counts(), static_cast<int>(budget)),
                                    stats.counts(), N);
  return to_replica_map(place_replicas(alloc, stats, N, C));
}

int main() {
  struct Cfg {
    int E, N, C;
    double zipf;
    uint64_t seed;
  } cfgs[] = {{64, 4, 20, 0, 0x5EED}, {128, 6, 27, 1.0, 0x235}, {256, 8, 40, 1.0, 0xD5},
              {256, 6, 54, 1.2, 0x5A}, {160, 8, 24, 0, 0xF12}};
  for (const Cfg& c : cfgs) {
    std::vector<double> w(c.E);
    for (int e = 0; e < c.E; ++e) w[e] = c.zipf > 0 ? 1.0 / std::pow(e + 1.0, c.zipf) : 1.0;
    RoutingPattern pat = c.zipf > 0 ? RoutingPattern::from_pmf(w)
                                    : RoutingPattern::gaussian(c.E, 0.15);
    ReplicaMap m = placed_map(pat, c.E, 8, c.N, c.C, c.seed);
    for (int T : {1, 16, 32, 128, 256, 512, 1024, 4096}) {
      ActivationBatch b = gen_batch(pat, T, 8, c.seed, T);
      Assignment ref = moesim::schedule(b, m);
      Assignment got = janus::schedule(b, m);
      CHECK(same(got, ref));
      CHECK(same(got, moesim::schedule_reference(b, m)));
      CHECK(dump(got, b) == dump(ref, b));
      CHECK(same(janus::schedule_random(b, m, T), moesim::schedule_random(b, m, T)));
    }
  }
  // error path: same exception type and message as schedule() (aebs.cpp:22-25)
  ReplicaMap small;
  small.num_experts = 2;
  small.num_instances = 2;
  small.slots_per_instance = 2;
  small.hosts = {{0}, {1}};
  small.replica_ids = {{0}, {2}};
  ActivationBatch bad;
  bad.num_tokens = 3;
  bad.top_k = 1;
  bad.experts = {0, 7, 5};
  std::string want, got;
  try {
    moesim::schedule(bad, small);
  } catch (const ValidationError& e) {
    want = e.what();
  }
  try {
    janus::schedule(bad, small);
  } catch (const ValidationError& e) {
    got = e.what();
  }
  CHECK(!want.empty() && want == got);
  // the latency model with the reference's accounting is moe_layer_latency
  // (latency.cpp:17-32) on the reference's own InstanceLoad / ModelSpec
  {
    ModelSpec ms;
    ms.hidden_dim = 4096;
    ms.expert_dim = 1536;
    HardwareSpec hw;
    std::vector<InstanceLoad> loads;
    for (int g = 0; g < 6; ++g) loads.push_back(InstanceLoad{g * 7 % 23, (long long)g * 1337});
    const janus_latency_model rm{hw.kernel_launch_overhead, hw.hbm_bandwidth, hw.peak_flops, 0.0,
                                 2, ms.bytes_per_param, 1};
    CHECK(janus::calibrated_moe_layer_latency(loads, ms.hidden_dim, ms.expert_dim, rm) ==
          moe_layer_latency(loads, ms, hw));
  }
  std::printf("test_dropin: %d checks, %d failures\n", checks, failures);
  return failures ? 1 : 0;
}
