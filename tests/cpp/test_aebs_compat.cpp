// C++ parity test through the drop-in header: the reference's own scheduler
// tests (tests/test_aebs.cpp in /root/reference/proj) restated against
// moesim::schedule from include/janus_moesim_compat.hpp (GPU), checked against
// the CPU oracle (oracle/liboracle.so, C ABI).  Needs a GPU; run by
// tests/test_gpu_cpp.py.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "janus_moesim_compat.hpp"

extern "C" {
uint64_t or_splitmix64(uint64_t* state);
uint64_t or_derive_seed(uint64_t root, const char* label, uint64_t extra);
uint64_t or_next_below(uint64_t* state, uint64_t n);
int or_schedule(int policy, int bad_mode, uint64_t seed, const int32_t* experts, int T, int k,
                int E, int N, int C, const int32_t* off, const int32_t* hosts, const int32_t* rid,
                int32_t* instance, int32_t* replica, int32_t* expert_instance, int32_t* load,
                long long* routed, long long* expert_tokens, int32_t* bad);
}

using namespace moesim;

static int failures = 0, checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++checks;                                                              \
    if (!(cond)) {                                                         \
      ++failures;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)

static ReplicaMap map_from(int N, int slots, std::vector<std::vector<int32_t>> hosts) {
  ReplicaMap m;
  m.num_experts = static_cast<int>(hosts.size());
  m.num_instances = N;
  m.slots_per_instance = slots;
  m.hosts = std::move(hosts);
  m.replica_ids.assign(m.num_experts, {});
  std::vector<int32_t> next(N, 0);
  for (int e = 0; e < m.num_experts; ++e) {
    std::sort(m.hosts[e].begin(), m.hosts[e].end());
    for (int32_t g : m.hosts[e]) m.replica_ids[e].push_back(g * slots + next[g]++);
  }
  return m;
}

static ActivationBatch batch_from(int k, std::vector<int32_t> ex) {
  ActivationBatch b;
  b.top_k = k;
  b.num_tokens = static_cast<int>(ex.size()) / k;
  b.experts = std::move(ex);
  return b;
}

static Assignment oracle(const ActivationBatch& b, const ReplicaMap& m, int policy, uint64_t seed) {
  std::vector<int32_t> off(m.num_experts + 1, 0), hosts, rid;
  for (int e = 0; e < m.num_experts; ++e) {
    off[e + 1] = off[e] + static_cast<int32_t>(m.hosts[e].size());
    hosts.insert(hosts.end(), m.hosts[e].begin(), m.hosts[e].end());
    rid.insert(rid.end(), m.replica_ids[e].begin(), m.replica_ids[e].end());
  }
  Assignment a;
  a.instance.resize(b.experts.size());
  a.replica.resize(b.experts.size());
  a.expert_instance.resize(m.num_experts);
  a.load.resize(m.num_instances);
  a.routed_tokens.resize(m.num_instances);
  int32_t bad = 0;
  or_schedule(policy, 0, seed, b.experts.data(), b.num_tokens, b.top_k, m.num_experts,
              m.num_instances, m.slots_per_instance, off.data(), hosts.data(), rid.data(),
              a.instance.data(), a.replica.data(), a.expert_instance.data(), a.load.data(),
              a.routed_tokens.data(), nullptr, &bad);
  return a;
}

static bool same(const Assignment& a, const Assignment& b) {
  return a.instance == b.instance && a.replica == b.replica &&
         a.expert_instance == b.expert_instance && a.load == b.load &&
         a.routed_tokens == b.routed_tokens;
}

// tests/test_aebs.cpp:47-78 random_case
struct SmallCase {
  ReplicaMap map;
  ActivationBatch batch;
};
static SmallCase random_case(uint64_t seed) {
  uint64_t st = or_derive_seed(seed, "aebs/case", 0);
  int E = 2 + static_cast<int>(or_next_below(&st, 5));
  int N = 1 + static_cast<int>(or_next_below(&st, 3));
  int T = 1 + static_cast<int>(or_next_below(&st, 8));
  int k = 1 + static_cast<int>(or_next_below(&st, std::min(E, 3)));
  std::vector<std::vector<int32_t>> hosts(E);
  for (int e = 0; e < E; ++e) {
    int r = 1 + static_cast<int>(or_next_below(&st, N));
    std::vector<int32_t> all(N);
    for (int g = 0; g < N; ++g) all[g] = g;
    for (int i = 0; i < r; ++i) std::swap(all[i], all[i + or_next_below(&st, N - i)]);
    all.resize(r);
    hosts[e] = all;
  }
  SmallCase c;
  c.map = map_from(N, E + 2, std::move(hosts));
  std::vector<int32_t> ex;
  for (int t = 0; t < T; ++t) {
    std::vector<int32_t> all(E);
    for (int e = 0; e < E; ++e) all[e] = e;
    for (int j = 0; j < k; ++j) {
      std::swap(all[j], all[j + or_next_below(&st, E - j)]);
      ex.push_back(all[j]);
    }
  }
  c.batch = batch_from(k, std::move(ex));
  return c;
}

int main() {
  {  // worked two-instance example, test_aebs.cpp:83-103
    ReplicaMap m = map_from(2, 4, {{0}, {0, 1}, {1}, {0, 1}});
    ActivationBatch b = batch_from(2, {0, 1, 2, 1, 3, 0});
    Assignment a = schedule(b, m);
    CHECK(a.expert_instance[0] == 0);
    CHECK(a.expert_instance[2] == 1);
    CHECK(a.expert_instance[1] == 0);
    CHECK(a.expert_instance[3] == 1);
    CHECK(a.max_load() == 2);
    CHECK((a.load == std::vector<int32_t>{2, 2}));
    CHECK((a.routed_tokens == std::vector<long long>{4, 2}));
    for (int t = 0; t < b.num_tokens; ++t)
      for (int j = 0; j < b.top_k; ++j)
        CHECK(a.instance[t * b.top_k + j] == a.expert_instance[b.at(t, j)]);
  }
  {  // greedy max-load 2 where the optimum is 1, test_aebs.cpp:105-114
    ReplicaMap m = map_from(3, 3, {{0, 1, 2}, {0, 1}, {0, 1}});
    CHECK(schedule(batch_from(1, {0, 1, 2}), m).max_load() == 2);
  }
  {  // 300 seeded instances vs the oracle, test_aebs.cpp:116-145
    for (uint64_t s = 0; s < 300; ++s) {
      SmallCase c = random_case(s);
      Assignment fast = schedule(c.batch, c.map);
      Assignment ref = schedule_reference(c.batch, c.map);
      CHECK(same(fast, oracle(c.batch, c.map, 0, 0)));
      CHECK(same(fast, ref));
      CHECK(same(schedule_random(c.batch, c.map, s), oracle(c.batch, c.map, 1, s)));
      for (int t = 0; t < c.batch.num_tokens; ++t)
        for (int j = 0; j < c.batch.top_k; ++j) {
          int e = c.batch.at(t, j);
          int g = fast.instance[t * c.batch.top_k + j];
          auto it = std::find(c.map.hosts[e].begin(), c.map.hosts[e].end(), g);
          CHECK(it != c.map.hosts[e].end());
          CHECK(fast.replica[t * c.batch.top_k + j] ==
                c.map.replica_ids[e][it - c.map.hosts[e].begin()]);
        }
    }
  }
  {  // unknown expert, test_aebs.cpp:160-167
    ReplicaMap m = map_from(2, 2, {{0}, {1}});
    bool threw = false;
    try {
      schedule(batch_from(1, {0, 3}), m);
    } catch (const ValidationError& e) {
      threw = std::string(e.what()).find("unknown-expert") != std::string::npos;
    }
    CHECK(threw);
    threw = false;
    try {
      schedule_random(batch_from(1, {0, 3}), m, 1);
    } catch (const ValidationError&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // deterministic under concurrent invocation, test_aebs.cpp:182-192
    SmallCase c = random_case(123);
    Assignment base = schedule(c.batch, c.map);
    std::vector<Assignment> out(8);
    std::vector<std::thread> th;
    for (int w = 0; w < 4; ++w)
      th.emplace_back([&, w] {
        for (int i = w; i < 8; i += 4) out[i] = schedule(c.batch, c.map);
      });
    for (auto& t : th) t.join();
    for (const Assignment& a : out) CHECK(same(a, base));
  }
  {  // invalid map is rejected with the reference message (aebs.cpp:49-77)
    ReplicaMap m = map_from(2, 1, {{0, 1}, {0, 1}});
    bool threw = false;
    try {
      schedule(batch_from(1, {0}), m);
    } catch (const ValidationError& e) {
      threw = std::string(e.what()) == "replica map: instance 0 holds 2 replicas, capacity 1";
    }
    CHECK(threw);
  }
  std::printf("test_aebs_compat: %d checks, %d failures\n", checks, failures);
  return failures ? 1 : 0;
}
