// janus_moesim_compat.hpp — C++ drop-in for the reference moesim scheduling API
// (include/moesim/aebs.hpp:63-71 and latency.hpp:34-35 in /root/reference/proj;
// calibrated_moe_layer_latency for sim.cpp:193-195),
// implemented over the C ABI in janus_b200.h.  Header-only; link
// libjanus_b200.so.
//
// Two ways to use it:
//  * standalone: this header defines moesim::ActivationBatch / ReplicaMap /
//    Assignment / ValidationError with the reference's field names and
//    semantics, and moesim::schedule / schedule_reference / schedule_random.
//  * inside the reference build: define JANUS_USE_REFERENCE_TYPES and include
//    it after "moesim/aebs.hpp"; the functions are then provided as
//    janus::schedule(...) etc. on the reference's own types, so aebs.cpp's
//    bodies can forward to them without a name clash.
//
// Semantics kept: value-semantics outputs, ValidationError("unknown-expert:
// batch references expert X with no replica in the map") with X the minimum
// bad id (aebs.cpp:22-25,137-162), ReplicaMap::validate's messages on the map.
// Thread safety: one device context per thread (thread_local), so concurrent
// callers are independent, as the reference's pure function is
// (tests/test_aebs.cpp:182-192).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "janus_b200.h"

#ifndef JANUS_USE_REFERENCE_TYPES
namespace moesim {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct ActivationBatch {
  int num_tokens = 0;
  int top_k = 0;
  std::vector<int32_t> experts;
  int32_t at(int token, int j) const { return experts[static_cast<size_t>(token) * top_k + j]; }
  long long slots() const { return static_cast<long long>(num_tokens) * top_k; }
};

struct ReplicaMap {
  int num_experts = 0;
  int num_instances = 0;
  int slots_per_instance = 0;
  std::vector<std::vector<int32_t>> hosts;
  std::vector<std::vector<int32_t>> replica_ids;
  int replica_count(int e) const { return static_cast<int>(hosts[e].size()); }
};

struct Assignment {
  std::vector<int32_t> instance;
  std::vector<int32_t> replica;
  std::vector<int32_t> expert_instance;
  std::vector<int32_t> load;
  std::vector<long long> routed_tokens;
  int max_load() const {
    int m = 0;
    for (int32_t l : load) m = l > m ? l : m;
    return m;
  }
};

inline int max_activated_load(const Assignment& a) { return a.max_load(); }

}  // namespace moesim
#define JANUS_COMPAT_NS moesim
#else
#define JANUS_COMPAT_NS janus
#endif

namespace janus_detail {

struct Ctx {
  janus_ctx* ctx = nullptr;
  const void* map_key = nullptr;  // identity of the last uploaded map
  std::vector<int32_t> off, hosts, rid;
  Ctx() {
    if (janus_create(&ctx, 0) != JANUS_OK)
      throw std::runtime_error("janus: no CUDA device for the scheduler");
  }
  ~Ctx() { janus_destroy(ctx); }
};

inline Ctx& ctx() {
  thread_local Ctx c;
  return c;
}

// Upload the map when its contents changed (the reference re-pushes maps only
// on reconfiguration).
inline void sync_map(const moesim::ReplicaMap& m) {
  Ctx& c = ctx();
  std::vector<int32_t> off(m.num_experts + 1, 0), hosts, rid;
  for (int e = 0; e < m.num_experts; ++e) {
    off[e + 1] = off[e] + static_cast<int32_t>(m.hosts[e].size());
    hosts.insert(hosts.end(), m.hosts[e].begin(), m.hosts[e].end());
    if (m.replica_ids[e].size() != m.hosts[e].size())
      throw moesim::ValidationError("replica map: expert " + std::to_string(e) +
                                    " replica id list sized wrong");
    rid.insert(rid.end(), m.replica_ids[e].begin(), m.replica_ids[e].end());
  }
  if (c.map_key == &m && off == c.off && hosts == c.hosts && rid == c.rid) return;
  if (static_cast<int>(m.hosts.size()) != m.num_experts)
    throw moesim::ValidationError("replica map: per-expert tables sized wrong");
  janus_status st = janus_set_replica_map(c.ctx, m.num_experts, m.num_instances,
                                          m.slots_per_instance, off.data(), hosts.data(),
                                          rid.data());
  if (st == JANUS_EINVAL) throw moesim::ValidationError(janus_last_error(c.ctx));
  if (st != JANUS_OK) throw std::runtime_error(janus_last_error(c.ctx));
  c.map_key = &m;
  c.off.swap(off);
  c.hosts.swap(hosts);
  c.rid.swap(rid);
}

inline moesim::Assignment run(const moesim::ActivationBatch& b, const moesim::ReplicaMap& m,
                              int policy, uint64_t seed) {
  sync_map(m);
  Ctx& c = ctx();
  moesim::Assignment a;
  const size_t S = static_cast<size_t>(b.num_tokens) * b.top_k;
  a.instance.resize(S);
  a.replica.resize(S);
  a.expert_instance.resize(m.num_experts);
  a.load.resize(m.num_instances);
  std::vector<int64_t> routed(m.num_instances);
  janus_status st = janus_schedule(c.ctx, b.experts.data(), b.num_tokens, b.top_k, policy, seed,
                                   a.instance.data(), a.replica.data(), a.expert_instance.data(),
                                   a.load.data(), routed.data(), nullptr);
  if (st == JANUS_EUNKNOWN_EXPERT || st == JANUS_EINVAL)
    throw moesim::ValidationError(janus_last_error(c.ctx));
  if (st != JANUS_OK) throw std::runtime_error(janus_last_error(c.ctx));
  a.routed_tokens.assign(routed.begin(), routed.end());
  return a;
}

}  // namespace janus_detail

namespace JANUS_COMPAT_NS {

// aebs.hpp:63 — balanced scheduling pass, on the GPU.
inline moesim::Assignment schedule(const moesim::ActivationBatch& b, const moesim::ReplicaMap& m) {
  return janus_detail::run(b, m, JANUS_POLICY_AEBS, 0);
}
// aebs.hpp:65-67 — identical outputs by contract.
inline moesim::Assignment schedule_reference(const moesim::ActivationBatch& b,
                                             const moesim::ReplicaMap& m) {
  return janus_detail::run(b, m, JANUS_POLICY_AEBS, 0);
}
// aebs.hpp:69-71
inline moesim::Assignment schedule_random(const moesim::ActivationBatch& b,
                                          const moesim::ReplicaMap& m, uint64_t seed) {
  return janus_detail::run(b, m, JANUS_POLICY_RANDOM, seed);
}

// latency.hpp:34-35, calibrated to the measured layer (janus_latency_fit): the
// call DecodeEngine::eval_step makes (sim.cpp:193-195) with the reference's
// InstanceLoad {activated_experts, routed_tokens} (latency.hpp:28-31).
template <class InstanceLoadT>
inline double calibrated_moe_layer_latency(const std::vector<InstanceLoadT>& loads, int d_hidden,
                                           int d_expert, const janus_latency_model& model) {
  std::vector<int32_t> load(loads.size());
  std::vector<int64_t> routed(loads.size());
  for (size_t g = 0; g < loads.size(); ++g) {
    load[g] = static_cast<int32_t>(loads[g].activated_experts);
    routed[g] = static_cast<int64_t>(loads[g].routed_tokens);
  }
  return janus_latency_layer(&model, static_cast<int>(loads.size()), load.data(), routed.data(),
                             d_hidden, d_expert);
}

}  // namespace JANUS_COMPAT_NS

#undef JANUS_COMPAT_NS
