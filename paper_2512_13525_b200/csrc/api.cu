// api.cu — the C ABI (include/janus_b200.h): context, replica-map upload and
// validation, scheduling, MoE layer orchestration.  Host code only; kernels
// live in aebs.cu / ffn.cu.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "sm100.cuh"

using janus::DevMap;

namespace {

janus_status fail(janus_ctx *c, janus_status st, const std::string &msg) {
  if (c) c->err = msg;
  return st;
}

janus_status cuda_fail(janus_ctx *c, cudaError_t e, const char *where) {
  return fail(c, JANUS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                        \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call); \
  } while (0)

template <typename T>
cudaError_t dalloc(T **p, size_t n) {
  return cudaMalloc(reinterpret_cast<void **>(p), std::max<size_t>(n, 1) * sizeof(T));
}

void dfree(void *p) {
  if (p) cudaFree(p);
}

void free_map(DevMap &m) {
  dfree(m.blob);  // every table lives in the one allocation
  m = DevMap{};
}

// Internal assignments live in ONE allocation (few pages / TLB entries for
// the scheduler's output stores); `instance` is its base.
void free_assign(janus_assignment &a) {
  dfree(a.instance);
  a = janus_assignment{};
}

// Allocated zeroed: a layer call that fails before K1 writes them (or a
// reconfigured context) never reads recycled bytes.
cudaError_t alloc_assign(janus_assignment &a, int S, int E, int N, int R) {
  S = std::max(S, 1);
  size_t o = 0;
  auto take = [&o](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 255) & ~size_t(255);
    return at;
  };
  const size_t o_inst = take(4 * (size_t)S), o_rep = take(4 * (size_t)S),
               o_ei = take(4 * (size_t)E), o_load = take(4 * (size_t)N),
               o_routed = take(8 * (size_t)N), o_et = take(8 * (size_t)E),
               o_sr = take(4 * (size_t)S), o_rs = take(4 * (size_t)S),
               o_go = take(4 * (size_t)(R + 1)), o_st = take(8);
  unsigned char *d = nullptr;
  cudaError_t e = cudaMalloc(&d, o);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemset(d, 0, o)) != cudaSuccess) {
    cudaFree(d);
    return e;
  }
  a.instance = reinterpret_cast<int32_t *>(d + o_inst);
  a.replica = reinterpret_cast<int32_t *>(d + o_rep);
  a.expert_instance = reinterpret_cast<int32_t *>(d + o_ei);
  a.load = reinterpret_cast<int32_t *>(d + o_load);
  a.routed_tokens = reinterpret_cast<int64_t *>(d + o_routed);
  a.expert_tokens = reinterpret_cast<int64_t *>(d + o_et);
  a.slot_row = reinterpret_cast<int32_t *>(d + o_sr);
  a.row_slot = reinterpret_cast<int32_t *>(d + o_rs);
  a.group_off = reinterpret_cast<int32_t *>(d + o_go);
  a.status = reinterpret_cast<int32_t *>(d + o_st);
  return cudaSuccess;
}

// --- rng (include/moesim/rng.hpp:13-44), used for schedule_random seeds and
// the synthetic workload generator.
uint64_t splitmix64(uint64_t &s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t hash_label(const char *label) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const unsigned char *p = reinterpret_cast<const unsigned char *>(label); *p; ++p) {
    h ^= *p;
    h *= 0x100000001b3ULL;
  }
  return h;
}

// Captured layer graphs bake in buffers and tensor maps: drop them whenever
// the map, the workspace or the weight store changes.
void clear_graphs(janus_ctx *ctx) {
  for (auto &g : ctx->graphs) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
}

janus_status check_ready(janus_ctx *ctx) {
  if (!ctx) return JANUS_EINVAL;
  if (!ctx->have_map) return fail(ctx, JANUS_ESTATE, "janus: no replica map set");
  return JANUS_OK;
}

}  // namespace

extern "C" {

uint64_t janus_derive_seed(uint64_t root, const char *label, uint64_t extra) {
  uint64_t s = root;
  splitmix64(s);
  s ^= hash_label(label);
  splitmix64(s);
  uint64_t e = extra;
  s ^= splitmix64(e);
  return splitmix64(s);
}

janus_status janus_create(janus_ctx **out, int device) {
  if (!out) return JANUS_EINVAL;
  *out = nullptr;
  janus_ctx *ctx = new janus_ctx();
  ctx->device = device;
  const char *g = std::getenv("JANUS_GRAPH");
  ctx->use_graph = !(g && g[0] == '0');
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return JANUS_ECUDA;
  }
  *out = ctx;
  return JANUS_OK;
}

static void free_stats(janus::StatsState &st);
static void free_host_pipe(janus_ctx *ctx);
static void free_shared(janus_ctx *ctx);

void janus_destroy(janus_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  {  // the exchange's own streams (partial-sum push, copy-engine dispatch)
    janus::XferState &x = ctx->xfer;
    if (x.push_stream) {
      cudaStreamSynchronize(x.push_stream);
      cudaStreamDestroy(x.push_stream);
      x.push_stream = nullptr;
    }
    for (int i = 0; i < 2; ++i) {
      if (x.ffn_done[i]) cudaEventDestroy(x.ffn_done[i]);
      if (x.push_done[i]) cudaEventDestroy(x.push_done[i]);
      x.ffn_done[i] = x.push_done[i] = nullptr;
    }
    for (int i = 0; i < janus::kXferSlots; ++i) {
      if (x.own_disp[i]) cudaEventDestroy(x.own_disp[i]);
      if (x.own_sig[i]) cudaEventDestroy(x.own_sig[i]);
      if (x.comb_done[i]) cudaEventDestroy(x.comb_done[i]);
      x.own_disp[i] = x.own_sig[i] = x.comb_done[i] = nullptr;
    }
    for (cudaStream_t st : x.ce_streams) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
    x.ce_streams.clear();
    for (cudaEvent_t ev : x.ce_done) cudaEventDestroy(ev);
    x.ce_done.clear();
    if (x.ce_fork) cudaEventDestroy(x.ce_fork);
    x.ce_fork = nullptr;
  }
  free_map(ctx->dmap);
  dfree(ctx->d_in);
  free_assign(ctx->d_out);
  free_assign(ctx->ws);
  dfree(ctx->ws_tile_off);
  dfree(ctx->ffn.xp);
  dfree(ctx->ffn.h);
  dfree(ctx->ffn.y);
  dfree(ctx->ffn.y2);
  dfree(ctx->ffn.tile_ctr);
  dfree(ctx->gate_xchg);
  dfree(ctx->d_x);
  dfree(ctx->d_outbuf);
  dfree(ctx->d_experts);
  dfree(ctx->d_gw);
  for (cudaEvent_t e : ctx->prof_events) cudaEventDestroy(e);
  for (auto &g : ctx->graphs) cudaGraphExecDestroy(g.exec);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  janus::mc_free(ctx->xfer, ctx->device);
  free_stats(ctx->stats);
  free_host_pipe(ctx);
  free_shared(ctx);
  for (void *p : ctx->xfer.opened) cudaIpcCloseMemHandle(p);
  dfree(ctx->xfer.local);
  dfree(ctx->xfer.counter);
  dfree(ctx->xfer.err);
  free_assign(ctx->xfer.rws);
  dfree(ctx->xfer.dmask);
  for (int i = 0; i < janus::kXferSlots; ++i) {
    free_assign(ctx->xfer.lay[i]);
    dfree(ctx->xfer.lay_tile[i]);
  }
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char *janus_last_error(const janus_ctx *ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

uint64_t janus_launch_count(const janus_ctx *ctx) { return ctx ? ctx->launches : 0; }

// ReplicaMap::validate, src/aebs.cpp:49-77 (same messages).
janus_status janus_set_replica_map(janus_ctx *ctx, int E, int N, int C, const int32_t *off,
                                   const int32_t *hosts, const int32_t *rid) {
  if (!ctx) return JANUS_EINVAL;
  if (E <= 0 || N <= 0 || C <= 0)
    return fail(ctx, JANUS_EINVAL, "replica map: dimensions must be positive");
  if (!off || !hosts || !rid || off[0] != 0)
    return fail(ctx, JANUS_EINVAL, "replica map: per-expert tables sized wrong");
  std::vector<int> used(N, 0);
  for (int e = 0; e < E; ++e) {
    if (off[e + 1] <= off[e])
      return fail(ctx, JANUS_EINVAL,
                  "replica map: expert " + std::to_string(e) + " has no replica");
    for (int i = off[e]; i < off[e + 1]; ++i) {
      const int g = hosts[i];
      if (g < 0 || g >= N)
        return fail(ctx, JANUS_EINVAL,
                    "replica map: expert " + std::to_string(e) + " hosted on invalid instance " +
                        std::to_string(g));
      if (i > off[e] && hosts[i - 1] >= g)
        return fail(ctx, JANUS_EINVAL,
                    "replica map: expert " + std::to_string(e) +
                        " host list not strictly ascending");
      ++used[g];
    }
  }
  for (int g = 0; g < N; ++g)
    if (used[g] > C)
      return fail(ctx, JANUS_EINVAL,
                  "replica map: instance " + std::to_string(g) + " holds " +
                      std::to_string(used[g]) + " replicas, capacity " + std::to_string(C));
  const int R = off[E];
  if (E > JANUS_MAX_EXPERTS || N > JANUS_MAX_INSTANCES || R > JANUS_MAX_REPLICAS ||
      janus::schedule_smem_bytes(E, N, R) > 227 * 1024 - 1024)
    return fail(ctx, JANUS_EUNSUPPORTED, "replica map: exceeds kernel limits of this build");

  ctx->off.assign(off, off + E + 1);
  ctx->hosts.assign(hosts, hosts + R);
  ctx->rid.assign(rid, rid + R);
  // Replica order: per instance, sorted by (replica id, expert).
  std::vector<int32_t> expert_of(R);
  for (int e = 0; e < E; ++e)
    for (int p = off[e]; p < off[e + 1]; ++p) expert_of[p] = e;
  std::vector<int> order(R);
  for (int p = 0; p < R; ++p) order[p] = p;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (hosts[a] != hosts[b]) return hosts[a] < hosts[b];
    if (rid[a] != rid[b]) return rid[a] < rid[b];
    return expert_of[a] < expert_of[b];
  });
  ctx->qidx.assign(R, 0);
  ctx->qbase.assign(N + 1, 0);
  for (int i = 0; i < R; ++i) {
    ctx->qidx[order[i]] = i;
    ctx->qbase[hosts[order[i]] + 1]++;
  }
  for (int g = 0; g < N; ++g) ctx->qbase[g + 1] += ctx->qbase[g];
  std::vector<uint32_t> hm(E, 0);
  if (N <= 32)
    for (int e = 0; e < E; ++e)
      for (int p = off[e]; p < off[e + 1]; ++p) hm[e] |= 1u << hosts[p];

  CK(cudaSetDevice(ctx->device));
  free_map(ctx->dmap);
  DevMap &m = ctx->dmap;
  // Every map table in ONE allocation (a few KB: one page, one TLB entry for
  // the scheduler's whole map read), uploaded with one copy.
  const int W = (E + 31) / 32;
  const bool small = N <= 32, pairs = N <= 8 && C <= 255;
  std::vector<unsigned char> blob;
  auto put = [&blob](const void *src, size_t bytes) {
    const size_t at = (blob.size() + 15) & ~size_t(15);
    blob.resize(at + std::max<size_t>(bytes, 16));
    if (bytes) std::memcpy(blob.data() + at, src, bytes);
    return at;
  };
  const size_t o_off = put(off, sizeof(int32_t) * (E + 1));
  const size_t o_hosts = put(hosts, sizeof(int32_t) * R);
  const size_t o_rid = put(rid, sizeof(int32_t) * R);
  const size_t o_qidx = put(ctx->qidx.data(), sizeof(int32_t) * R);
  const size_t o_hm = put(hm.data(), sizeof(uint32_t) * E);
  size_t o_exi = 0, o_rpi = 0, o_multi = 0, o_pin = 0, o_hmk = 0, o_qb = 0, o_pi = 0, o_pbh = 0;
  if (small) {  // the single-CTA decode scheduler's tables (aebs.cu)
    std::vector<int4> exi(E);
    std::vector<int2> rpi(R);
    std::vector<uint32_t> multi(W, 0), pin((size_t)N * W, 0), hmk((size_t)N * W, 0);
    for (int e = 0; e < E; ++e) {
      const int r = off[e + 1] - off[e];
      exi[e] = make_int4(off[e], r, (int)hm[e], hosts[off[e]]);
      if (r > 1) {
        multi[e >> 5] |= 1u << (e & 31);
        for (int p = off[e]; p < off[e + 1]; ++p)
          hmk[(size_t)hosts[p] * W + (e >> 5)] |= 1u << (e & 31);
      } else {
        pin[(size_t)hosts[off[e]] * W + (e >> 5)] |= 1u << (e & 31);
      }
    }
    for (int p = 0; p < R; ++p) rpi[p] = make_int2(rid[p], ctx->qidx[p]);
    o_exi = put(exi.data(), sizeof(int4) * E);
    o_rpi = put(rpi.data(), sizeof(int2) * R);
    o_multi = put(multi.data(), sizeof(uint32_t) * W);
    o_pin = put(pin.data(), sizeof(uint32_t) * N * W);
    o_hmk = put(hmk.data(), sizeof(uint32_t) * N * W);
    o_qb = put(ctx->qbase.data(), sizeof(int32_t) * (N + 1));
    if (pairs) {
      std::vector<uint4> pi(E, make_uint4(0, 0, 0, 0));
      std::vector<uint32_t> pbh(E, 0);
      auto inc = [](uint32_t g, bool want_hi) -> uint32_t {
        return (g >= 4) == want_hi ? 1u << (8 * (g & 3)) : 0u;
      };
      for (int e = 0; e < E; ++e) {
        const int r = off[e + 1] - off[e];
        if (r == 2) {
          const uint32_t ga = hosts[off[e]], gb = hosts[off[e] + 1];
          pi[e] = make_uint4(ga << 12 | gb << 28, inc(ga, false), inc(ga, true), inc(gb, false));
          pbh[e] = inc(gb, true);
        } else if (r > 2) {
          pi[e] = make_uint4(0xffffffffu, hm[e], 0, 0);
        }
      }
      m.pairs_only = 1;
      for (int e = 0; e < E; ++e)
        if (off[e + 1] - off[e] > 2) m.pairs_only = 0;
      o_pi = put(pi.data(), sizeof(uint4) * E);
      o_pbh = put(pbh.data(), sizeof(uint32_t) * E);
    }
  }
  unsigned char *d = nullptr;
  CK(cudaMalloc(&d, blob.size()));
  m.blob = d;
  CK(cudaMemcpy(d, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  m.off = reinterpret_cast<int32_t *>(d + o_off);
  m.hosts = reinterpret_cast<int32_t *>(d + o_hosts);
  m.rid = reinterpret_cast<int32_t *>(d + o_rid);
  m.qidx = reinterpret_cast<int32_t *>(d + o_qidx);
  m.hmask = reinterpret_cast<uint32_t *>(d + o_hm);
  if (small) {
    m.ex_info = reinterpret_cast<int4 *>(d + o_exi);
    m.rep_info = reinterpret_cast<int2 *>(d + o_rpi);
    m.multi_mask = reinterpret_cast<uint32_t *>(d + o_multi);
    m.pin_mask = reinterpret_cast<uint32_t *>(d + o_pin);
    m.host_mask = reinterpret_cast<uint32_t *>(d + o_hmk);
    m.qbase = reinterpret_cast<int32_t *>(d + o_qb);
    if (pairs) {
      m.pair_info = reinterpret_cast<uint4 *>(d + o_pi);
      m.pair_bhi = reinterpret_cast<uint32_t *>(d + o_pbh);
    }
  }
  m.E = E;
  m.N = N;
  m.C = C;
  m.R = R;
  ctx->have_map = true;
  clear_graphs(ctx);
  // a new map invalidates the layer's weight store
  ctx->moe_ready = false;
  ctx->ffn.w13 = ctx->ffn.w2 = nullptr;
  return JANUS_OK;
}

janus_status janus_replica_order(const janus_ctx *ctx, int32_t *qidx, int32_t *qbase) {
  if (!ctx || !ctx->have_map) return JANUS_ESTATE;
  std::copy(ctx->qidx.begin(), ctx->qidx.end(), qidx);
  std::copy(ctx->qbase.begin(), ctx->qbase.end(), qbase);
  return JANUS_OK;
}

static janus_status launch_sched(janus_ctx *ctx, const int32_t *d_experts, int T, int k,
                                 int policy, uint64_t seed, const janus_assignment &out,
                                 int32_t *tile_off, cudaStream_t stream,
                                 int32_t *shared_off = nullptr, int shared_tile_n = 0,
                                 int shared_rows = 0, const int *abort_flag = nullptr) {
  if (T < 0 || k <= 0 || (int64_t)T * k > (int64_t)1 << 30)
    return fail(ctx, JANUS_EINVAL, "batch: num_tokens must be >= 0 and top_k >= 1");
  if (policy != JANUS_POLICY_AEBS && policy != JANUS_POLICY_RANDOM)
    return fail(ctx, JANUS_EINVAL, "schedule: unknown policy");
  if (!out.instance || !out.replica || !out.expert_instance || !out.load || !out.routed_tokens ||
      !out.status || (T > 0 && !d_experts))
    return fail(ctx, JANUS_EINVAL, "schedule: missing output buffer");
  janus::SchedArgs a{};
  a.experts = d_experts;
  a.S = T * k;
  a.k = k;
  a.map = ctx->dmap;
  a.id_bits = janus::id_bits_for(ctx->dmap.E);
  a.policy = policy;
  a.rng_state = janus_derive_seed(seed, "sched/random", 0);
  a.out = out;
  a.tile_off = tile_off;
  a.tile_n = ctx->ffn.tile_n > 0 ? ctx->ffn.tile_n : janus::kTileN;
  // decode tiles are weight-streaming bound: fold each group's remainder into
  // its last tile (one pass over the weights); in the tensor regime the wide
  // tile's halved weight prefetch depth costs more than it saves (measured)
  a.merge_tail = a.tile_n <= 64;
  a.shared_off = shared_off;
  a.shared_tile_n = shared_tile_n;
  a.shared_rows = shared_rows;
  a.abort_flag = abort_flag;
  cudaError_t e = janus::launch_schedule(a, stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "aebs_schedule_kernel");
  ctx->launches += 1;
  return JANUS_OK;
}

janus_status janus_schedule_async(janus_ctx *ctx, const int32_t *d_experts, int T, int k,
                                  int policy, uint64_t seed, const janus_assignment *out,
                                  void *stream) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (!out) return fail(ctx, JANUS_EINVAL, "schedule: null output");
  return launch_sched(ctx, d_experts, T, k, policy, seed, *out, nullptr,
                      static_cast<cudaStream_t>(stream));
}

static janus_status grow_sched(janus_ctx *ctx, int S) {
  if (S <= ctx->sched_cap && ctx->d_in) return JANUS_OK;
  const int cap = std::max(S, 1024);
  dfree(ctx->d_in);
  free_assign(ctx->d_out);
  ctx->d_in = nullptr;
  CK(dalloc(&ctx->d_in, cap));
  CK(alloc_assign(ctx->d_out, cap, JANUS_MAX_EXPERTS, JANUS_MAX_INSTANCES,
                  JANUS_MAX_REPLICAS));
  ctx->sched_cap = cap;
  return JANUS_OK;
}

janus_status janus_schedule(janus_ctx *ctx, const int32_t *experts, int T, int k, int policy,
                            uint64_t seed, int32_t *instance, int32_t *replica,
                            int32_t *expert_instance, int32_t *load, int64_t *routed_tokens,
                            int64_t *expert_tokens) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (T < 0 || k <= 0) return fail(ctx, JANUS_EINVAL, "batch: num_tokens must be >= 0 and top_k >= 1");
  CK(cudaSetDevice(ctx->device));
  const int S = T * k;
  st = grow_sched(ctx, S);
  if (st != JANUS_OK) return st;
  cudaStream_t s = ctx->stream;
  if (S) CK(cudaMemcpyAsync(ctx->d_in, experts, sizeof(int32_t) * S, cudaMemcpyHostToDevice, s));
  st = launch_sched(ctx, ctx->d_in, T, k, policy, seed, ctx->d_out, nullptr, s);
  if (st != JANUS_OK) return st;
  int32_t status[2];
  CK(cudaMemcpyAsync(status, ctx->d_out.status, sizeof(status), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (status[0] == JANUS_EUNKNOWN_EXPERT)
    return fail(ctx, JANUS_EUNKNOWN_EXPERT,
                "unknown-expert: batch references expert " + std::to_string(status[1]) +
                    " with no replica in the map");
  const DevMap &m = ctx->dmap;
  if (S) {
    CK(cudaMemcpyAsync(instance, ctx->d_out.instance, sizeof(int32_t) * S,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(replica, ctx->d_out.replica, sizeof(int32_t) * S, cudaMemcpyDeviceToHost,
                       s));
  }
  CK(cudaMemcpyAsync(expert_instance, ctx->d_out.expert_instance, sizeof(int32_t) * m.E,
                     cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(load, ctx->d_out.load, sizeof(int32_t) * m.N, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(routed_tokens, ctx->d_out.routed_tokens, sizeof(int64_t) * m.N,
                     cudaMemcpyDeviceToHost, s));
  if (expert_tokens)
    CK(cudaMemcpyAsync(expert_tokens, ctx->d_out.expert_tokens, sizeof(int64_t) * m.E,
                       cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return JANUS_OK;
}

janus_status janus_time_schedule(janus_ctx *ctx, const int32_t *d_experts, int T, int k,
                                 int policy, int reps, double *median_us) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  CK(cudaSetDevice(ctx->device));
  st = grow_sched(ctx, T * k);
  if (st != JANUS_OK) return st;
  cudaStream_t s = ctx->stream;
  constexpr int kPerGraph = 20;
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < kPerGraph; ++i) {
    st = launch_sched(ctx, d_experts, T, k, policy, 1, ctx->d_out, nullptr, s);
    if (st != JANUS_OK) {
      cudaStreamEndCapture(s, &graph);
      return st;
    }
  }
  CK(cudaStreamEndCapture(s, &graph));
  CK(cudaGraphInstantiate(&exec, graph, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(exec, s));
  std::vector<float> t(std::max(reps, 1));
  for (auto &x : t) {
    CK(cudaEventRecord(e0, s));
    CK(cudaGraphLaunch(exec, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&x, e0, e1));
  }
  ctx->launches += (uint64_t)kPerGraph * (t.size() + 3);
  std::nth_element(t.begin(), t.begin() + t.size() / 2, t.end());
  *median_us = 1000.0 * t[t.size() / 2] / kPerGraph;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  return JANUS_OK;
}

// ---------------------------------------------------------------- MoE -----

janus_status janus_moe_configure(janus_ctx *ctx, int d_h, int d_e, int max_tokens, int k) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (d_h <= 0 || d_e <= 0 || d_h % 256 || d_e % 128 || max_tokens <= 0 || k <= 0)
    return fail(ctx, JANUS_EUNSUPPORTED,
                "moe: need d_hidden % 256 == 0, d_expert % 128 == 0, max_tokens, top_k > 0");
  CK(cudaSetDevice(ctx->device));
  const int S = max_tokens * k;
  const int S_alloc = S + janus::kTileN;  // tail room for the last token box
  dfree(ctx->ffn.xp);
  dfree(ctx->ffn.h);
  dfree(ctx->ffn.y);
  dfree(ctx->ffn.y2);
  ctx->ffn.y2 = nullptr;
  dfree(ctx->ffn.tile_ctr);
  ctx->ffn.tile_ctr = nullptr;
  free_host_pipe(ctx);  // staging sized by max_tokens
  free_shared(ctx);
  free_assign(ctx->ws);
  dfree(ctx->ws_tile_off);
  dfree(ctx->d_x);
  dfree(ctx->d_outbuf);
  dfree(ctx->d_experts);
  dfree(ctx->d_gw);
  ctx->ffn.xp = ctx->ffn.h = ctx->ffn.y = nullptr;
  ctx->ws_tile_off = nullptr;
  ctx->d_x = ctx->d_outbuf = nullptr;
  ctx->d_experts = nullptr;
  ctx->d_gw = nullptr;
  const DevMap &m = ctx->dmap;
  CK(cudaMalloc(&ctx->ffn.xp, (size_t)S_alloc * d_h * 2));
  CK(cudaMalloc(&ctx->ffn.h, (size_t)S_alloc * d_e * 2));
  CK(cudaMalloc(&ctx->ffn.y, (size_t)S_alloc * d_h * 2));
  CK(cudaMemset(ctx->ffn.xp, 0, (size_t)S_alloc * d_h * 2));
  CK(cudaMemset(ctx->ffn.h, 0, (size_t)S_alloc * d_e * 2));
  CK(dalloc(&ctx->ffn.tile_ctr, 4));
  CK(cudaMemset(ctx->ffn.tile_ctr, 0, 4 * sizeof(unsigned)));
  // per-map arrays at the build's limits: a later janus_set_replica_map
  // (reconfiguration) may grow E / N / R without a reconfigure
  (void)m;
  CK(alloc_assign(ctx->ws, S, JANUS_MAX_EXPERTS, JANUS_MAX_INSTANCES, JANUS_MAX_REPLICAS));
  CK(dalloc(&ctx->ws_tile_off, JANUS_MAX_REPLICAS + 1));
  CK(cudaMemset(ctx->ws_tile_off, 0, sizeof(int32_t) * (JANUS_MAX_REPLICAS + 1)));
  CK(cudaMalloc(&ctx->d_x, (size_t)max_tokens * d_h * 2));
  CK(cudaMalloc(&ctx->d_outbuf, (size_t)max_tokens * d_h * 2));
  CK(dalloc(&ctx->d_experts, S));
  CK(dalloc(&ctx->d_gw, S));
  ctx->d_h = d_h;
  ctx->d_e = d_e;
  ctx->max_tokens = max_tokens;
  ctx->top_k = k;
  ctx->ffn.d_h = d_h;
  ctx->ffn.d_e = d_e;
  ctx->ffn.S_alloc = S_alloc;
  ctx->moe_ready = false;
  clear_graphs(ctx);
  return JANUS_OK;
}

static void free_shared(janus_ctx *ctx) {
  janus::FfnPlan &ps = ctx->ffn_shared;
  dfree(ps.xp);
  dfree(ps.h);
  dfree(ps.y);
  dfree(ps.tile_ctr);
  dfree(ctx->shared_off);
  ctx->shared_off = nullptr;
  ps = janus::FfnPlan{};
  ctx->shared = false;
}

janus_status janus_moe_set_shared(janus_ctx *ctx, const void *w13, const void *w2) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (!ctx->ffn.h) return fail(ctx, JANUS_ESTATE, "moe: janus_moe_configure first");
  CK(cudaSetDevice(ctx->device));
  clear_graphs(ctx);
  if (!w13 || !w2) {  // disable
    free_shared(ctx);
    return JANUS_OK;
  }
  janus::FfnPlan &ps = ctx->ffn_shared;
  if (!ps.xp) {
    const int rows = ctx->max_tokens + janus::kTileN;  // tail room for the last token box
    ps.d_h = ctx->d_h;
    ps.d_e = ctx->d_e;
    ps.S_alloc = rows;
    CK(cudaMalloc(&ps.xp, (size_t)rows * ps.d_h * 2));
    CK(cudaMalloc(&ps.h, (size_t)rows * ps.d_e * 2));
    CK(cudaMalloc(&ps.y, (size_t)rows * ps.d_h * 2));
    CK(cudaMemset(ps.xp, 0, (size_t)rows * ps.d_h * 2));
    CK(cudaMemset(ps.h, 0, (size_t)rows * ps.d_e * 2));
    CK(dalloc(&ps.tile_ctr, 4));
    CK(cudaMemset(ps.tile_ctr, 0, 4 * sizeof(unsigned)));
    CK(dalloc(&ctx->shared_off, 4));
    CK(cudaMemset(ctx->shared_off, 0, 4 * sizeof(int32_t)));
  }
  ps.q_begin = 0;
  ps.q_end = 1;
  ps.w13 = w13;
  ps.w2 = w2;
  CK(janus::build_ffn_tensor_maps(ps));
  ctx->shared = true;
  return JANUS_OK;
}

janus_status janus_moe_set_shared_split(janus_ctx *ctx, int split) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (split != 0 && split != 1) return fail(ctx, JANUS_EINVAL, "moe: shared split must be 0 or 1");
  clear_graphs(ctx);
  ctx->shared_split = split;
  return JANUS_OK;
}

janus_status janus_moe_set_weights(janus_ctx *ctx, int instance, const void *w13, const void *w2) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (!ctx->ffn.h) return fail(ctx, JANUS_ESTATE, "moe: janus_moe_configure first");
  if (!w13 || !w2 || instance >= ctx->dmap.N)
    return fail(ctx, JANUS_EINVAL, "moe: bad weight store");
  CK(cudaSetDevice(ctx->device));
  ctx->instance = instance;
  ctx->ffn.q_begin = instance < 0 ? 0 : ctx->qbase[instance];
  ctx->ffn.q_end = instance < 0 ? ctx->dmap.R : ctx->qbase[instance + 1];
  ctx->ffn.w13 = w13;
  ctx->ffn.w2 = w2;
  CK(janus::build_ffn_tensor_maps(ctx->ffn));
  ctx->moe_ready = true;
  clear_graphs(ctx);
  return JANUS_OK;
}

}  // extern "C"

// The layer body shared by the single-GPU entry point and the MoE rank of the
// box exchange: K1 schedule -> K3 permute -> K4 GEMMs -> K5 combine, where
// the combine either writes `d_out` locally or (push_epoch != 0) pushes this
// instance's partial sums into the owning attention ranks' memory.
// GEMM n-tile: decode steps (few rows per replica group) use 64-row tiles
// and the deep 9-stage weight ring; larger steps 256-row tiles.
// Crossover measured on the c2 shape (FFN µs, 64 vs 256-row tiles): 24 rows
// per expert 194.5 vs 196.0, 32: 204.2 vs 200.9, 48: 218.5 vs 209.2.
static int layer_tile_n(const janus_ctx *ctx, int T) {
  return (int64_t)T * ctx->top_k <= 28LL * ctx->dmap.E ? 64 : janus::kTileN;
}

// pre / pre_tile (optional): this step's layout, computed earlier by the same
// context's attention role (colocated routed box) — K1 is then not rerun.
// Blocks (4 warps each) of the side-stream partial-sum push: enough warps in
// flight for its gather latency without flooding the SMs beside the next
// step's GEMMs.  Measured (4-GPU box, tok/s/GPU): 1 x SMs 7.1 M, 2 x 8.9 M,
// 3 x 9.4 M, 4 x 9.7-9.8 M, 5 x 9.6 M, 6 x 9.3 M, uncapped 9.1 M.
static int push_blocks() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // JANUS_PUSH_BLOCKS: tuning override of the measured default
  static const int over = getenv("JANUS_PUSH_BLOCKS") ? atoi(getenv("JANUS_PUSH_BLOCKS")) : 0;
  return over > 0 ? over : 4 * sms;
}

static janus_status layer_run(janus_ctx *ctx, const void *d_x, const int32_t *d_experts,
                              const float *d_gate_w, int T, void *d_out,
                              const janus_assignment *assign, cudaStream_t s,
                              unsigned long long push_epoch, const int *abort_flag = nullptr,
                              const janus_assignment *pre = nullptr,
                              int32_t *pre_tile = nullptr) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (!ctx->moe_ready) return fail(ctx, JANUS_ESTATE, "moe: weights not set");
  if (T < 0 || T > ctx->max_tokens)
    return fail(ctx, JANUS_EINVAL, "moe: num_tokens outside [0, max_tokens]");
  const int k = ctx->top_k;
  janus_assignment a = ctx->ws;
  a.row_slot = nullptr;  // the inverse permutation is not needed by the layer
  if (assign) {  // caller wants the scheduling outputs: write into its buffers
    a.instance = assign->instance ? assign->instance : a.instance;
    a.replica = assign->replica ? assign->replica : a.replica;
    a.expert_instance = assign->expert_instance ? assign->expert_instance : a.expert_instance;
    a.load = assign->load ? assign->load : a.load;
    a.routed_tokens = assign->routed_tokens ? assign->routed_tokens : a.routed_tokens;
    a.expert_tokens = assign->expert_tokens ? assign->expert_tokens : a.expert_tokens;
    a.slot_row = assign->slot_row ? assign->slot_row : a.slot_row;
    a.row_slot = assign->row_slot;  // opt-in: the layer permutes slot-major
    a.group_off = assign->group_off ? assign->group_off : a.group_off;
    a.status = assign->status ? assign->status : a.status;
  }
  ctx->ffn.tile_n = layer_tile_n(ctx, T);
  if (pre) {
    a = *pre;
    a.row_slot = nullptr;
  }
  int32_t *tile_off = pre ? pre_tile : ctx->ws_tile_off;
  cudaEvent_t *ev = nullptr;
  if (ctx->profiling) {
    const size_t need = 4 * (size_t)(ctx->prof_calls + 1);
    while (ctx->prof_events.size() < need) {
      cudaEvent_t x;
      CK(cudaEventCreate(&x));
      ctx->prof_events.push_back(x);
    }
    ev = &ctx->prof_events[4 * (size_t)ctx->prof_calls];
    ctx->prof_calls++;
    CK(cudaEventRecord(ev[0], s));
  }
  janus::sm100::pdl_enabled = ev == nullptr;  // events between PDL kernels would mis-time them
  // the shared expert (every token) runs on the single-GPU layer; in a box
  // on MoE instance 0 (its partial sums carry it), or with shared_split on
  // every MoE instance for an even share of the tokens (remainder to the low
  // instances), so no instance straggles by a dense FFN over the whole step
  int sh0 = 0, sh1 = 0;
  if (ctx->shared) {
    if (ctx->instance < 0 || (!ctx->shared_split && ctx->instance == 0)) {
      sh1 = T;
    } else if (ctx->shared_split) {
      const int n = ctx->dmap.N, g = ctx->instance, base = T / n, rem = T % n;
      sh0 = g * base + std::min(g, rem);
      sh1 = sh0 + base + (g < rem ? 1 : 0);
    }
  }
  const bool shared = sh1 > sh0;
  janus::FfnPlan &ps = ctx->ffn_shared;
  if (shared) ps.tile_n = sh1 - sh0 <= 64 ? 64 : janus::kTileN;
  if (!pre) {
    st = launch_sched(ctx, d_experts, T, k, JANUS_POLICY_AEBS, 0, a, tile_off, s,
                      shared ? ctx->shared_off : nullptr, shared ? ps.tile_n : 0, sh1 - sh0,
                      abort_flag);
    if (st != JANUS_OK) return st;
  } else if (abort_flag) {  // a shard never arrived: reject the precomputed layout
    janus::SchedArgs g{};
    g.S = T * k;
    g.map = ctx->dmap;
    g.out = a;
    g.tile_off = tile_off;
    g.abort_flag = abort_flag;
    cudaError_t ge = janus::launch_abort_gate(g, s);
    if (ge != cudaSuccess) return cuda_fail(ctx, ge, "abort_gate_kernel");
    ctx->launches += 1;
  }
  if (ev) CK(cudaEventRecord(ev[1], s));
  janus::FfnPlan &p = ctx->ffn;
  cudaError_t e = janus::launch_permute(d_x, a.slot_row, a.instance, ctx->instance, T * k, k,
                                        p.d_h, p.xp, shared ? ps.xp : nullptr, sh0, sh1, s,
                                        a.status);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "permute_kernel");
  int launches = 0;
  if (ev) CK(cudaEventRecord(ev[2], s));
  // the colocated routed MoE role pushes its partial sums on a side stream
  // over y[epoch parity], beside the next step's permute and GEMMs (measured:
  // the push is ~85 us of a 4-GPU step); the GEMMs that write y[parity] again
  // two steps later wait for that push
  const janus::XferState &xs = ctx->xfer;
  const int psl = (int)(push_epoch & 1);
  const bool side_push = push_epoch && pre && !shared && !xs.mc && xs.push_stream && p.y2 &&
                         xs.transport == janus::kXferRouted && !xs.local_connect;
  if (side_push) CK(cudaStreamWaitEvent(s, xs.push_done[psl], 0));
  e = janus::launch_ffn(p, a.group_off, tile_off, s, &launches, side_push ? psl : 0);
  if (e == cudaSuccess && shared)
    e = janus::launch_ffn(ps, ctx->shared_off, ctx->shared_off + 2, s, &launches);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "grouped_gemm_kernel");
  if (ev) CK(cudaEventRecord(ev[3], s));
  if (push_epoch) {
    // box exchange: this instance's per-token partial sums go to the tokens'
    // owners — into this rank's multicast backing (NVLS: the owners'
    // switch-reduced reads add them up) or pushed into the owners' regions
    // (P2P / routed, K5 fused with the NVLink transfer) — then the step's
    // status and the combine flag are published on every attention rank
    const janus::XferState &x = ctx->xfer;
    if (x.mc && x.mc_reduce) {
      e = janus::launch_combine(p.y, a.slot_row, a.instance, ctx->instance, d_gate_w, T, k, p.d_h,
                                reinterpret_cast<void *>(x.uc_va + x.mpart_off +
                                                         janus::xfer_slot(push_epoch) * x.mslot),
                                s, shared ? ps.y : nullptr, sh0, sh1, a.status);
    } else {
      if (shared && x.transport == janus::kXferRouted)
        return fail(ctx, JANUS_EUNSUPPORTED,
                    "moe: the shared expert needs a broadcast transport (P2P or NVLS)");
      const janus::PushDst pd = janus::push_dst(x, push_epoch);
      if (side_push) {
        CK(cudaEventRecord(x.ffn_done[psl], s));
        CK(cudaStreamWaitEvent(x.push_stream, x.ffn_done[psl], 0));
        e = janus::launch_combine(psl ? p.y2 : p.y, a.slot_row, a.instance, ctx->instance,
                                  d_gate_w, T, k, p.d_h, nullptr, x.push_stream, nullptr, 0, 0,
                                  a.status, &pd, push_blocks());
        if (e == cudaSuccess) e = janus::launch_signal_combine(x, a.status, push_epoch, x.push_stream);
        if (e == cudaSuccess) e = cudaEventRecord(x.push_done[psl], x.push_stream);
        const cudaEvent_t own = x.own_sig[janus::xfer_slot(push_epoch)];
        if (e == cudaSuccess && own) e = cudaEventRecord(own, x.push_stream);
        launches += 1;
        if (e != cudaSuccess) return cuda_fail(ctx, e, "combine_kernel");
        ctx->launches += 2 + launches;
        return JANUS_OK;
      }
      e = janus::launch_combine(p.y, a.slot_row, a.instance, ctx->instance, d_gate_w, T, k, p.d_h,
                                nullptr, s, shared ? ps.y : nullptr, sh0, sh1, a.status, &pd);
    }
    if (e == cudaSuccess) e = janus::launch_signal_combine(x, a.status, push_epoch, s);
    if (e == cudaSuccess && x.own_sig[janus::xfer_slot(push_epoch)])
      e = cudaEventRecord(x.own_sig[janus::xfer_slot(push_epoch)], s);
    launches += 1;
  } else
    e = janus::launch_combine(p.y, a.slot_row, a.instance, ctx->instance, d_gate_w, T, k, p.d_h,
                              d_out, s, shared ? ps.y : nullptr, sh0, sh1, a.status);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "combine_kernel");
  ctx->launches += 2 + launches;  // permute, combine, GEMMs (launch_sched counts itself)
  return JANUS_OK;
}

extern "C" {

// The layer's kernel sequence is captured once per (buffers, T) into a CUDA
// graph and replayed: one launch per step instead of five, no host work per
// kernel.  Disabled while profiling (events), when the caller asks for the
// scheduling outputs, or with JANUS_GRAPH=0.
janus_status janus_moe_layer_async(janus_ctx *ctx, const void *d_x, const int32_t *d_experts,
                                   const float *d_gate_w, int T, void *d_out,
                                   const janus_assignment *assign, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!ctx || !ctx->use_graph || ctx->profiling || assign)
    return layer_run(ctx, d_x, d_experts, d_gate_w, T, d_out, assign, s, 0);
  const janus_ctx::GraphKey key{d_x, d_experts, d_gate_w, d_out, T};
  janus_ctx::GraphEntry *hit = nullptr;
  for (auto &g : ctx->graphs)
    if (g.key == key) hit = &g;
  if (!hit) {
    constexpr size_t kMaxGraphs = 16;
    if (ctx->graphs.size() >= kMaxGraphs) {  // evict the least recently used
      auto lru = std::min_element(ctx->graphs.begin(), ctx->graphs.end(),
                                  [](const auto &a, const auto &b) {
                                    return a.last_use < b.last_use;
                                  });
      cudaGraphExecDestroy(lru->exec);
      ctx->graphs.erase(lru);
    }
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    const uint64_t before = ctx->launches;
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    janus_status st = layer_run(ctx, d_x, d_experts, d_gate_w, T, d_out, nullptr,
                                ctx->cap_stream, 0);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &g);
    if (st != JANUS_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
    ctx->graphs.push_back({key, exec, ctx->launches - before, 0});
    ctx->launches = before;
    hit = &ctx->graphs.back();
  }
  hit->last_use = ++ctx->graph_clock;
  CK(cudaGraphLaunch(hit->exec, s));
  ctx->launches += hit->kernels;
  return JANUS_OK;
}

// ------------------------------------------------ box exchange (K6) -----

static void xfer_release(janus_ctx *ctx) {
  janus::XferState &x = ctx->xfer;
  janus::mc_free(x, ctx->device);
  if (x.local) cudaFree(x.local);
  for (void *p : x.opened) cudaIpcCloseMemHandle(p);
  dfree(x.counter);
  dfree(x.err);
  free_assign(x.rws);
  dfree(x.dmask);
  for (int i = 0; i < janus::kXferSlots; ++i) {
    free_assign(x.lay[i]);
    dfree(x.lay_tile[i]);
  }
  if (x.push_stream) {
    cudaStreamSynchronize(x.push_stream);
    cudaStreamDestroy(x.push_stream);
  }
  for (int i = 0; i < 2; ++i) {
    if (x.ffn_done[i]) cudaEventDestroy(x.ffn_done[i]);
    if (x.push_done[i]) cudaEventDestroy(x.push_done[i]);
  }
  for (int i = 0; i < janus::kXferSlots; ++i) {
    if (x.own_disp[i]) cudaEventDestroy(x.own_disp[i]);
    if (x.own_sig[i]) cudaEventDestroy(x.own_sig[i]);
    if (x.comb_done[i]) cudaEventDestroy(x.comb_done[i]);
  }
  for (cudaStream_t st : x.ce_streams) cudaStreamDestroy(st);
  for (cudaEvent_t ev : x.ce_done) cudaEventDestroy(ev);
  if (x.ce_fork) cudaEventDestroy(x.ce_fork);
  x = janus::XferState{};
  ctx->xfer_ready = false;
}

static janus_status xfer_setup(janus_ctx *ctx, int n_attn, int n_moe, int rank, int max_tokens,
                               int d_h, int k, bool colocated) {
  if (!ctx) return JANUS_EINVAL;
  const int world = colocated ? n_attn : n_attn + n_moe;
  if (n_attn < 1 || n_moe < 1 || rank < 0 || rank >= world || max_tokens < 1 || d_h <= 0 ||
      d_h % 8 || k < 1)
    return fail(ctx, JANUS_EINVAL, "xfer: bad configuration");
  if (world > 16 || n_moe > 32)
    return fail(ctx, JANUS_EUNSUPPORTED, "xfer: at most 16 ranks in one box");
  CK(cudaSetDevice(ctx->device));
  xfer_release(ctx);
  janus::XferState &x = ctx->xfer;
  x.rank = rank;
  x.world = world;
  x.moe0 = colocated ? 0 : n_attn;
  x.A = n_attn;
  x.M = n_moe;
  x.d_h = d_h;
  x.k = k;
  x.T_max = max_tokens;
  x.L = janus::xfer_layout(n_attn, n_moe, max_tokens, d_h, k);
  CK(cudaMalloc(&x.local, x.L.bytes));
  CK(cudaMemset(x.local, 0, x.L.bytes));
  CK(dalloc(&x.counter, janus::kXferSlots * janus::kCounterKinds));
  CK(dalloc(&x.err, janus::kErrWords));
  CK(cudaMemset(x.counter, 0, sizeof(unsigned) * janus::kXferSlots * janus::kCounterKinds));
  CK(cudaMemset(x.err, 0, sizeof(int) * janus::kErrWords));
  x.peer_base.assign(x.world, nullptr);
  x.peer_base[rank] = x.local;
  for (int i = 0; i < janus::kXferSlots; ++i) {
    if (colocated) {
      CK(cudaEventCreateWithFlags(&x.own_disp[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&x.own_sig[i], cudaEventDisableTiming));
    }
    if (rank < n_attn) CK(cudaEventCreateWithFlags(&x.comb_done[i], cudaEventDisableTiming));
  }
  return JANUS_OK;
}

janus_status janus_xfer_configure(janus_ctx *ctx, int n_attn, int n_moe, int rank, int max_tokens,
                                  int d_h, int k) {
  return xfer_setup(ctx, n_attn, n_moe, rank, max_tokens, d_h, k, false);
}

janus_status janus_xfer_configure_colocated(janus_ctx *ctx, int n, int rank, int max_tokens,
                                            int d_h, int k) {
  return xfer_setup(ctx, n, n, rank, max_tokens, d_h, k, true);
}

janus_status janus_xfer_set_transport(janus_ctx *ctx, int transport) {
  if (!ctx || !ctx->xfer.local) return fail(ctx, JANUS_ESTATE, "xfer: configure first");
  if (transport < 0 || transport > 2)
    return fail(ctx, JANUS_EINVAL, "xfer: transport must be 0 (P2P), 1 (routed) or 2 (copy engine)");
  janus::XferState &x = ctx->xfer;
  if (transport == janus::kXferCE) {
    if (x.mc) return fail(ctx, JANUS_EINVAL, "xfer: the copy-engine transport is point to point (no NVLS)");
    CK(cudaSetDevice(ctx->device));
    if (x.ce_streams.empty() && x.rank < x.A) {
      x.ce_streams.resize(x.M);
      x.ce_done.resize(x.M);
      for (int g = 0; g < x.M; ++g) {
        CK(cudaStreamCreateWithFlags(&x.ce_streams[g], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&x.ce_done[g], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&x.ce_fork, cudaEventDisableTiming));
    }
    x.transport = janus::kXferCE;
    return JANUS_OK;
  }
  const bool routed = transport == janus::kXferRouted;
  if (routed && x.mc)
    return fail(ctx, JANUS_EINVAL, "xfer: the routed transport is point to point (no NVLS)");
  if (routed && x.M > 32)
    return fail(ctx, JANUS_EUNSUPPORTED, "xfer: routed transport needs <= 32 MoE ranks");
  CK(cudaSetDevice(ctx->device));
  if (routed && x.rank < x.A && !x.dmask) {
    // attention side: the step's schedule (K1 over every shard's routing) and
    // the destination masks of its tokens, per epoch slot
    CK(alloc_assign(x.rws, (int)std::min<long long>(x.T_max * x.k, INT_MAX), JANUS_MAX_EXPERTS,
                    JANUS_MAX_INSTANCES, JANUS_MAX_REPLICAS));
    CK(dalloc(&x.dmask, janus::kXferSlots * x.L.ta_max));
    CK(cudaMemset(x.dmask, 0, sizeof(uint32_t) * janus::kXferSlots * x.L.ta_max));
    if (x.moe0 == 0 && ctx->ffn.h) {  // colocated with a configured layer: one K1 per step
      for (int i = 0; i < janus::kXferSlots; ++i) {
        CK(alloc_assign(x.lay[i], (int)std::min<long long>(x.T_max * x.k, INT_MAX),
                        JANUS_MAX_EXPERTS, JANUS_MAX_INSTANCES, JANUS_MAX_REPLICAS));
        CK(dalloc(&x.lay_tile[i], JANUS_MAX_REPLICAS + 1));
        CK(cudaMemset(x.lay_tile[i], 0, sizeof(int32_t) * (JANUS_MAX_REPLICAS + 1)));
      }
      // the MoE role's partial-sum push on its own stream over a second y
      janus::FfnPlan &p = ctx->ffn;
      if (!p.y2) {
        CK(cudaMalloc(&p.y2, (size_t)p.S_alloc * p.d_h * 2));
        if (p.w13) CK(janus::build_ffn_tensor_maps(p));  // with y2's map
      }
      CK(cudaStreamCreateWithFlags(&x.push_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&x.ffn_done[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&x.push_done[i], cudaEventDisableTiming));
      }
    }
  }
  x.transport = routed ? janus::kXferRouted : janus::kXferP2P;
  return JANUS_OK;
}

janus_status janus_xfer_set_combine(janus_ctx *ctx, int switch_reduce) {
  if (!ctx || !ctx->xfer.local) return fail(ctx, JANUS_ESTATE, "xfer: configure first");
  if (switch_reduce != 0 && switch_reduce != 1)
    return fail(ctx, JANUS_EINVAL, "xfer: combine mode must be 0 or 1");
  ctx->xfer.mc_reduce = switch_reduce != 0;
  return JANUS_OK;
}

janus_status janus_xfer_set_timeout(janus_ctx *ctx, uint64_t timeout_ns) {
  if (!ctx || !ctx->xfer.local) return fail(ctx, JANUS_ESTATE, "xfer: configure first");
  if (timeout_ns == 0) return fail(ctx, JANUS_EINVAL, "xfer: timeout must be > 0");
  ctx->xfer.timeout_ns = timeout_ns;
  return JANUS_OK;
}

janus_status janus_xfer_handle(const janus_ctx *ctx, uint8_t *handle) {
  if (!ctx || !ctx->xfer.local || !handle) return JANUS_ESTATE;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, ctx->xfer.local) != cudaSuccess) return JANUS_ECUDA;
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle, &h, 64);
  return JANUS_OK;
}

janus_status janus_xfer_connect(janus_ctx *ctx, const uint8_t *handles) {
  if (!ctx || !ctx->xfer.local) return JANUS_ESTATE;
  CK(cudaSetDevice(ctx->device));
  janus::XferState &x = ctx->xfer;
  for (int r = 0; r < x.world; ++r) {
    if (r == x.rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * r, 64);
    void *p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    x.peer_base[r] = p;
    x.opened.push_back(p);
  }
  ctx->xfer_ready = true;
  return JANUS_OK;
}

janus_status janus_xfer_connect_local(janus_ctx *ctx, janus_ctx *const *peers) {
  if (!ctx || !ctx->xfer.local || !peers) return JANUS_ESTATE;
  CK(cudaSetDevice(ctx->device));
  janus::XferState &x = ctx->xfer;
  for (int r = 0; r < x.world; ++r) {
    const janus_ctx *p = peers[r];
    if (!p || !p->xfer.local || p->xfer.world != x.world || p->xfer.rank != r ||
        p->xfer.L.bytes != x.L.bytes)
      return fail(ctx, JANUS_EINVAL, "xfer: peer " + std::to_string(r) +
                                          " is not configured for this box");
    if (p->device != ctx->device) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(p->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (e != cudaSuccess)
        return cuda_fail(ctx, e, "cudaDeviceEnablePeerAccess");
    }
    x.peer_base[r] = p->xfer.local;
  }
  x.local_connect = true;
  ctx->xfer_ready = true;
  return JANUS_OK;
}

// A dispatch (or routing push) into epoch slot e % kXferSlots reuses the slot
// of epoch e - kXferSlots: every MoE rank must have finished that step (its
// partial sums pushed — it no longer reads the rows, routing or layout there)
// and this rank's own combine must have summed the partials the slot holds.
// Stream order gives both when dispatch and combine share one stream; this
// makes a dispatch on a stream of its own safe: the combine by its event, the
// own MoE role by its event, the other MoE ranks by their combine flags (a
// wait kernel spinning on other GPUs only).  Once per epoch.
static janus_status slot_free_wait(janus_ctx *ctx, uint64_t epoch, cudaStream_t s) {
  janus::XferState &x = ctx->xfer;
  if (epoch <= (uint64_t)janus::kXferSlots || (x.slot_epoch == epoch && x.slot_stream == s))
    return JANUS_OK;
  const size_t sl = janus::xfer_slot(epoch);
  if (x.comb_done[sl]) CK(cudaStreamWaitEvent(s, x.comb_done[sl], 0));
  const cudaEvent_t own = x.own_sig[sl];
  if (own) CK(cudaStreamWaitEvent(s, own, 0));
  cudaError_t e = janus::launch_wait(x, 3, epoch - janus::kXferSlots, s, own ? x.rank - x.moe0 : -1);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "wait_flags_kernel");
  ctx->launches += 1;
  x.slot_epoch = epoch;
  x.slot_stream = s;
  return JANUS_OK;
}

janus_status janus_attn_route_async(janus_ctx *ctx, const int32_t *d_experts, const float *d_gate_w,
                                    int64_t T, uint64_t epoch, void *stream) {
  if (!ctx || !ctx->xfer_ready) return fail(ctx, JANUS_ESTATE, "xfer: not connected");
  janus::XferState &x = ctx->xfer;
  if (x.rank >= x.A) return fail(ctx, JANUS_EINVAL, "xfer: routing from a non-attention rank");
  if (x.transport != janus::kXferRouted)
    return fail(ctx, JANUS_ESTATE, "xfer: routing phase of the routed transport only");
  if (T < 0 || T > x.T_max || epoch == 0 || !d_experts || !d_gate_w)
    return fail(ctx, JANUS_EINVAL, "xfer: num_tokens outside [0, max_tokens], epoch 0 or no routing");
  janus_status st = slot_free_wait(ctx, epoch, static_cast<cudaStream_t>(stream));
  if (st != JANUS_OK) return st;
  cudaError_t e = janus::launch_route_push(x, d_experts, d_gate_w, T, epoch,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "route_push_kernel");
  ctx->launches += 1;
  x.routed_epoch = epoch;
  return JANUS_OK;
}

janus_status janus_attn_dispatch_async(janus_ctx *ctx, const void *d_x, const int32_t *d_experts,
                                       const float *d_gate_w, int64_t T, uint64_t epoch,
                                       void *stream) {
  if (!ctx || !ctx->xfer_ready) return fail(ctx, JANUS_ESTATE, "xfer: not connected");
  const janus::XferState &x = ctx->xfer;
  if (x.rank >= x.A) return fail(ctx, JANUS_EINVAL, "xfer: dispatch from a non-attention rank");
  if (T < 0 || T > x.T_max || epoch == 0)
    return fail(ctx, JANUS_EINVAL, "xfer: num_tokens outside [0, max_tokens] or epoch 0");
  if (!d_experts != !d_gate_w)
    return fail(ctx, JANUS_EINVAL, "xfer: pass both routing arrays, or neither (MoE-side gating)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  janus_status fs = slot_free_wait(ctx, epoch, s);
  if (fs != JANUS_OK) return fs;
  // a colocated rank's MoE role waits for this dispatch by an event
  const cudaEvent_t own = x.own_disp[janus::xfer_slot(epoch)];
  if (x.transport == janus::kXferCE) {  // copy engines: no kernel
    cudaError_t e = janus::launch_dispatch_ce(x, d_x, d_experts, d_gate_w, T, epoch, s);
    if (e == cudaSuccess && own) e = cudaEventRecord(own, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "copy-engine dispatch");
    return JANUS_OK;
  }
  if (x.transport != janus::kXferRouted) {
    cudaError_t e = janus::launch_dispatch(x, d_x, d_experts, d_gate_w, T, epoch, s);
    if (e == cudaSuccess && own) e = cudaEventRecord(own, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "dispatch_kernel");
    ctx->launches += 1;
    return JANUS_OK;
  }
  // routed: the routing first (every rank), then K1 over the whole step here —
  // identical to every MoE rank's — then each row only to its instances
  if (!d_experts)
    return fail(ctx, JANUS_EINVAL, "xfer: the routed transport needs the routing on the attention side");
  if (!ctx->have_map)
    return fail(ctx, JANUS_ESTATE, "xfer: the routed transport needs the replica map on attention ranks");
  if (ctx->dmap.N != x.M)
    return fail(ctx, JANUS_EINVAL, "xfer: replica map instances != MoE ranks");
  cudaError_t e = cudaSuccess;
  if (x.routed_epoch != epoch) {  // not pushed ahead by janus_attn_route_async
    janus_status rs = janus_attn_route_async(ctx, d_experts, d_gate_w, T, epoch, stream);
    if (rs != JANUS_OK) return rs;
  }
  const int32_t *full = d_experts;  // one attention rank: its shard is the step
  const int *abort_flag = nullptr;
  if (x.A > 1) {
    e = janus::launch_wait(x, 2, epoch, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "wait_flags_kernel");
    ctx->launches += 1;
    full = reinterpret_cast<const int32_t *>(static_cast<const unsigned char *>(x.local) +
                                             x.L.ex_off + janus::xfer_slot(epoch) * x.L.slot_stride);
    abort_flag = x.err + janus::kErrSkip + 2;
  }
  const int sl = (int)janus::xfer_slot(epoch);
  const bool full_layout = x.lay[sl].instance != nullptr;  // colocated: the MoE role reuses it
  janus_assignment ra = full_layout ? x.lay[sl] : x.rws;
  ra.row_slot = nullptr;
  if (!full_layout) ra.slot_row = ra.group_off = nullptr;
  if (full_layout) ctx->ffn.tile_n = layer_tile_n(ctx, (int)T);
  janus_status st = launch_sched(ctx, full, (int)T, x.k, JANUS_POLICY_AEBS, 0, ra,
                                 full_layout ? x.lay_tile[sl] : nullptr, s, nullptr, 0, 0,
                                 abort_flag);
  if (st != JANUS_OK) return st;
  e = janus::launch_routed_dispatch(x, d_x, ra.instance, ra.status, T, epoch, s);
  if (e == cudaSuccess && own) e = cudaEventRecord(own, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "routed_dispatch_kernel");
  ctx->launches += 1;
  return JANUS_OK;
}

janus_status janus_moe_layer_xfer_async(janus_ctx *ctx, int64_t T, uint64_t epoch, void *stream) {
  if (!ctx || !ctx->xfer_ready) return fail(ctx, JANUS_ESTATE, "xfer: not connected");
  const janus::XferState &x = ctx->xfer;
  if (x.rank < x.moe0 || ctx->instance != x.rank - x.moe0)
    return fail(ctx, JANUS_EINVAL, "xfer: MoE rank must hold instance rank - n_attn");
  if (T < 0 || T > x.T_max || epoch == 0)
    return fail(ctx, JANUS_EINVAL, "xfer: num_tokens outside [0, max_tokens] or epoch 0");
  if (ctx->router && x.transport == janus::kXferRouted)
    return fail(ctx, JANUS_EINVAL, "xfer: MoE-side gating needs a broadcast transport");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // own attention role (colocated): ordered by its event, not spun on (the
  // host enqueues a step's dispatch before its MoE step)
  const cudaEvent_t own = x.own_disp[janus::xfer_slot(epoch)];
  if (own) CK(cudaStreamWaitEvent(s, own, 0));
  cudaError_t e = janus::launch_wait(x, 0, epoch, s, own ? x.rank : -1);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "wait_flags_kernel");
  ctx->launches += 1;
  const int *abort_flag = x.err + janus::kErrSkip + 0;  // a shard never arrived
  if (ctx->router) {  // MoE-side gating: routing from the received rows
    unsigned char *base =
        x.mc ? reinterpret_cast<unsigned char *>(x.uc_va) + janus::xfer_slot(epoch) * x.mslot
             : static_cast<unsigned char *>(x.local) + janus::xfer_slot(epoch) * x.L.slot_stride;
    const void *xr = base + (x.mc ? x.mx_off : x.L.x_off);
    janus_status gs = janus_gate_async(ctx, xr, ctx->router, T, ctx->d_h, ctx->dmap.E,
                                       ctx->top_k, ctx->d_experts, ctx->d_gw, stream);
    if (gs != JANUS_OK) return gs;
    return layer_run(ctx, xr, ctx->d_experts, ctx->d_gw, (int)T, nullptr, nullptr, s, epoch,
                     abort_flag);
  }
  if (x.mc) {  // rows / routing landed in this rank's multicast backing
    unsigned char *base = reinterpret_cast<unsigned char *>(x.uc_va) + janus::xfer_slot(epoch) * x.mslot;
    return layer_run(ctx, base + x.mx_off, reinterpret_cast<const int32_t *>(base + x.mex_off),
                     reinterpret_cast<const float *>(base + x.mgw_off), (int)T, nullptr, nullptr,
                     s, epoch, abort_flag);
  }
  unsigned char *base =
      static_cast<unsigned char *>(x.local) + janus::xfer_slot(epoch) * x.L.slot_stride;
  const int sl = (int)janus::xfer_slot(epoch);
  if (x.transport == janus::kXferRouted && x.lay[sl].instance && !ctx->shared)
    // this rank's own dispatch of the epoch (flagged before the wait above
    // returned) computed the step's layout: no second K1
    return layer_run(ctx, base + x.L.x_off, nullptr,
                     reinterpret_cast<const float *>(base + x.L.gw_off), (int)T, nullptr, nullptr,
                     s, epoch, abort_flag, &x.lay[sl], x.lay_tile[sl]);
  return layer_run(ctx, base + x.L.x_off, reinterpret_cast<const int32_t *>(base + x.L.ex_off),
                   reinterpret_cast<const float *>(base + x.L.gw_off), (int)T, nullptr, nullptr, s,
                   epoch, abort_flag);
}

janus_status janus_attn_combine_async(janus_ctx *ctx, void *d_out, int64_t T, uint64_t epoch,
                                      void *stream) {
  if (!ctx || !ctx->xfer_ready) return fail(ctx, JANUS_ESTATE, "xfer: not connected");
  const janus::XferState &x = ctx->xfer;
  if (x.rank >= x.A) return fail(ctx, JANUS_EINVAL, "xfer: combine on a non-attention rank");
  if (T < 0 || T > x.T_max || epoch == 0)
    return fail(ctx, JANUS_EINVAL, "xfer: num_tokens outside [0, max_tokens] or epoch 0");
  int64_t first = 0, Ta = 0;
  janus_shard_tokens(T, x.A, x.rank, &first, &Ta);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // own MoE role (colocated): ordered by its event (the host enqueues a
  // step's MoE step before its combine), not spun on
  const cudaEvent_t own = x.own_sig[janus::xfer_slot(epoch)];
  if (own) CK(cudaStreamWaitEvent(s, own, 0));
  cudaError_t e = janus::launch_wait(x, 1, epoch, s, own ? x.rank - x.moe0 : -1);
  if (e == cudaSuccess)
    e = x.mc && x.mc_reduce ? janus::launch_reduce_mc(x, d_out, first, Ta, epoch, s)
                            : janus::launch_reduce_partials(x, d_out, Ta, epoch, s);
  if (e != cudaSuccess)
    return cuda_fail(ctx, e, x.mc && x.mc_reduce ? "reduce_mc_kernel" : "reduce_partials_kernel");
  // the slot's next dispatch (kXferSlots epochs on) waits for this combine
  if (x.comb_done[janus::xfer_slot(epoch)])
    CK(cudaEventRecord(x.comb_done[janus::xfer_slot(epoch)], s));
  ctx->launches += 2;
  return JANUS_OK;
}

janus_status janus_xfer_recv_rows(const janus_ctx *ctx, uint64_t epoch, void **rows) {
  if (!ctx || !ctx->xfer.local || !rows) return JANUS_ESTATE;
  const janus::XferState &x = ctx->xfer;
  *rows = x.mc ? reinterpret_cast<void *>(x.uc_va + x.mx_off + janus::xfer_slot(epoch) * x.mslot)
               : static_cast<unsigned char *>(x.local) + x.L.x_off +
                     janus::xfer_slot(epoch) * x.L.slot_stride;
  return JANUS_OK;
}

janus_status janus_xfer_check(janus_ctx *ctx) {
  if (!ctx || !ctx->xfer.err) return fail(ctx, JANUS_ESTATE, "xfer: configure first");
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  int w[janus::kErrWords];
  CK(cudaMemcpy(w, ctx->xfer.err, sizeof(w), cudaMemcpyDeviceToHost));
  if (w[janus::kErrStatus] == JANUS_OK) return JANUS_OK;
  const int st = w[janus::kErrStatus], bad = w[janus::kErrBad];
  // report once: clear the sticky words (the timeout flag stays for janus_xfer_status)
  CK(cudaMemset(ctx->xfer.err + janus::kErrStatus, 0, 2 * sizeof(int)));
  if (st == JANUS_EUNKNOWN_EXPERT)
    return fail(ctx, JANUS_EUNKNOWN_EXPERT,
                "unknown-expert: batch references expert " + std::to_string(bad) +
                    " with no replica in the map");
  if (st == JANUS_EPEER)
    return fail(ctx, JANUS_EPEER, "xfer: a peer rank never published its step (wait bound expired)");
  return fail(ctx, (janus_status)st, "xfer: a step of the box failed (status " +
                                         std::to_string(st) + ")");
}

// the gate's split-K exchange buffer: once per context, at its largest size
// (bounded by the SM count), so no call allocates inside a stream capture after
// the first
static cudaError_t alloc_gate_xchg(janus_ctx *ctx) {
  if (ctx->gate_xchg) return cudaSuccess;
  int sms = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (e != cudaSuccess) return e;
  return cudaMalloc(&ctx->gate_xchg, janus::gate_xchg_bytes(sms));
}

janus_status janus_gate_async(janus_ctx *ctx, const void *d_x, const void *d_router, int64_t T,
                              int d_hidden, int num_experts, int top_k, int32_t *d_experts,
                              float *d_gate_w, void *stream) {
  if (!ctx) return JANUS_EINVAL;
  if (T < 0 || T > (1 << 26) || (T > 0 && (!d_x || !d_router || !d_experts || !d_gate_w)))
    return fail(ctx, JANUS_EINVAL, "gate: bad arguments");
  if (!janus::gate_shape_ok(d_hidden, num_experts, top_k))
    return fail(ctx, JANUS_EUNSUPPORTED,
                "gate: need d_hidden % 64 == 0, 16 <= num_experts <= 256, num_experts % 16 == 0, "
                "1 <= top_k <= min(16, num_experts)");
  CK(cudaSetDevice(ctx->device));
  CK(alloc_gate_xchg(ctx));
  cudaError_t e = janus::launch_gate(d_x, d_router, (int)T, d_hidden, num_experts, top_k,
                                     d_experts, d_gate_w, ctx->gate_xchg,
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gate_kernel");
  if (T > 0) ctx->launches += 1;
  return JANUS_OK;
}

janus_status janus_moe_set_router(janus_ctx *ctx, const void *d_router) {
  if (!ctx) return JANUS_EINVAL;
  if (!d_router) return fail(ctx, JANUS_EINVAL, "gate: null router");
  CK(cudaSetDevice(ctx->device));
  CK(alloc_gate_xchg(ctx));
  ctx->router = d_router;
  return JANUS_OK;
}

janus_status janus_moe_layer_gated_async(janus_ctx *ctx, const void *d_x, int T, void *d_out,
                                         void *stream) {
  if (!ctx) return JANUS_EINVAL;
  if (!ctx->router) return fail(ctx, JANUS_ESTATE, "gate: janus_moe_set_router first");
  if (!ctx->d_experts) return fail(ctx, JANUS_ESTATE, "moe: janus_moe_configure first");
  if (T < 0 || T > ctx->max_tokens)
    return fail(ctx, JANUS_EINVAL, "moe: num_tokens outside [0, max_tokens]");
  janus_status st = janus_gate_async(ctx, d_x, ctx->router, T, ctx->d_h, ctx->dmap.E,
                                     ctx->top_k, ctx->d_experts, ctx->d_gw, stream);
  if (st != JANUS_OK) return st;
  return janus_moe_layer_async(ctx, d_x, ctx->d_experts, ctx->d_gw, T, d_out, nullptr, stream);
}

static void free_stats(janus::StatsState &st) {
  dfree(st.counts);
  dfree(st.coact);
  dfree(st.ring);
  dfree(st.mask);
  dfree(st.step);
  dfree(st.bad);
  st = janus::StatsState{};
}

janus_status janus_stats_configure(janus_ctx *ctx, int num_experts, int window) {
  if (!ctx) return JANUS_EINVAL;
  if (num_experts <= 0) return fail(ctx, JANUS_EINVAL, "stats: num_experts must be > 0");
  if (window <= 0) return fail(ctx, JANUS_EINVAL, "stats: window must be > 0");
  if (num_experts > JANUS_MAX_EXPERTS)
    return fail(ctx, JANUS_EUNSUPPORTED, "stats: at most JANUS_MAX_EXPERTS experts");
  CK(cudaSetDevice(ctx->device));
  janus::StatsState &st = ctx->stats;
  free_stats(st);
  const int words = (num_experts + 31) / 32;
  st.E = num_experts;
  st.W = window;
  CK(dalloc(&st.counts, num_experts));
  CK(dalloc(&st.coact, (size_t)num_experts * num_experts));
  CK(dalloc(&st.ring, (size_t)window * words));
  CK(dalloc(&st.mask, words));
  CK(dalloc(&st.step, 1));
  CK(dalloc(&st.bad, 1));
  CK(cudaMemset(st.counts, 0, sizeof(long long) * num_experts));
  CK(cudaMemset(st.coact, 0, sizeof(long long) * num_experts * num_experts));
  CK(cudaMemset(st.ring, 0, sizeof(uint32_t) * window * words));
  CK(cudaMemset(st.step, 0, sizeof(long long)));
  const int none = INT_MAX;
  CK(cudaMemcpy(st.bad, &none, sizeof(int), cudaMemcpyHostToDevice));
  return JANUS_OK;
}

janus_status janus_stats_record_async(janus_ctx *ctx, const int32_t *d_experts, int64_t T,
                                      int top_k, void *stream) {
  if (!ctx) return JANUS_EINVAL;
  if (!ctx->stats.counts) return fail(ctx, JANUS_ESTATE, "stats: janus_stats_configure first");
  if (T < 0 || top_k < 1 || (T > 0 && !d_experts))
    return fail(ctx, JANUS_EINVAL, "stats: bad batch");
  cudaError_t e = janus::launch_stats_record(ctx->stats, d_experts, T * top_k,
                                             static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "stats kernels");
  ctx->launches += 3;
  return JANUS_OK;
}

janus_status janus_stats_read(janus_ctx *ctx, int64_t *counts, int64_t *coact, int *recorded) {
  if (!ctx) return JANUS_EINVAL;
  const janus::StatsState &st = ctx->stats;
  if (!st.counts) return fail(ctx, JANUS_ESTATE, "stats: janus_stats_configure first");
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  if (counts) CK(cudaMemcpy(counts, st.counts, sizeof(int64_t) * st.E, cudaMemcpyDeviceToHost));
  if (coact)
    CK(cudaMemcpy(coact, st.coact, sizeof(int64_t) * st.E * st.E, cudaMemcpyDeviceToHost));
  if (recorded) {
    long long step = 0;
    CK(cudaMemcpy(&step, st.step, sizeof(long long), cudaMemcpyDeviceToHost));
    *recorded = (int)std::min<long long>(step, st.W);
  }
  return JANUS_OK;
}

janus_status janus_stats_status(janus_ctx *ctx, int *bad_expert) {
  if (!ctx) return JANUS_EINVAL;
  if (!ctx->stats.bad) return fail(ctx, JANUS_ESTATE, "stats: janus_stats_configure first");
  CK(cudaSetDevice(ctx->device));
  int bad = INT_MAX;
  CK(cudaMemcpy(&bad, ctx->stats.bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad_expert) *bad_expert = bad == INT_MAX ? -1 : bad;
  if (bad != INT_MAX)
    return fail(ctx, JANUS_EINVAL,
                "stats: activated expert " + std::to_string(bad) + " out of range");
  return JANUS_OK;
}

janus_status janus_xfer_mc_supported(janus_ctx *ctx, int *yes) {
  if (!ctx || !yes) return JANUS_EINVAL;
  *yes = janus::mc_supported(ctx->device) ? 1 : 0;
  return JANUS_OK;
}

janus_status janus_xfer_mc_create(janus_ctx *ctx, int *fd) {
  if (!ctx || !fd) return JANUS_EINVAL;
  if (!ctx->xfer_ready) return fail(ctx, JANUS_ESTATE, "xfer: connect before the multicast setup");
  CK(cudaSetDevice(ctx->device));
  const std::string e = janus::mc_create(ctx->xfer, ctx->device, fd);
  if (!e.empty()) return fail(ctx, JANUS_ECUDA, e);
  return JANUS_OK;
}

janus_status janus_xfer_mc_join(janus_ctx *ctx, int fd) {
  if (!ctx) return JANUS_EINVAL;
  if (!ctx->xfer_ready) return fail(ctx, JANUS_ESTATE, "xfer: connect before the multicast setup");
  CK(cudaSetDevice(ctx->device));
  const std::string e = janus::mc_join(ctx->xfer, ctx->device, fd);
  if (!e.empty()) return fail(ctx, JANUS_ECUDA, e);
  return JANUS_OK;
}

janus_status janus_xfer_mc_bind(janus_ctx *ctx) {
  if (!ctx) return JANUS_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const std::string e = janus::mc_bind(ctx->xfer, ctx->device);
  if (!e.empty()) return fail(ctx, JANUS_ECUDA, e);
  return JANUS_OK;
}

janus_status janus_xfer_status(janus_ctx *ctx, int *timed_out) {
  if (!ctx || !ctx->xfer.err) return JANUS_ESTATE;
  CK(cudaMemcpy(timed_out, ctx->xfer.err, sizeof(int), cudaMemcpyDeviceToHost));
  return JANUS_OK;
}

janus_status janus_moe_layer(janus_ctx *ctx, const void *x, const int32_t *experts,
                             const float *gate_w, int T, void *out) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (!ctx->moe_ready) return fail(ctx, JANUS_ESTATE, "moe: weights not set");
  if (T < 0 || T > ctx->max_tokens)
    return fail(ctx, JANUS_EINVAL, "moe: num_tokens outside [0, max_tokens]");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t S = (size_t)T * ctx->top_k;
  CK(cudaMemcpyAsync(ctx->d_x, x, (size_t)T * ctx->d_h * 2, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->d_experts, experts, S * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->d_gw, gate_w, S * 4, cudaMemcpyHostToDevice, s));
  st = janus_moe_layer_async(ctx, ctx->d_x, ctx->d_experts, ctx->d_gw, T, ctx->d_outbuf, nullptr,
                             s);
  if (st != JANUS_OK) return st;
  int32_t status[2];
  CK(cudaMemcpyAsync(out, ctx->d_outbuf, (size_t)T * ctx->d_h * 2, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(status, ctx->ws.status, sizeof(status), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (status[0] == JANUS_EUNKNOWN_EXPERT)
    return fail(ctx, JANUS_EUNKNOWN_EXPERT,
                "unknown-expert: batch references expert " + std::to_string(status[1]) +
                    " with no replica in the map");
  return JANUS_OK;
}

namespace {
// keep the first non-OK scheduler status of the pipelined host calls
__global__ void sticky_status_kernel(const int32_t *status, int32_t *sticky) {
  if (status[0] != JANUS_OK && sticky[0] == JANUS_OK) {
    sticky[0] = status[0];
    sticky[1] = status[1];
  }
}
}  // namespace

static void free_host_pipe(janus_ctx *ctx) {
  auto &hp = ctx->hp;
  if (!hp.ready) return;
  cudaDeviceSynchronize();
  for (int b = 0; b < janus_ctx::kHostSets; ++b) {
    dfree(hp.x[b]);
    dfree(hp.out[b]);
    dfree(hp.ex[b]);
    dfree(hp.gw[b]);
    cudaEventDestroy(hp.h2d_ev[b]);
    cudaEventDestroy(hp.comp_ev[b]);
    cudaEventDestroy(hp.free_ev[b]);
  }
  dfree(hp.sticky);
  cudaStreamDestroy(hp.h2d);
  cudaStreamDestroy(hp.d2h);
  hp = janus_ctx::HostPipe{};
}

janus_status janus_moe_layer_host_async(janus_ctx *ctx, const void *x, const int32_t *experts,
                                        const float *gate_w, int T, void *out) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  if (!ctx->moe_ready) return fail(ctx, JANUS_ESTATE, "moe: weights not set");
  if (T < 0 || T > ctx->max_tokens)
    return fail(ctx, JANUS_EINVAL, "moe: num_tokens outside [0, max_tokens]");
  CK(cudaSetDevice(ctx->device));
  auto &hp = ctx->hp;
  if (!hp.ready) {
    CK(cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking));
    const size_t S = (size_t)ctx->max_tokens * ctx->top_k;
    for (int b = 0; b < janus_ctx::kHostSets; ++b) {
      CK(cudaMalloc(&hp.x[b], (size_t)ctx->max_tokens * ctx->d_h * 2));
      CK(cudaMalloc(&hp.out[b], (size_t)ctx->max_tokens * ctx->d_h * 2));
      CK(dalloc(&hp.ex[b], S));
      CK(dalloc(&hp.gw[b], S));
      CK(cudaEventCreateWithFlags(&hp.h2d_ev[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&hp.comp_ev[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&hp.free_ev[b], cudaEventDisableTiming));
    }
    CK(dalloc(&hp.sticky, 2));
    CK(cudaMemset(hp.sticky, 0, 2 * sizeof(int32_t)));
    hp.ready = true;
  }
  const int b = (int)(hp.calls % janus_ctx::kHostSets);
  const size_t S = (size_t)T * ctx->top_k;
  // H2D into set b once the call that last used it has been copied out
  CK(cudaStreamWaitEvent(hp.h2d, hp.free_ev[b], 0));
  CK(cudaMemcpyAsync(hp.x[b], x, (size_t)T * ctx->d_h * 2, cudaMemcpyHostToDevice, hp.h2d));
  CK(cudaMemcpyAsync(hp.ex[b], experts, S * 4, cudaMemcpyHostToDevice, hp.h2d));
  CK(cudaMemcpyAsync(hp.gw[b], gate_w, S * 4, cudaMemcpyHostToDevice, hp.h2d));
  CK(cudaEventRecord(hp.h2d_ev[b], hp.h2d));
  CK(cudaStreamWaitEvent(ctx->stream, hp.h2d_ev[b], 0));
  st = janus_moe_layer_async(ctx, hp.x[b], hp.ex[b], hp.gw[b], T, hp.out[b], nullptr, ctx->stream);
  if (st != JANUS_OK) return st;
  sticky_status_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ws.status, hp.sticky);
  CK(cudaGetLastError());
  ctx->launches += 1;
  CK(cudaEventRecord(hp.comp_ev[b], ctx->stream));
  CK(cudaStreamWaitEvent(hp.d2h, hp.comp_ev[b], 0));
  CK(cudaMemcpyAsync(out, hp.out[b], (size_t)T * ctx->d_h * 2, cudaMemcpyDeviceToHost, hp.d2h));
  CK(cudaEventRecord(hp.free_ev[b], hp.d2h));
  hp.calls++;
  return JANUS_OK;
}

janus_status janus_moe_host_sync(janus_ctx *ctx) {
  if (!ctx) return JANUS_EINVAL;
  auto &hp = ctx->hp;
  if (!hp.ready) return JANUS_OK;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(hp.h2d));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaStreamSynchronize(hp.d2h));
  int32_t sticky[2];
  CK(cudaMemcpy(sticky, hp.sticky, sizeof(sticky), cudaMemcpyDeviceToHost));
  if (sticky[0] != JANUS_OK) {
    CK(cudaMemset(hp.sticky, 0, sizeof(sticky)));
    return fail(ctx, JANUS_EUNKNOWN_EXPERT,
                "unknown-expert: batch references expert " + std::to_string(sticky[1]) +
                    " with no replica in the map");
  }
  return JANUS_OK;
}

janus_status janus_trace_schedule(janus_ctx *ctx, const int32_t *d_experts, int T, int k,
                                  int64_t *ns) {
  janus_status st = check_ready(ctx);
  if (st != JANUS_OK) return st;
  CK(cudaSetDevice(ctx->device));
  st = grow_sched(ctx, T * k);
  if (st != JANUS_OK) return st;
  uint64_t *d_trace = nullptr;
  CK(cudaMalloc(&d_trace, 16 * sizeof(uint64_t)));
  CK(cudaMemset(d_trace, 0, 16 * sizeof(uint64_t)));
  janus::SchedArgs a{};
  a.experts = d_experts;
  a.S = T * k;
  a.k = k;
  a.map = ctx->dmap;
  a.id_bits = janus::id_bits_for(ctx->dmap.E);
  a.policy = JANUS_POLICY_AEBS;
  a.out = ctx->d_out;
  a.trace = d_trace;
  a.tile_n = janus::kTileN;
  // three passes, the last one traced warm (the first pays instruction-cache
  // misses on every phase)
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 3 && e == cudaSuccess; ++i) e = janus::launch_schedule(a, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  uint64_t h[16] = {0};
  if (e == cudaSuccess) e = cudaMemcpy(h, d_trace, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d_trace);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "janus_trace_schedule");
  ctx->launches += 3;
  for (int i = 0; i < 7; ++i) ns[i] = (int64_t)(h[i] - h[0]);
  ns[7] = (int64_t)h[7];  // SM cycles of the pass (0 where not recorded)
  return JANUS_OK;
}

janus_status janus_profile(janus_ctx *ctx, int enable) {
  if (!ctx) return JANUS_EINVAL;
  ctx->profiling = enable != 0;
  ctx->prof_calls = 0;
  return JANUS_OK;
}

janus_status janus_profile_read(janus_ctx *ctx, double *sched_ms, double *ffn_ms, int *calls) {
  if (!ctx) return JANUS_EINVAL;
  CK(cudaSetDevice(ctx->device));
  double a = 0, b = 0;
  for (int i = 0; i < ctx->prof_calls; ++i) {
    cudaEvent_t *ev = &ctx->prof_events[4 * (size_t)i];
    float x = 0, y = 0;
    CK(cudaEventSynchronize(ev[3]));
    CK(cudaEventElapsedTime(&x, ev[0], ev[1]));
    CK(cudaEventElapsedTime(&y, ev[2], ev[3]));
    a += x;
    b += y;
  }
  if (sched_ms) *sched_ms = a;
  if (ffn_ms) *ffn_ms = b;
  if (calls) *calls = ctx->prof_calls;
  ctx->prof_calls = 0;
  return JANUS_OK;
}

void janus_shard_tokens(int64_t T, int A, int a, int64_t *first, int64_t *count) {
  // src/comm.cpp:76-81: even split, remainder to the lowest instance ids
  const int64_t base = T / A, rem = T % A;
  *count = base + (a < rem ? 1 : 0);
  *first = a * base + std::min<int64_t>(a, rem);
}

// src/latency.cpp:17-32 (the reference's accounting, unchanged).
double janus_moe_layer_latency(int N, const int32_t *load, const int64_t *routed, int d_h,
                               int d_e, int bpp, double peak_flops, double hbm_bw,
                               double t_launch) {
  double worst = 0;
  for (int g = 0; g < N; ++g) {
    if (load[g] <= 0) continue;
    const double mem = load[g] * (2.0 * d_h * d_e * bpp) / hbm_bw;
    const double comp = 2.0 * static_cast<double>(routed[g]) * d_h * d_e / peak_flops;
    worst = std::max(worst, t_launch + std::max(mem, comp));
  }
  return worst;
}

}  // extern "C"
