// internal.h — context and shared declarations of libjanus_b200.so.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "janus_b200.h"

namespace janus {

constexpr int kSchedThreads = 1024;  // one CTA, 32 warps

// Map-derived tables on the device (uploaded once per janus_set_replica_map).
struct DevMap {
  int E = 0, N = 0, C = 0, R = 0;
  void *blob = nullptr;  // the one allocation every table below points into
  int32_t *off = nullptr, *hosts = nullptr, *rid = nullptr, *qidx = nullptr;
  uint32_t *hmask = nullptr;  // per-expert host bitmask (N <= 32 only)
  // compact tables of the single-CTA decode scheduler (N <= 32): per expert
  // {off, replicas, host bitmask, first host}; per replica {rid, qidx}; the
  // multi-replica experts and, per instance, its single-replica experts as
  // bitmasks of ceil(E/32) words ([E/32] and [N][E/32])
  int4 *ex_info = nullptr;
  int2 *rep_info = nullptr;
  uint32_t *multi_mask = nullptr, *pin_mask = nullptr;
  // host_mask [N][E/32]: the multi-replica experts hosted on instance g (the
  // greedy's candidate test without a shuffle); qbase [N+1]: first replica of
  // instance g in replica order (routed_tokens from the scanned group offsets)
  uint32_t *host_mask = nullptr;
  int32_t *qbase = nullptr;
  // pair_info [E] + pair_bhi [E] (N <= 8 and C <= 255: loads fit a byte), the
  // one-lane greedy's record per multi-replica expert.  Two hosts a < b:
  // {a << 12 | b << 28 (PRMT selectors: load[a] / load[b] as the top byte
  // over identical low bytes), +1 at a in the lo / hi load word, +1 at b in
  // the lo word}, pair_bhi = +1 at b in the hi word.  Three or more:
  // {~0, host bitmask, 0, 0}.
  uint4 *pair_info = nullptr;
  uint32_t *pair_bhi = nullptr;
  int pairs_only = 0;  // every multi-replica expert has exactly two hosts
};

struct SchedArgs {
  const int32_t *experts;
  int S, k;
  DevMap map;
  int policy;
  uint64_t rng_state;  // derive_seed(seed, "sched/random")
  janus_assignment out;
  int32_t *tile_off;   // [R+1] n-tile prefix for the grouped GEMM, optional
  int tile_n;          // token rows per GEMM n-tile (64 or 256)
  uint64_t *trace;     // [7] phase timestamps (%globaltimer), optional
  int id_bits;         // bits of the largest expert id (ballot-based peer matching)
  int merge_tail;      // 1: a group's last n-tile also takes the remainder (wide tiles)
  int32_t *shared_off;  // optional [4]: the shared expert's {0, rows} and {0, n-tiles}
  int shared_tile_n;
  int shared_rows;      // tokens this instance runs the shared expert on
  const int *abort_flag;  // optional: non-zero -> reject the step (JANUS_EPEER)
};

inline int id_bits_for(int E) {
  int b = 1;
  while ((1 << b) < E) ++b;
  return b;
}

// Launches the fused scheduler + layout kernel (aebs.cu).
cudaError_t launch_schedule(const SchedArgs &a, cudaStream_t stream);
// A layout computed earlier is used as is, unless *a.abort_flag: then the
// error layout (JANUS_EPEER) is written over it (aebs.cu).
cudaError_t launch_abort_gate(const SchedArgs &a, cudaStream_t stream);
size_t schedule_smem_bytes(int E, int N, int R);

// MoE FFN workspace (ffn.cu).
constexpr int kTileN = 256;  // token rows per GEMM tile (CTA-pair UMMA N <= 256)

struct FfnPlan {
  int d_h = 0, d_e = 0, S_alloc = 0;
  int q_begin = 0, q_end = 0;   // replica groups computed here
  int tile_n = kTileN;          // token rows per n-tile for this call (64 decode / 256)
  const void *w13 = nullptr, *w2 = nullptr;
  void *xp = nullptr, *h = nullptr, *y = nullptr;  // bf16 [S_alloc][.]
  unsigned *tile_ctr = nullptr;  // [4] per GEMM: next-tile counter, finished CTAs (self-resetting)
  CUtensorMap tm_w13, tm_w2;
  CUtensorMap tm_xp[5], tm_h[5];  // box rows 8/16/32/64/128 (half of a pair's N)
  CUtensorMap tm_h_out, tm_y_out;  // epilogue TMA stores (box 16 / 32 features x 32 rows)
  // a second y for the box's MoE role (colocated routed ranks): step s's
  // partial-sum push reads y[s & 1] on a side stream while step s+1's GEMMs
  // write the other one
  void *y2 = nullptr;
  CUtensorMap tm_y_out2;
  bool maps_ready = false;
};

cudaError_t build_ffn_tensor_maps(FfnPlan &p);
// xp_shared (optional): also store row t of x at xp_shared[t - sh0] for
// t in [sh0, sh1) (the shared expert's token rows, in token order)
cudaError_t launch_permute(const void *x, const int32_t *slot_row, const int32_t *slot_instance,
                           int instance, int S, int k, int d_h, void *xp, void *xp_shared,
                           int sh0, int sh1,
                           cudaStream_t s, const int32_t *status = nullptr);
// gate/up GEMM with fused SwiGLU, then the down GEMM; 2 launches.
cudaError_t launch_ffn(const FfnPlan &p, const int32_t *group_off, const int32_t *tile_off,
                       cudaStream_t s, int *launches, int ybuf = 0);
// K5 push mode (box exchange): token t's partial sum goes to its owning
// attention rank a (shard rule, comm.cpp:76-81) at part[g][t - first_a] of that
// rank's region; skip_empty: tokens with no slot on this instance send nothing.
constexpr int kPushMaxPeers = 16;
struct PushDst {
  unsigned char *base[kPushMaxPeers];  // attention ranks' regions (A == 0: local out)
  size_t part_off;
  long long ta_max;
  int A, g, skip_empty;
};

// y_shared (optional): + y_shared[t - sh0] (weight 1) after the k routed
// slots, for t in [sh0, sh1)
cudaError_t launch_combine(const void *y, const int32_t *slot_row, const int32_t *slot_instance,
                           int instance, const float *gate_w, int T, int k, int d_h, void *out,
                           cudaStream_t s, const void *y_shared = nullptr, int sh0 = 0,
                           int sh1 = 0, const int32_t *status = nullptr,
                           const PushDst *push = nullptr, int max_blocks = 0);

// MoE-side gating (gate.cu): router GEMM + top-k + softmax of the top-k logits.
bool gate_shape_ok(int d_h, int E, int k);
// xchg: the split-K exchange buffer, gate_xchg_bytes(SM count) bytes
size_t gate_xchg_bytes(int sms);
cudaError_t launch_gate(const void *x, const void *wr, int T, int d_h, int E, int k,
                        int32_t *experts, float *gw, float *xchg, cudaStream_t s);

// GPU activation statistics (stats.cu): ActivationStats on the device.
struct StatsState {
  int E = 0, W = 0;
  long long *counts = nullptr;  // [E]
  long long *coact = nullptr;   // [E*E]
  uint32_t *ring = nullptr;     // [W][ceil(E/32)]
  uint32_t *mask = nullptr;     // [ceil(E/32)] this step's set
  long long *step = nullptr;    // steps recorded
  int *bad = nullptr;           // INT_MAX, or the min out-of-range id of the last step
};
cudaError_t launch_stats_record(const StatsState &st, const int32_t *experts, long long S,
                                cudaStream_t s);

// Epoch slots of the exchange: three, so the dispatch of step s+1 can run
// while step s computes and step s-1's partial sums are still in flight
// (dispatch and combine on different streams); a dispatch into a slot waits
// until every MoE rank's push of the epoch kXferSlots back has landed.
constexpr int kXferSlots = 3;

// Attention <-> MoE exchange (xfer.cu).  Ranks [0, A) own token shards,
// ranks [A, A+M) are MoE instances g = rank - A.  One exchange region per
// rank, identical layout everywhere.
struct XferLayout {
  // flags (u64, epoch-valued): dispatch[A] (rows landed), combine[M] (partial
  // sums landed), route[A] (routing landed; routed transport).
  size_t flag_dispatch_off, flag_combine_off, flag_route_off;
  // x/ex/gw/part/err offsets are slot 0's; slot i (epoch % kXferSlots == i) is
  // + i * slot_stride, so a dispatch can run ahead of the previous steps'
  // combines (dispatch of step s+1 while step s computes and step s-1's
  // partial sums are still being pushed and summed).
  // err[M] = {status, bad expert} of MoE instance g's step, written before its
  // combine flag (a failed MoE step is reported on the attention ranks).
  size_t x_off, ex_off, gw_off, part_off, err_off, slot_stride, bytes;
  long long ta_max;  // largest attention shard
};
XferLayout xfer_layout(int A, int M, long long T_max, int d_h, int k);

// NVLS: XferState::mc.  kXferCE: the P2P broadcast's rows moved by the copy
// engines (cudaMemcpyAsync into the peers' mapped regions, the flag by a
// stream memory write after them), so the dispatch takes no SM time from the
// MoE role's kernels running on the same GPU (colocated boxes).
enum XferTransport { kXferP2P = 0, kXferRouted = 1, kXferCE = 2 };

// Device error words of one rank's exchange endpoint (x.err, int[8]).
enum XferErr {
  kErrTimeout = 0,  // sticky: a bounded wait expired
  kErrStatus = 1,   // sticky: first failed step's status (a remote MoE step's, or this rank's)
  kErrBad = 2,      // sticky: its bad expert id
  kErrSkip = 3,     // + wait kind (0 dispatch, 1 combine, 2 route, 3 slot free): this step's verdict of
                    // that wait, 1 -> the step's later kernels skip their work
  kErrWords = 8
};

struct XferState {
  int rank = -1, world = 0, A = 0, M = 0, d_h = 0, k = 0;
  // first MoE rank: A for a split box; 0 when every rank is both an attention
  // shard owner and an MoE instance (janus_xfer_configure_colocated)
  int moe0 = 0;
  long long T_max = 0;
  unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;
  XferLayout L{};
  void *local = nullptr;              // this rank's exchange region
  std::vector<void *> peer_base;      // every rank's region (mapped), by rank
  std::vector<void *> opened;         // IPC mappings to close
  unsigned *counter = nullptr;        // last-block counters [kinds][kXferSlots] (device)
  int *err = nullptr;                 // XferErr words (device)
  int transport = kXferP2P;
  unsigned long long routed_epoch = 0;  // routed: routing of this epoch already pushed
  unsigned long long slot_epoch = 0;    // the slot-free wait of this epoch already enqueued
  void *slot_stream = nullptr;          // ... on this stream
  // routed transport, attention side: the step's schedule (K1 over every
  // shard's routing) and each owned token's destination-instance mask per
  // epoch slot ([kXferSlots][ta_max])
  janus_assignment rws{};
  uint32_t *dmask = nullptr;
  // colocated routed ranks: the attention role's K1 writes the whole layout of
  // the step per epoch slot, and the rank's MoE role runs on it (one K1 per
  // step per GPU instead of two)
  janus_assignment lay[kXferSlots] = {};
  int32_t *lay_tile[kXferSlots] = {};
  // NVLS multicast transport (mc.cpp): the bulk rows / routing / partial sums
  // go through one multicast object; flags stay in the IPC regions above.
  bool mc = false, mc_bound = false;
  // NVLS combine: false (default) -> the MoE ranks push partial sums point to
  // point (K5 push mode) and the owner adds them; true -> multimem.ld_reduce
  // in the switch.  Measured (profiles/r2): push 27-51 us vs switch 114-127 us
  // at 1A+3E / 4 colocated, c2 shape.
  bool mc_reduce = false;
  unsigned long long mc_handle = 0, mem_handle = 0;  // CUmemGenericAllocationHandle
  unsigned long long mc_va = 0, uc_va = 0;           // multicast / own-backing mappings
  size_t mc_bytes = 0, mc_gran = 0;
  size_t mx_off = 0, mex_off = 0, mgw_off = 0, mpart_off = 0, mslot = 0;  // slot 0; slot i = + i * mslot
  // copy-engine transport: one stream per MoE rank (the copies to different
  // ranks run on different engines at once), forked from / joined into the
  // caller's stream
  std::vector<cudaStream_t> ce_streams;
  std::vector<cudaEvent_t> ce_done;
  cudaEvent_t ce_fork = nullptr;
  // colocated routed MoE role: step s's partial-sum push (K5 + signal) runs on
  // push_stream, beside step s+1's permute and GEMMs (ffn_done / push_done per
  // y buffer (epoch parity) order it after its GEMMs and the GEMMs two steps
  // later after it)
  cudaStream_t push_stream = nullptr;
  cudaEvent_t ffn_done[2] = {nullptr, nullptr}, push_done[2] = {nullptr, nullptr};
  // a colocated rank's two roles run on different streams of one GPU: the MoE
  // role orders itself after its own attention role's dispatch, and the
  // attention role's combine after its own MoE role's signal, by these events
  // (per epoch slot) — it spins only on the other GPUs' flags
  cudaEvent_t own_disp[kXferSlots] = {}, own_sig[kXferSlots] = {};
  // attention ranks: the combine of each epoch slot done (a dispatch into the
  // slot waits for the combine kXferSlots epochs back, whatever stream it ran on)
  cudaEvent_t comb_done[kXferSlots] = {};
  bool local_connect = false;  // every rank in this process (janus_xfer_connect_local)
};
constexpr int kCounterKinds = 2;  // 0: row dispatch, 1: routing push

bool mc_supported(int device);
std::string mc_create(XferState &x, int device, int *fd);  // rank 0
std::string mc_join(XferState &x, int device, int fd);     // other ranks
std::string mc_bind(XferState &x, int device);             // every rank, after all joined
void mc_free(XferState &x, int device);

inline size_t xfer_slot(unsigned long long epoch) { return (size_t)(epoch % kXferSlots); }
// Attention rank: broadcast dispatch — shard rows (+ routing) into every MoE
// rank (P2P) or the multicast mapping (NVLS); flag_dispatch.
cudaError_t launch_dispatch(const XferState &x, const void *d_x, const int32_t *d_ex,
                            const float *d_gw, long long T, unsigned long long epoch,
                            cudaStream_t s);
// Copy-engine broadcast (kXferCE), attention rank: the shard rows (+ routing)
// into every MoE rank's region by cudaMemcpyAsync, then flag_dispatch by
// cuStreamWriteValue64 (ordered after the copies, with a memory barrier).
// Grid cap for an exchange kernel that runs beside this GPU's grouped GEMMs.
int side_grid(long long work);
cudaError_t launch_dispatch_ce(const XferState &x, const void *d_x, const int32_t *d_ex,
                               const float *d_gw, long long T, unsigned long long epoch,
                               cudaStream_t s);
// Routed transport, attention rank: shard routing into every rank; flag_route.
cudaError_t launch_route_push(const XferState &x, const int32_t *d_ex, const float *d_gw,
                              long long T, unsigned long long epoch, cudaStream_t s);
// Routed transport, attention rank: each owned row only to the MoE ranks its
// slots were scheduled on (inst = K1's per-slot instance over the whole step);
// records the destination masks; flag_dispatch.
cudaError_t launch_routed_dispatch(const XferState &x, const void *d_x, const int32_t *inst,
                                   const int32_t *status, long long T, unsigned long long epoch,
                                   cudaStream_t s);
// Wait for flags (kind 0 dispatch, 1 combine, 2 route) of `epoch`; the combine
// wait also collects the MoE ranks' error slots.  Sets err[kErrSkip].
// skip: a flag index not to spin on (a colocated rank's own role: ordered by
// an event instead — no kernel waits on another of the same GPU by spinning)
cudaError_t launch_wait(const XferState &x, int kind, unsigned long long epoch, cudaStream_t s,
                        int skip = -1);
// MoE rank: publish {status} + flag_combine[g] = epoch on every attention rank,
// after this rank's partial sums landed (P2P push, or its multicast backing).
cudaError_t launch_signal_combine(const XferState &x, const int32_t *status,
                                  unsigned long long epoch, cudaStream_t s);
// Attention rank: out = sum over the MoE partials (P2P / routed: fixed
// instance order, fp32; NVLS: switch-reduced).
cudaError_t launch_reduce_partials(const XferState &x, void *d_out, long long Ta,
                                   unsigned long long epoch, cudaStream_t s);
cudaError_t launch_reduce_mc(const XferState &x, void *d_out, long long first, long long Ta,
                             unsigned long long epoch, cudaStream_t s);
// K5 in push mode: where the MoE rank's per-token partial sums go.
PushDst push_dst(const XferState &x, unsigned long long epoch);

}  // namespace janus

struct janus_ctx {
  int device = 0;
  std::string err;
  uint64_t launches = 0;
  cudaStream_t stream = nullptr;  // internal stream for host-API calls

  // replica map (host copies + device tables)
  bool have_map = false;
  std::vector<int32_t> off, hosts, rid, qidx, qbase;
  janus::DevMap dmap;

  // scratch for the host scheduling API (grown on demand)
  int sched_cap = 0;
  int32_t *d_in = nullptr;
  janus_assignment d_out{};
  int32_t *d_status = nullptr;

  // MoE layer
  bool moe_ready = false;
  int d_h = 0, d_e = 0, max_tokens = 0, top_k = 0, instance = -1;
  janus::FfnPlan ffn;
  // DeepSeek-V3-style shared expert (janus_moe_set_shared): a dense SwiGLU over
  // every token, its own GEMM plan over token-ordered rows that K3 also writes
  bool shared = false;
  janus::FfnPlan ffn_shared;
  int32_t *shared_off = nullptr;  // [4] {0, rows}, {0, n-tiles}
  int shared_split = 0;  // 1: every MoE instance takes an even share of the tokens
  janus_assignment ws{};      // device workspace for the layer's assignment
  int32_t *ws_tile_off = nullptr;
  // staging for the host MoE API
  void *d_x = nullptr, *d_outbuf = nullptr;
  int32_t *d_experts = nullptr;
  float *d_gw = nullptr;
  const void *router = nullptr;  // [E][d_h] bf16 (janus_moe_set_router; caller-owned)
  float *gate_xchg = nullptr;    // the gate's split-K exchange buffer (allocated on first use)

  // CUDA-graph replay of the single-GPU layer (janus_moe_layer_async)
  struct GraphKey {
    const void *x, *experts, *gw, *out;
    int T;
    bool operator==(const GraphKey &o) const {
      return x == o.x && experts == o.experts && gw == o.gw && out == o.out && T == o.T;
    }
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    uint64_t kernels;  // kernel nodes in the graph
    uint64_t last_use;
  };
  bool use_graph = true;
  cudaStream_t cap_stream = nullptr;
  std::vector<GraphEntry> graphs;  // small LRU cache (a serving loop rotates few buffers)
  uint64_t graph_clock = 0;

  // pipelined host API (janus_moe_layer_host_async): kHostSets device staging
  // sets; H2D on one stream, the layer on `stream`, D2H on a third, so the
  // copies of neighbouring calls overlap the layer.  A set is busy from its
  // H2D to its D2H (~H2D + layer + D2H), so three sets keep the layer fed.
  static constexpr int kHostSets = 3;
  struct HostPipe {
    bool ready = false;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t h2d_ev[kHostSets] = {}, comp_ev[kHostSets] = {}, free_ev[kHostSets] = {};
    void *x[kHostSets] = {}, *out[kHostSets] = {};
    int32_t *ex[kHostSets] = {};
    float *gw[kHostSets] = {};
    int32_t *sticky = nullptr;  // first failing call's scheduler status (device)
    uint64_t calls = 0;
  } hp;

  // activation statistics (janus_stats_*)
  janus::StatsState stats;

  // attention <-> MoE exchange
  bool xfer_ready = false;
  janus::XferState xfer;

  // instrumentation (janus_profile)
  bool profiling = false;
  std::vector<cudaEvent_t> prof_events;  // 4 per recorded call
  int prof_calls = 0;
};
