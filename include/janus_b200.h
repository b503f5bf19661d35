/*
 * janus_b200.h — C ABI of the B200-native MoE-side hot path of Janus
 * (arXiv 2512.13525): activation-balanced expert scheduling (AEBS), the
 * dispatch layout, the per-GPU SwiGLU expert FFN, combine, and the
 * attention->MoE / MoE->attention exchange inside one NVLink box.
 *
 * Plain C types only (no torch types).  Entry points marked "device" take
 * device pointers and are stream-ordered and asynchronous (no host sync);
 * entry points marked "host" take host buffers and synchronise.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   janus_set_replica_map  <- ReplicaMap + ReplicaMap::validate
 *                             (include/moesim/aebs.hpp:29-38, src/aebs.cpp:49-77)
 *   janus_schedule[_async] <- moesim::schedule / schedule_reference /
 *                             schedule_random (include/moesim/aebs.hpp:63-71,
 *                             src/aebs.cpp:172-262) returning Assignment
 *                             (aebs.hpp:42-50)
 *   janus_moe_layer[_async]<- moe_layer_latency's subject: the MoE layer the
 *                             reference only models (src/latency.cpp:17-32)
 *   janus_moe_layer_latency<- moesim::moe_layer_latency (latency.hpp:34-35)
 *   janus_latency_layer    <- the same, calibrated to the measured layer
 *                             (janus_latency_fit; sim.cpp:193-195 callers)
 *   janus_shard_tokens     <- StepTraffic token ownership (src/comm.cpp:76-81)
 * See INTEGRATION.md for the binding a maintainer adds on the reference side.
 */
#ifndef JANUS_B200_H_
#define JANUS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  JANUS_OK = 0,
  JANUS_EINVAL = 1,          /* ValidationError-class input problem (types.hpp:20-22) */
  JANUS_EUNKNOWN_EXPERT = 2, /* aebs.cpp:22-25 "unknown-expert: ..." */
  JANUS_ECUDA = 3,           /* CUDA runtime/driver failure */
  JANUS_ESTATE = 4,          /* call order: no map / no weights / not reserved */
  JANUS_EUNSUPPORTED = 5,    /* shape outside this build's kernel limits */
  JANUS_EPEER = 6            /* box exchange: a peer rank never published its
                                step (bounded wait expired) or failed it */
} janus_status;

typedef enum {
  JANUS_POLICY_AEBS = 0,   /* schedule() == schedule_reference() outputs */
  JANUS_POLICY_RANDOM = 1  /* schedule_random(seed) */
} janus_policy;

/* Kernel limits of this build. */
#define JANUS_MAX_EXPERTS 1024
#define JANUS_MAX_INSTANCES 1024
#define JANUS_MAX_REPLICAS 8192

typedef struct janus_ctx janus_ctx;

/* One scheduling pass, device side.  Every pointer is a caller-owned device
 * buffer.  The first five are the reference Assignment (aebs.hpp:42-50); the
 * rest are the dispatch layout and may be NULL.
 * status[0] receives JANUS_OK / JANUS_EUNKNOWN_EXPERT, status[1] the bad
 * expert id (the minimum one, as schedule() reports it, aebs.cpp:137-162). */
typedef struct {
  int32_t *instance;        /* [T*k]  instance of each token slot            */
  int32_t *replica;         /* [T*k]  physical replica id of each slot       */
  int32_t *expert_instance; /* [E]    -1 when inactive                       */
  int32_t *load;            /* [N]    activated replicas hosted              */
  int64_t *routed_tokens;   /* [N]    token activations routed               */
  int64_t *expert_tokens;   /* [E]    token activations per expert (opt)     */
  int32_t *slot_row;        /* [T*k]  row of each slot in the dispatch layout */
  int32_t *row_slot;        /* [T*k]  inverse permutation                    */
  int32_t *group_off;       /* [R+1]  row offset of each replica group       */
  int32_t *status;          /* [2]    {status, bad expert}                   */
} janus_assignment;

/* ---- context ------------------------------------------------------------ */
janus_status janus_create(janus_ctx **ctx, int device);
void janus_destroy(janus_ctx *ctx);
/* Last error message of this context, in the reference's wording. */
const char *janus_last_error(const janus_ctx *ctx);
/* Number of kernels this context has launched (instrumentation). */
uint64_t janus_launch_count(const janus_ctx *ctx);

/* ---- replica map (host) ------------------------------------------------- */
/* CSR: hosts[off[e]..off[e+1]) strictly ascending instance ids of expert e,
 * rid[] parallel opaque physical replica ids.  Validated as
 * ReplicaMap::validate (aebs.cpp:49-77), then uploaded once. */
janus_status janus_set_replica_map(janus_ctx *ctx, int num_experts, int num_instances,
                                   int slots_per_instance, const int32_t *off,
                                   const int32_t *hosts, const int32_t *rid);
/* Replica order used by the dispatch layout and the weight store: for each
 * CSR entry p, qidx[p] = flat index of that replica (instance-major, ordered
 * by (replica id, expert) within an instance); qbase[g] = first index of
 * instance g (N+1 entries).  Host buffers. */
janus_status janus_replica_order(const janus_ctx *ctx, int32_t *qidx, int32_t *qbase);

/* ---- scheduler ---------------------------------------------------------- */
/* device: one fused kernel (K1+K2), stream-ordered, no host sync. */
janus_status janus_schedule_async(janus_ctx *ctx, const int32_t *d_experts, int num_tokens,
                                  int top_k, int policy, uint64_t seed,
                                  const janus_assignment *out, void *stream);
/* host: the drop-in for moesim::schedule()/schedule_random().  Host buffers,
 * synchronous.  Returns JANUS_EUNKNOWN_EXPERT with janus_last_error() set to
 * the reference message.  expert_tokens may be NULL. */
janus_status janus_schedule(janus_ctx *ctx, const int32_t *experts, int num_tokens, int top_k,
                            int policy, uint64_t seed, int32_t *instance, int32_t *replica,
                            int32_t *expert_instance, int32_t *load, int64_t *routed_tokens,
                            int64_t *expert_tokens);
/* Median device time (µs, CUDA events, graph-replayed) of `reps` scheduler
 * passes over a device-resident batch. */
janus_status janus_time_schedule(janus_ctx *ctx, const int32_t *d_experts, int num_tokens,
                                 int top_k, int policy, int reps, double *median_us);

/* ---- MoE layer ---------------------------------------------------------- */
/* Expert FFN shape (SwiGLU, bf16 weights, fp32 accumulate) and the largest
 * step this context must hold (allocates workspace). */
janus_status janus_moe_configure(janus_ctx *ctx, int d_hidden, int d_expert, int max_tokens,
                                 int top_k);
/* Weight store of the local instance `instance` (or -1: this GPU holds every
 * instance's replicas): device bf16 buffers in replica order (qidx, qbase)
 *   w13: [Q][2*d_expert][d_hidden]  rows 0..d_e-1 gate, d_e..2d_e-1 up
 *   w2 : [Q][d_hidden][d_expert]    down projection
 * Q = replicas hosted (qbase[g+1]-qbase[g], or R).  Not copied: must outlive
 * the context. */
janus_status janus_moe_set_weights(janus_ctx *ctx, int instance, const void *d_w13,
                                   const void *d_w2);
/* device: K1 schedule -> K3 permute -> K4 grouped SwiGLU GEMMs -> K5 combine.
 *   x [T][d_h] bf16, experts [T*k] int32, gate_w [T*k] fp32, out [T][d_h] bf16.
 * With a single-instance weight store (instance >= 0) out receives this
 * instance's partial sum (tokens routed elsewhere contribute 0).
 * If `assign` is non-NULL the scheduling outputs are also written there. */
/* DeepSeek-V3-style shared expert (one expert on every
 * token, weight 1, added after the routed slots): w13 [2*d_e][d_h] = [Wg; Wu],
 * w2 [d_h][d_e], bf16, caller-owned; NULL disables.  Computed by the
 * single-GPU layer, and by MoE instance 0 of a box (NVLS transport). */
janus_status janus_moe_set_shared(janus_ctx *ctx, const void *d_w13, const void *d_w2);
/* Shared expert placement in a box: 0 (default) = MoE instance 0 runs it on
 * every token; 1 = every MoE instance runs it on an even share of the step's
 * tokens (instance g of N: [g*(T/N) + min(g, T%N), +T/N + (g < T%N)) — the
 * same split as the attention shards), so no instance straggles by a dense
 * FFN over the whole step.  Set the weights on every MoE instance for 1. */
janus_status janus_moe_set_shared_split(janus_ctx *ctx, int split);
janus_status janus_moe_layer_async(janus_ctx *ctx, const void *d_x, const int32_t *d_experts,
                                   const float *d_gate_w, int num_tokens, void *d_out,
                                   const janus_assignment *assign, void *stream);
/* host: end to end from (pinned) host buffers: H2D, layer, D2H, sync. */
janus_status janus_moe_layer(janus_ctx *ctx, const void *x, const int32_t *experts,
                             const float *gate_w, int num_tokens, void *out);

/* ---- instrumentation ---------------------------------------------------- */
/* host, pipelined: janus_moe_layer with the copies of neighbouring calls
 * overlapped — H2D of call i+1 and D2H of call i-1 run on their own streams
 * (pinned host buffers needed for overlap) while call i's layer runs.  Returns
 * once enqueued; the caller must keep the host buffers alive and not reuse
 * `out` / refill the inputs of a call until janus_moe_host_sync.  Errors of the scheduled batches (unknown
 * expert) are reported by janus_moe_host_sync. */
janus_status janus_moe_layer_host_async(janus_ctx *ctx, const void *x, const int32_t *experts,
                                        const float *gate_w, int num_tokens, void *out);
janus_status janus_moe_host_sync(janus_ctx *ctx);
/* While enabled, every janus_moe_layer_async call records CUDA events on its
 * stream around the scheduler kernel (K1+K2) and around the grouped GEMMs (K4).
 * janus_profile_read synchronises, returns the summed device times (ms) and
 * the number of layer calls recorded, and resets. */
janus_status janus_profile(janus_ctx *ctx, int enable);
janus_status janus_profile_read(janus_ctx *ctx, double *sched_ms, double *ffn_ms, int *calls);
/* One scheduler pass over a device batch with in-kernel phase timestamps
 * (%globaltimer, ns): ns[0..6] = start, loads issued + map staged, pass 1,
 * scan + pins, sequential greedy, finish + scans, pass 2; ns[7] = SM clock
 * cycles of the pass where recorded (the decode-size kernel), else 0.
 * ns has 8 entries. */
janus_status janus_trace_schedule(janus_ctx *ctx, const int32_t *d_experts, int num_tokens,
                                  int top_k, int64_t *ns);
/* Debug: the grouped GEMMs' tile timeline.  With JANUS_GEMM_TRACE=1 in the
 * environment when the layer is configured, every tile stamps %globaltimer
 * (draw, MMA start, accumulator ready, epilogue done, producer waits, ...) and
 * CTA 0 its stages; this copies [2 GEMMs][16384 tiles][16] u64 to host and
 * clears them (tools/gemm_timeline.py reads it).  Returns 0, or 4 when the
 * trace was not enabled, 3 on a CUDA error. */
int janus_debug_ffn_trace(unsigned long long *host, int cap_words);

/* ---- MoE-side gating ------------------------------------ */
/* Janus gates on the MoE side; the reference only consumes
 * top-k ids (ActivationBatch, aebs.hpp:15-24).  device: logits = x · Wrᵀ
 * (x [T][d_h] bf16, Wr [E][d_h] bf16, fp32 accumulation on tcgen05), top-k ids
 * by descending logit — ties to the lower id — into experts [T*k] in rank
 * order, softmax of the k selected logits into gate_w [T*k].
 * Needs d_h % 64 == 0, E % 16 == 0, 16 <= E <= 256, 1 <= k <= min(16, E). */
janus_status janus_gate_async(janus_ctx *ctx, const void *d_x, const void *d_router, int64_t T,
                              int d_hidden, int num_experts, int top_k, int32_t *d_experts,
                              float *d_gate_w, void *stream);
/* Router weights [E][d_h] bf16 for janus_moe_layer_gated_async (device
 * pointer, caller-owned; E from the replica map, d_h / k from
 * janus_moe_configure). */
janus_status janus_moe_set_router(janus_ctx *ctx, const void *d_router);
/* device: the gating kernel on this GPU, then janus_moe_layer_async on its
 * ids and weights (kept in the context's workspace). */
janus_status janus_moe_layer_gated_async(janus_ctx *ctx, const void *d_x, int num_tokens,
                                         void *d_out, void *stream);

/* ---- activation statistics ------------------------------ */
/* ActivationStats (experts.hpp:18-43, experts.cpp:11-62) on the device:
 * per-expert activation counts and the symmetric co-activation matrix over the
 * last `window` steps.  Configure allocates and zeroes the state (errors as
 * the reference's constructor). */
janus_status janus_stats_configure(janus_ctx *ctx, int num_experts, int window);
/* device: record_step for the activated set of one step's routing (the
 * distinct ids of experts[T*k]).  An id outside [0, E) rejects the step (state
 * unchanged, janus_stats_status reports it) — the reference's
 * "stats: activated expert X out of range". */
janus_status janus_stats_record_async(janus_ctx *ctx, const int32_t *d_experts, int64_t num_tokens,
                                      int top_k, void *stream);
/* host (synchronises the context's device): counts [E], coact [E*E] (zero
 * diagonal), steps recorded in the window (reference recorded_steps()). */
janus_status janus_stats_read(janus_ctx *ctx, int64_t *counts, int64_t *coact, int *recorded);
/* host: the last recorded step's verdict: JANUS_OK, or JANUS_EINVAL with the
 * reference message in janus_last_error (bad_expert = the offending id). */
janus_status janus_stats_status(janus_ctx *ctx, int *bad_expert);

/* ---- attention <-> MoE exchange (one NVLink box) ------------------------ */
/* Token ownership on the attention side: even split, remainder to the lowest
 * ids (comm.cpp:76-81).  Writes first token and count of shard a. */
void janus_shard_tokens(int64_t num_tokens, int attn_instances, int a, int64_t *first,
                        int64_t *count);
/* One process per GPU.  Ranks [0, n_attn) own token shards (attention side),
 * ranks [n_attn, n_attn + n_moe) are MoE instances g = rank - n_attn (their
 * context holds the replica map and instance g's weight store).  Every rank
 * allocates one exchange region (identical layout) and exports it; each rank
 * then maps all peers' regions (CUDA IPC over NVLink P2P). */
janus_status janus_xfer_configure(janus_ctx *ctx, int n_attn, int n_moe, int rank,
                                  int max_tokens, int d_hidden, int top_k);
/* The MoE-only box (SURVEY §8(e) "c4 N=4 MoE-only"): all n ranks own a token
 * shard AND are MoE instances g = rank; every dispatch / MoE / combine call
 * below is then legal on every rank. */
janus_status janus_xfer_configure_colocated(janus_ctx *ctx, int n, int rank, int max_tokens,
                                            int d_hidden, int top_k);
janus_status janus_xfer_handle(const janus_ctx *ctx, uint8_t *handle /* 64 bytes */);
janus_status janus_xfer_connect(janus_ctx *ctx, const uint8_t *handles /* world x 64, by rank */);
/* device, attention rank a: push this rank's shard (janus_shard_tokens of the
 * step's num_tokens) — rows x [T_a][d_h] bf16, experts / gate_w [T_a*k] — into
 * every MoE rank, then publish `epoch` (> 0, increasing per step).  Three
 * epoch slots: call janus_attn_combine_async(epoch - 3) (and, colocated, the
 * MoE step of epoch - 3) before this; the dispatch then waits on the device
 * until that step is done everywhere, so dispatch and combine may use
 * different streams.  With both
 * routing pointers NULL only the rows move: the MoE ranks gate themselves
 * (janus_moe_set_router on their contexts; Janus gates on the MoE side,
 * PAPER.md:671-678). */
janus_status janus_attn_dispatch_async(janus_ctx *ctx, const void *d_x, const int32_t *d_experts,
                                       const float *d_gate_w, int64_t num_tokens, uint64_t epoch,
                                       void *stream);
/* device, attention rank, routed transport only (optional): the routing phase
 * of janus_attn_dispatch_async alone — this shard's ids and gate weights into
 * every rank, flag.  A later dispatch of the same epoch then skips it; callers
 * that drive several ranks from one stream call it on every attention rank
 * first (each dispatch waits for every shard's routing). */
janus_status janus_attn_route_async(janus_ctx *ctx, const int32_t *d_experts, const float *d_gate_w,
                                    int64_t num_tokens, uint64_t epoch, void *stream);
/* device, MoE rank: wait for every shard of `epoch`, run K1-K4 on the received
 * step, and push this instance's per-token partial sums to their owners. */
janus_status janus_moe_layer_xfer_async(janus_ctx *ctx, int64_t num_tokens, uint64_t epoch,
                                        void *stream);
/* device, attention rank: wait for every MoE partial of `epoch` and reduce
 * them (instance order, fp32) into out [T_a][d_h] bf16. */
janus_status janus_attn_combine_async(janus_ctx *ctx, void *d_out, int64_t num_tokens,
                                      uint64_t epoch, void *stream);
/* host: 1 if a wait exceeded its bound (a peer never published). */
janus_status janus_xfer_status(janus_ctx *ctx, int *timed_out);
/* host (synchronises the device): the first failed step this rank saw since
 * the last check — its own, or on the attention side any MoE rank's (each MoE
 * rank publishes its scheduler status with its combine flag).  JANUS_OK,
 * JANUS_EUNKNOWN_EXPERT with the reference message in janus_last_error
 * (aebs.cpp:22-25), or JANUS_EPEER (a bounded wait expired).  A failed step's
 * later kernels skip their work; the owners' output rows of it are zeros. */
janus_status janus_xfer_check(janus_ctx *ctx);
/* Instrumentation: device address of this rank's received token rows
 * [max_tokens][d_h] bf16 in epoch's slot (MoE ranks: the dispatch target). */
janus_status janus_xfer_recv_rows(const janus_ctx *ctx, uint64_t epoch, void **rows);
/* NVLS transport's combine, on every rank: 0 (default) = each MoE rank
 * pushes its partial sums point to point into the owners' regions and the
 * owner adds them in instance order; 1 = the owner reads them summed by the
 * NVSwitch (multimem.ld_reduce).  The dispatch stays multicast either way. */
janus_status janus_xfer_set_combine(janus_ctx *ctx, int switch_reduce);
/* Bound of every flag wait of this endpoint (default 20 s). */
janus_status janus_xfer_set_timeout(janus_ctx *ctx, uint64_t timeout_ns);
/* Same-process connect (all ranks' contexts in one process, on one or several
 * devices): peers[r] = rank r's context, configured for the same box; replaces
 * the IPC handle exchange.  Kernels that wait on one another must then still
 * be enqueued in causal order (a rank's wait only after its producers). */
janus_status janus_xfer_connect_local(janus_ctx *ctx, janus_ctx *const *peers);
/* Transport (0: broadcast by SM peer stores, the default; 1: routed; 2:
 * broadcast by the copy engines), after configure, on every rank.  Copy
 * engine: the P2P broadcast's rows and routing go by cudaMemcpyAsync into the
 * MoE ranks' mapped regions and flag_dispatch by a stream memory write after
 * them — no dispatch kernel, so a colocated rank's MoE kernels keep every SM.
 * Routed: each attention rank ships its shard's routing to every
 * rank, runs the scheduler over the whole step (identical to the MoE ranks'),
 * and sends each row only to the MoE ranks its slots were scheduled on
 * (north_star's per-GPU buffers; StepTraffic, comm.hpp:20-39); each MoE rank
 * pushes partial sums only for the tokens it computed.  Needs the replica map
 * on the attention ranks' contexts too (janus_set_replica_map), routing shipped
 * (no MoE-side gating) and no shared expert; point to point only (no NVLS). */
janus_status janus_xfer_set_transport(janus_ctx *ctx, int transport);
/* NVLS multicast transport (optional, after janus_xfer_connect on every rank):
 * rows, routing and partial sums then move through one NVSwitch multicast
 * object — dispatch leaves an attention GPU once instead of once per MoE GPU,
 * and the combine's sum over MoE GPUs is done by the switch
 * (multimem.ld_reduce).  Rank 0 creates it and exports a POSIX fd, which the
 * caller passes to every other rank (e.g. SCM_RIGHTS); each other rank joins
 * with it; after all ranks joined, every rank binds its backing.  Flags keep
 * using the IPC regions.  Without this call sequence the P2P path is used. */
janus_status janus_xfer_mc_supported(janus_ctx *ctx, int *yes);
janus_status janus_xfer_mc_create(janus_ctx *ctx, int *fd);
janus_status janus_xfer_mc_join(janus_ctx *ctx, int fd);
janus_status janus_xfer_mc_bind(janus_ctx *ctx);

/* ---- model / workload --------------------------------------------------- */
/* The MoE-layer latency model, calibrated.  The reference
 * prices an instance as t_launch + max(A*W_e/beta, F(b)/pi) with
 * W_e = 2*d_h*d_e*bpp and F(b) = 2*b*d_h*d_e (latency.cpp:17-24, types.hpp:42-44)
 * and a layer as the max over instances with work (latency.cpp:26-32).  This
 * model generalises it:
 *   t = t_launch + (mem^p + comp^p)^(1/p),
 *   mem = A * matrices*d_h*d_e*bytes_per_param / hbm_bandwidth,
 *   comp = b * 2*flop_matrices*d_h*d_e / peak_flops;
 * p <= 0 is the reference's max, matrices = 2 / flop_matrices = 1 its
 * accounting (3 / 3: the SwiGLU expert this library computes).  Units:
 * seconds, B/s, FLOP/s. */
typedef struct {
  double t_launch;
  double hbm_bandwidth;
  double peak_flops;
  double p;
  int matrices;        /* weight matrices streamed per activated expert */
  int bytes_per_param;
  int flop_matrices;   /* matrices multiplied per routed row */
} janus_latency_model;
/* One instance with `activated_experts` replicas and `routed_tokens` rows
 * (0 when it has none); a layer: the max over instances with load > 0 — the
 * replacement for moe_instance_latency / moe_layer_latency that
 * DecodeEngine::eval_step calls (sim.cpp:193-195). */
double janus_latency_instance(const janus_latency_model *m, int activated_experts,
                              int64_t routed_tokens, int d_hidden, int d_expert);
double janus_latency_layer(const janus_latency_model *m, int num_instances, const int32_t *load,
                           const int64_t *routed_tokens, int d_hidden, int d_expert);
/* host: fit t_launch, hbm_bandwidth, peak_flops and p (> 1) to n >= 4 measured
 * points (activated experts, routed rows, seconds) — minimum mean squared
 * relative error; `model` gives the start (and matrices / bytes_per_param,
 * kept) and receives the fit; mean_abs_rel_err (optional) its residual. */
janus_status janus_latency_fit(int n, const int32_t *activated, const int64_t *routed_tokens,
                               const double *seconds, int d_hidden, int d_expert,
                               janus_latency_model *model, double *mean_abs_rel_err);
/* The reference roofline prediction (latency.cpp:17-32), kept for comparison
 * with measured layer times. */
double janus_moe_layer_latency(int num_instances, const int32_t *load,
                               const int64_t *routed_tokens, int d_hidden, int d_expert,
                               int bytes_per_param, double peak_flops, double hbm_bandwidth,
                               double t_launch);
/* derive_seed (rng.hpp:34-44): the seed of schedule_random and of the
 * synthetic weights.  (Synthetic routing, gen_batch, is test infrastructure:
 * oracle/routing.py — not part of this library.) */
uint64_t janus_derive_seed(uint64_t root, const char *label, uint64_t extra);

#ifdef __cplusplus
}
#endif
#endif /* JANUS_B200_H_ */
