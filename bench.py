"""Benchmark: MoE-layer tokens/s/GPU + scheduler µs/iter (Qwen3-MoE shape) on B200.

Contract (see task spec): one JSON line on rank 0.
  python bench.py [--gpus N] [--steps K] [--warmup W] [--tokens T] [--impl ours|reference]

Workload (BASELINE.json configs[1], "c2"): Qwen3-30B-A3B-shaped MoE layer —
128 experts, top-8, d_h=2048, d_e=768, SwiGLU, bf16 random-init weights, the
committed c2 replica map (N=1, reference placement pipeline), Zipf(1.0)
routing from the reference's own gen_batch (oracle/_ref; seed 0x30).  One step
= one MoE layer over one batch of T tokens: K1 schedule + K3 permute + K4
grouped GEMMs + K5 combine.  The weight store (1.21 GB) is far larger than L2,
so every step streams it from HBM.

Under torchrun (N > 1) the ranks form one NVLink box (BoxPlan.for_gpus: 1A+1E,
1A+3E, 2A+6E): attention GPUs dispatch their token shards to the MoE GPUs and
combine the partial sums.  ``value`` is the whole job's
tokens/s over all N GPUs (the contract's aggregate; metric
"moe_layer_tokens_per_s"); BASELINE's per-GPU figure is the side field
``tokens_per_s_per_gpu`` (= value / N), the per-MoE-GPU one
another.

Input generation (routing batches) is test infrastructure — the reference's
gen_batch through oracle/_ref, or the pinned oracle restatement — and runs
outside every timed region.

``--impl reference`` times the reference's CPU path on the host cores without
importing this package: the reference's own schedule() and
schedule_reference() (oracle/_ref, compiled from /root/reference) on the same
batches, plus a CPU SwiGLU FFN from the build's parity oracle (the reference
has no FFN; labelled "build_oracle"), and the reference's moe_layer_latency
model (latency.cpp:17-32) beside it, labelled modelled.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E, K_TOP, D_H, D_E = 128, 8, 2048, 768
SEED = 0x30
MAP = "c2"
SHARED = False
SHAPE_NAME = "c2: Qwen3-30B-A3B-shaped MoE layer (128 experts, top-8, d_h=2048, d_e=768, SwiGLU)"
N_BATCHES = 8  # distinct routing batches rotated through the timed steps
# `value` is the whole job (all N GPUs); BASELINE's tokens/s/GPU is a side field
METRIC = "moe_layer_tokens_per_s"
METRIC_NOTE = ("whole-job MoE-layer tokens/s over all n_gpus; BASELINE's MoE-layer "
               "tokens/s/GPU is tokens_per_s_per_gpu = value / n_gpus")

# --shape: the BASELINE configs' expert shapes (the default c2 is the headline;
# the others are reported in profiles/, not the driver's scaling line)
SHAPES = {
    "c2": (128, 8, 2048, 768, 0x30, "c2", False, SHAPE_NAME),
    "c3": (128, 8, 4096, 1536, 0x235, "c3", False,
           "c3: Qwen3-235B-A22B-shaped MoE layer (128 experts, top-8, d_h=4096, d_e=1536)"),
    "c4": (256, 8, 7168, 2048, 0xD5, "c4", True,
           "c4: DeepSeek-V3-shaped MoE layer (256 routed experts + 1 shared, top-8, d_h=7168, "
           "d_e=2048)"),
}


def apply_shape(name):
    global E, K_TOP, D_H, D_E, SEED, MAP, SHARED, SHAPE_NAME
    E, K_TOP, D_H, D_E, SEED, MAP, SHARED, SHAPE_NAME = SHAPES[name]


def shape_map(J, M):
    """Replica map for M MoE instances of the current shape."""
    if MAP == "c2":
        return J.config_map("c2" if M == 1 else f"c2_m{M}"), f"c2{'' if M == 1 else f'_m{M}'}"
    if MAP == "c3":
        return J.config_map(f"c3_m{M}"), f"c3_m{M}"
    if M == 1:  # c4 on one GPU: every expert local
        return J.ReplicaMap.from_hosts(1, E, [[0]] * E), "one replica per expert"
    return J.config_map(f"c4_n{M}"), f"c4_n{M}"


def set_shared_expert(layer, dev, split=False):
    """split (box): every MoE instance runs the shared expert on its even share
    of the tokens (janus_moe_set_shared_split) instead of instance 0 on all."""
    if SHARED and (split or layer.instance <= 0):
        import torch
        from paper_2512_13525_b200.moe import expert_weights
        wg, wu, wd = expert_weights(E, D_H, D_E, 1, dev)
        layer.set_shared(torch.cat([wg, wu]).contiguous(), wd.contiguous(), split=split)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.05)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        pw = []
        for r in self.rows:
            try:
                pw.append(float(r[2]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w": float(np.median(pw)) if pw else None,  # instantaneous draw
                "power_max_w": max(pw) if pw else None,
                "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_mod():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    return oracle


def gen_batches(T, n=N_BATCHES, E_=None, s=1.0, seed=None, k=None):
    """Routing batches (input generation, never timed): the reference's own
    gen_batch from_pmf(1/(e+1)^s) (oracle/_ref) when built, else the pinned
    oracle restatement (bit-identical, tests/test_oracle_vs_ref.py)."""
    o = oracle_mod()
    E_ = E if E_ is None else E_
    k = K_TOP if k is None else k
    seed = SEED if seed is None else seed
    w = np.array([1.0 / (e + 1) ** s for e in range(E_)])
    try:
        ref = o.Ref()
        return [ref.gen_batch("pmf", E_, T, k, seed, T * 1000 + i, weights=w) for i in range(n)]
    except FileNotFoundError:
        orc = o.Oracle()
        _, cdf = orc.pattern("pmf", E_, weights=w)
        return [orc.gen_batch(cdf, T, k, seed, T * 1000 + i) for i in range(n)]


def csr_map(name):
    """A committed config map as the oracle's CSRMap (no product import)."""
    o = oracle_mod()
    return o.CSRMap.from_map_text(open(os.path.join(ROOT, "paper_2512_13525_b200", "maps",
                                                   f"{name}.map")).read())


def map_name(M):
    if MAP == "c2":
        return "c2" if M == 1 else f"c2_m{M}"
    if MAP == "c3":
        return f"c3_m{M}"
    return None if M == 1 else f"c4_n{M}"


def cpu_map(M=1):
    o = oracle_mod()
    name = map_name(M)
    if name is None:  # c4 on one GPU: every expert local
        return o.CSRMap.from_lists(1, E, [[0]] * E)
    return csr_map(name)


def cpu_weights_fn():
    """Deterministic CPU-side bf16 expert weights for the CPU sample (numbers
    only need the right shape)."""
    o = oracle_mod()
    orc = o.Oracle()
    cache = {}

    def fn(e):
        if e not in cache:
            r = np.random.default_rng(e)
            cache[e] = tuple(orc.f32_to_bf16(r.standard_normal(sh).astype(np.float32) * sc)
                             for sh, sc in (((D_E, D_H), D_H ** -0.5), ((D_E, D_H), D_H ** -0.5),
                                            ((D_H, D_E), D_E ** -0.5)))
        return cache[e]
    return fn


def cpu_sample(T, tokens_sample, batches, wfn, nthreads, hbm, tf_sus):
    """The CPU side of the path on a bounded sample, every piece labelled:
      * the reference's schedule() (4-thread OMP team as shipped) and
        schedule_reference() (1 core) on the full batches — oracle/_ref;
      * a CPU SwiGLU FFN for `tokens_sample` tokens' top-k rows — the build's
        parity oracle (the reference has no FFN): kind "build_oracle";
      * the reference's moe_layer_latency model (latency.cpp:17-32) on the
        same schedule at the measured B200 peaks: kind "modelled".
    Returns the composite tokens/s (reference schedule() + build-oracle FFN,
    pro-rated to the sample) and the components."""
    o = oracle_mod()
    ref, orc = o.Ref(), o.Oracle()
    m = cpu_map(1)
    allb = np.concatenate(batches)
    t_sched = ref.time_schedule(allb, T, K_TOP, m, "schedule", reps=21) * 1e-6
    t_sched_ref = ref.time_schedule(allb, T, K_TOP, m, "reference", reps=21) * 1e-6
    a0 = ref.schedule(batches[0], T, K_TOP, m, "schedule")
    # the model as shipped (2 matrices) at the measured peaks, t_launch 5 us
    t_model = ref.moe_layer_latency(a0.load, a0.routed_tokens, D_H, D_E, 2, tf_sus * 1e12,
                                    hbm * 1e9, 5e-6)
    ex = batches[0].reshape(T, K_TOP)[:tokens_sample]
    by_e = {}
    for t in range(tokens_sample):
        for j in range(K_TOP):
            by_e.setdefault(int(ex[t, j]), []).append(t)
    rng = np.random.default_rng(0)
    xu = orc.f32_to_bf16(rng.standard_normal((tokens_sample, D_H)).astype(np.float32))
    ws_ = {e: wfn(e) for e in by_e}  # weight generation outside the timing
    t0 = time.perf_counter()
    for e, toks in by_e.items():
        wg, wu, wd = ws_[e]
        orc.expert_swiglu(xu[toks], wg, wu, wd, round_h=True, nthreads=nthreads)
    t_ffn = time.perf_counter() - t0
    t_step_sample = t_ffn + t_sched * tokens_sample / T
    comp = [
        {"name": "schedule()", "kind": "reference", "source": "oracle/_ref (aebs.cpp:172-197)",
         "us_per_call": t_sched * 1e6, "cores": 4, "tokens": T},
        {"name": "schedule_reference()", "kind": "reference",
         "source": "oracle/_ref (aebs.cpp:199-248)", "us_per_call": t_sched_ref * 1e6, "cores": 1,
         "tokens": T},
        {"name": "fp32 SwiGLU expert FFN", "kind": "build_oracle",
         "source": "oracle/oracle.c or_expert_swiglu (build oracle, not reference: the "
                   "reference has no FFN)", "seconds": t_ffn, "cores": nthreads,
         "tokens": tokens_sample, "tokens_per_s": tokens_sample / t_ffn},
        {"name": "moe_layer_latency", "kind": "modelled",
         "source": "oracle/_ref latency.cpp:17-32 at the measured peaks (HBM "
                   f"{hbm:.1f} GB/s, bf16 {tf_sus:.1f} TFLOP/s), t_launch 5 us; 2 matrices, "
                   "2 FLOP per (token, d_h, d_e) as shipped",
         "us_per_layer": t_model * 1e6, "tokens_per_s": T / t_model},
    ]
    return {"tok_s": tokens_sample / t_step_sample, "t_sched_us": t_sched * 1e6,
            "t_sched_reference_us": t_sched_ref * 1e6, "components": comp,
            "sample_tokens": tokens_sample}


def c5_scheduler_cpu(tokens=(32, 256, 4096)):
    """BASELINE c5 (E=256, N=6, Zipf 1.2, seed 0x5A): the reference's
    schedule() / schedule_reference() µs and AEBS vs random max-load, on the
    host cores (oracle/_ref)."""
    o = oracle_mod()
    ref = o.Ref()
    m = csr_map("c5")
    rows = {}
    for T in tokens:
        b = gen_batches(T, 1, 256, 1.2, 0x5A)[0]
        a = ref.schedule(b, T, 8, m, "schedule")
        r = ref.schedule(b, T, 8, m, "random", seed=7)
        rows[T] = {"cpu_schedule_us": ref.time_schedule(b, T, 8, m, "schedule", reps=101),
                   "cpu_schedule_reference_us": ref.time_schedule(b, T, 8, m, "reference",
                                                                  reps=101),
                   "max_load_aebs": int(a.load.max()), "max_load_random": int(r.load.max()),
                   "batch": b}
    return rows


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    T = args.tokens
    batches = gen_batches(T)
    nthreads = os.cpu_count() or 1
    wfn = cpu_weights_fn()
    hbm, tf_burst, tf_sus, src = peaks()
    sample = max(1, min(T, args.cpu_sample_tokens))
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(T, sample, batches, wfn, nthreads, hbm, tf_sus or tf_burst)
        if i >= args.warmup:
            vals.append(r)
    tok_s = float(np.median([v["tok_s"] for v in vals]))
    c5 = c5_scheduler_cpu()
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s,
        "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": workload_config(T, args),
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": nthreads, "kind": "port",
                         "sample": f"reference schedule() (oracle/_ref, 4-thread OMP team as "
                                   f"shipped) on the full T={T} batch, pro-rated, + the build "
                                   f"oracle's fp32 SwiGLU FFN (the reference has no FFN) for "
                                   f"{sample} tokens x top-8 rows on {nthreads} threads",
                         "components": vals[-1]["components"]},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "scheduler": {"cpu_schedule_us": float(np.median([v["t_sched_us"] for v in vals])),
                      "cpu_schedule_reference_us": float(np.median(
                          [v["t_sched_reference_us"] for v in vals])),
                      "c5": {str(t): {k_: v_ for k_, v_ in r.items() if k_ != "batch"}
                             for t, r in c5.items()}},
        "imports_product": "paper_2512_13525_b200" in sys.modules,
    }
    print(json.dumps(line), flush=True)


def workload_config(T, args):
    wbytes = E * 3 * D_H * D_E * 2 + (3 * D_H * D_E * 2 if SHARED else 0)
    return {"workload": SHAPE_NAME + " on 1 B200 per rank: AEBS scheduler + grouped FFN",
            "tokens_per_step": T, "experts": E, "top_k": K_TOP, "d_hidden": D_H,
            "d_expert": D_E, "shared_expert": SHARED,
            "routing": f"Zipf s=1.0 via gen_batch, seed {SEED:#x}",
            "replica_map": f"{shape_map_name(1)} (reference placement pipeline)",
            "l2": f"inputs > L2: {wbytes / 1e9:.2f} GB expert weights streamed from HBM every step",
            "parallelism": f"replicas x{args.gpus}"}


def shape_map_name(M):
    return {"c2": "maps/c2.map" if M == 1 else f"maps/c2_m{M}.map", "c3": f"maps/c3_m{M}.map",
            "c4": "one replica per expert" if M == 1 else f"maps/c4_n{M}.map"}[MAP]


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2512_13525_b200 as J
    from paper_2512_13525_b200._lib import lib
    from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    T = args.tokens

    rmap, _ = shape_map(J, 1)
    layer = MoELayer(rmap, D_H, D_E, T, K_TOP, instance=-1, device=local)
    set_shared_expert(layer, dev)
    w13, w2 = build_weight_store(layer, seed=1)
    layer.set_weights(w13, w2)
    batches = [torch.from_numpy(b).to(dev) for b in gen_batches(T)]
    x, gw = make_inputs(T, K_TOP, D_H, 3, dev)
    out = torch.empty_like(x)

    # algorithmic bytes / flops of the grouped GEMMs for each batch
    sched = layer.sched
    alg_bytes, alg_flops = [], []
    for b in gen_batches(T):
        a = sched.schedule(J.ActivationBatch(T, K_TOP, b))
        A = int((a.expert_instance >= 0).sum())
        rows = T * K_TOP
        if SHARED:  # the shared expert: one more weight set, T more rows
            A, rows = A + 1, rows + T
        alg_bytes.append(A * 3 * D_H * D_E * 2 + rows * (D_H + D_E) * 2 * 2)
        alg_flops.append(6.0 * D_H * D_E * rows)

    def step(i):
        layer.forward(x, batches[i % N_BATCHES], gw, out=out)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches0 = layer.launches()
    s = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # timed region: the layer as a serving loop runs it (CUDA-graph replay of
    # the five kernels, one graph per routing buffer)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(s)
        for i in range(args.steps):
            step(i)
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = layer.launches() - launches0
    # second timed pass, launched without the graph so the library can record
    # CUDA events on its launch stream around the scheduler and the grouped
    # GEMMs of every step (events cannot be re-armed per step inside a replay)
    import ctypes as C
    lib.janus_profile(layer.ctx, 1)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(s)
    for i in range(args.steps):
        step(i)
    f1.record(s)
    torch.cuda.synchronize()
    ms_nograph = f0.elapsed_time(f1)
    sched_ms, ffn_ms, calls = C.c_double(), C.c_double(), C.c_int()
    lib.janus_profile_read(layer.ctx, C.byref(sched_ms), C.byref(ffn_ms), C.byref(calls))
    lib.janus_profile(layer.ctx, 0)
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = T * args.steps * ws / (ms / 1e3)

    # e2e through the public host API: pinned host buffers, H2D + layer + D2H each step
    xh = x.cpu().pin_memory()
    gh = gw.cpu().pin_memory()
    bh = [b.cpu().pin_memory() for b in batches]
    oh = torch.empty(T, D_H, dtype=torch.bfloat16).pin_memory()
    # the same host<->device copies without the layer (3 device buffer sets,
    # one stream per direction, as janus_moe_layer_host_async issues them): the
    # host link's ceiling for e2e — the copies of a step outlast its layer
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    xs = [torch.empty_like(x) for _ in range(3)]
    bs = [torch.empty_like(batches[0]) for _ in range(3)]
    gs = [torch.empty_like(gw) for _ in range(3)]

    # pipelined host API (janus_moe_layer_host_async): every step still copies
    # its inputs in and its output out, but the copies of neighbouring steps
    # overlap the layer on separate streams
    def e2e_pass():
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            layer.forward_host_async(xh, bh[i % N_BATCHES], gh, oh)
        layer.host_sync()
        e = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([e], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e = float(t.item())
        return e

    def copies_pass():
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        for i in range(args.steps):
            k = i % 3
            with torch.cuda.stream(h2d_s):
                xs[k].copy_(xh, non_blocking=True)
                bs[k].copy_(bh[i % N_BATCHES], non_blocking=True)
                gs[k].copy_(gh, non_blocking=True)
            with torch.cuda.stream(d2h_s):
                oh.copy_(xs[(k + 1) % 3], non_blocking=True)
        torch.cuda.synchronize()
        return time.perf_counter() - c0

    for i in range(max(1, args.warmup)):
        layer.forward_host_async(xh, bh[i % N_BATCHES], gh, oh)
    layer.host_sync()
    # three passes of K steps each, alternating with the copies-only passes:
    # the pinned-host link of a shared host varies by +-20 % within seconds
    # (measured, profiles/README.md), so the median pass of each is reported
    e2e_runs, copies_runs = [], []
    for _ in range(3):
        e2e_runs.append(e2e_pass())
        copies_runs.append(copies_pass())
    e2e_s, copies_s = float(np.median(e2e_runs)), float(np.median(copies_runs))
    e2e_val = T * args.steps * ws / e2e_s
    del xs, bs, gs

    # scheduler µs/iter (graph-replayed) on the same batch
    sched_us = sched.time_schedule(batches[0], T, K_TOP, reps=51)

    hbm, tf_burst, tf_sus, src = peaks()
    ffn_s = ffn_ms.value / 1e3 / max(calls.value, 1)
    bytes_avg = float(np.mean([alg_bytes[i % N_BATCHES] for i in range(args.steps)]))
    flops_avg = float(np.mean([alg_flops[i % N_BATCHES] for i in range(args.steps)]))
    gbs = bytes_avg / ffn_s / 1e9
    tfs = flops_avg / ffn_s / 1e12
    # tensor peak: the burst figure for a short timed region, the sustained
    # (power-capped) one for a run long enough to settle (B200_PROFILING.md)
    tf_peak, tf_which = ((tf_burst, "burst") if ms / 1e3 < 2.0 or not tf_sus
                         else (tf_sus, "sustained"))
    hbm_bound = gbs / hbm >= tfs / tf_peak
    # DRAM bytes of the two grouped GEMMs from the committed ncu --set full
    # capture of this workload (profiles/r1/ncu_traffic.json), per step like
    # `achieved`'s bytes; null for shapes / sizes not captured
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r1", "ncu_traffic.json")
    if MAP == "c2" and os.path.exists(tpath):
        tr = json.load(open(tpath)).get(str(T))
        traffic = tr["grouped_gemm_dram_bytes_per_step"] if tr else None
    roofline = ({"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                 "traffic": traffic} if hbm_bound else
                {"bound": "tensor", "achieved": tfs, "peak": tf_peak,
                 "unit": "TFLOP/s", "frac": tfs / tf_peak, "traffic": traffic})
    roofline["traffic_unit"] = "DRAM bytes per step (ncu), vs alg_bytes_per_step"
    roofline.update({"kernel": "grouped_gemm_kernel (gate-up SwiGLU + down), per layer call",
                     "peak_source": f"{src} (MEASURED_PEAKS.json)",
                     "ffn_us_per_step": ffn_s * 1e6,
                     "ffn_share_of_step": ffn_s * 1e3 / (ms_nograph / args.steps),
                     "how": "CUDA events recorded by the library on its launch stream around "
                            "both grouped-GEMM launches of every step, over a second timed pass "
                            "of the same steps launched without the CUDA graph",
                     "ms_per_step_without_graph": ms_nograph / args.steps,
                     "alg_bytes_per_step": bytes_avg, "alg_flops_per_step": flops_avg,
                     "hbm_frac": gbs / hbm, "tensor_frac": tfs / tf_peak,
                     "tensor_peak": f"{tf_which} bf16 {tf_peak} TFLOP/s (timed region "
                                    f"{ms / 1e3:.2f} s)"})
    if rank != 0:
        dist.destroy_process_group() if ws > 1 else None
        return

    cpu = None
    cpu_sched = (None, None)
    c5 = {}
    if not args.no_cpu:
        try:
            r = cpu_sample(T, max(1, min(T, args.cpu_sample_tokens)), gen_batches(T),
                           cpu_weights_fn(), os.cpu_count() or 1, hbm, tf_sus or tf_burst)
            cpu = {"value": r["tok_s"], "unit": "tokens/s", "cores": os.cpu_count() or 1,
                   "kind": "port",
                   "sample": f"reference schedule() (oracle/_ref) on the full batch, pro-rated, "
                             f"+ the build oracle's fp32 SwiGLU FFN (the reference has no FFN) "
                             f"for {r['sample_tokens']} tokens (x top-8 rows)",
                   "components": r["components"]}
            cpu_sched = (r["t_sched_us"], r["t_sched_reference_us"])
            c5 = c5_scheduler_cpu()
        except Exception as ex:  # oracle/_ref missing on this box
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "port",
                   "sample": f"unavailable: {ex}"}
    # BASELINE c5 (E=256, N=6, Zipf 1.2): the GPU scheduler on the same batches
    # as the CPU numbers, and the AEBS vs random max-activated-experts/GPU
    c5_line = {}
    if c5:
        s5 = J.Scheduler(J.config_map("c5"), local)
        for t5, r5 in c5.items():
            d5 = torch.from_numpy(r5["batch"]).to(dev)
            b5 = J.ActivationBatch(t5, 8, r5["batch"])
            c5_line[str(t5)] = {
                "gpu_us_per_iter": s5.time_schedule(d5, t5, 8, reps=51),
                "cpu_schedule_us": r5["cpu_schedule_us"],
                "cpu_schedule_reference_us": r5["cpu_schedule_reference_us"],
                "max_load_aebs": s5.schedule(b5).max_load(),
                "max_load_random": s5.schedule_random(b5, 7).max_load(),
                "cpu_max_load_aebs": r5["max_load_aebs"],
                "cpu_max_load_random": r5["max_load_random"]}
        s5.close()

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (gen_batch Zipf routing, random-init bf16 weights)",
        "config": workload_config(T, args),
        "tokens_per_s_per_gpu": value / ws,
        "value_is": METRIC_NOTE,
        "scheduler": {"us_per_iter": sched_us, "how": "CUDA-graph replay of 20 passes, median",
                      "cpu_schedule_us": cpu_sched[0], "cpu_schedule_reference_us": cpu_sched[1],
                      "c5": c5_line},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "tokens/s",
                "h2d_bytes_per_step": T * D_H * 2 + T * K_TOP * 8,
                "d2h_bytes_per_step": T * D_H * 2,
                "copies_only_value": T * args.steps / copies_s,
                "copies_only_note": "the same pinned-host copies alone (both directions at "
                                    "once), no layer: the host link's ceiling for e2e",
                "passes": "median of 3 passes of `steps` steps, alternating with the "
                          "copies-only passes",
                "pass_values": [T * args.steps * ws / v for v in e2e_runs]},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def box_trace(box, run_steps, s, s_moe, s_comb, att, moe, rank, epoch, n=30):
    """JANUS_BOX_TRACE=1: the pipelined box loop again with CUDA events around
    every enqueued call (dispatch / combine on the attention stream, the MoE
    step on its own), written to gpurun_out/boxtrace_rank{r}.json — when each
    stream reached and finished each call, relative to the first event."""
    import torch
    import torch.distributed as dist
    orig = (box.dispatch, box.moe_step, box.combine)
    evs = []

    def wrap(name, fn, st):
        def f(*a):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn(*a)
            e1.record(st)
            evs.append((name, int(a[-2]), e0, e1))
        return f
    box.dispatch = wrap("dispatch", orig[0], s)
    box.moe_step = wrap("moe", orig[1], s_moe)
    box.combine = wrap("combine", orig[2], s_comb)
    torch.cuda.synchronize()
    dist.barrier()
    base = torch.cuda.Event(enable_timing=True)
    base.record(s)
    run_steps(n)
    torch.cuda.synchronize()
    box.dispatch, box.moe_step, box.combine = orig
    rows = [(nm, ep, base.elapsed_time(a), base.elapsed_time(b)) for nm, ep, a, b in evs]
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/boxtrace_rank{rank}.json", "w") as f:
        json.dump(rows, f)
    dist.barrier()


def run_box(args):
    """N > 1: one NVLink box.  Default (``--box moe-only``): every GPU owns a
    token shard AND is an MoE instance (the attention and MoE sub-groups are
    the same N GPUs), routed transport — each token row crosses NVLink only to
    the instances its slots are scheduled on.  ``--box split``: the paper's
    disaggregated split into A attention + M MoE GPUs (BoxPlan.for_gpus: 1A+1E,
    1A+3E, 2A+6E), NVLS multicast dispatch; its attention GPUs run no attention
    math here, so its per-GPU figure carries A idle GPUs.  Same c2 expert shape
    as N=1; the replica map is the reference placement for M instances
    (maps/c2_m{M}).  Weak scaling in the MoE sub-group: T = tokens x M per
    step, so every MoE GPU sees ~T*k/M = tokens*k slots, as the single GPU
    does at N=1."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2512_13525_b200 as J
    from paper_2512_13525_b200._lib import lib
    from paper_2512_13525_b200.dist import BoxPlan, JanusBox
    from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    plan = BoxPlan.moe_only(ws) if args.box == "moe-only" else BoxPlan.for_gpus(ws)
    # measured defaults (profiles/r2/box4): MoE-only box -> routed transport,
    # push combine; split box -> NVLS dispatch, combine summed in the switch
    # (one attention GPU would otherwise take M full partial pushes)
    if args.transport == "default":
        args.transport = "routed" if plan.colocated else "auto"
    if args.combine == "default":
        args.combine = "push" if plan.colocated else "switch"
    A, M = plan.n_attn, plan.n_moe
    T = args.tokens * M
    att, moe = plan.is_attention(rank), plan.is_moe(rank)
    layer = None
    if moe:
        rmap, _ = shape_map(J, M)
        layer = MoELayer(rmap, D_H, D_E, T, K_TOP, instance=plan.instance(rank), device=local)
        layer.set_weights(*build_weight_store(layer, seed=1))
        set_shared_expert(layer, dev, split=True)  # DS-V3 shape: shared expert split over instances
        if args.gate:  # MoE-side gating: this GPU routes the rows itself
            from paper_2512_13525_b200.moe import router_weights
            layer.set_router(router_weights(E, D_H, 13, dev))
    box = JanusBox(plan, rank, T, D_H, K_TOP, layer=layer, device=local,
                   transport=args.transport, rmap=shape_map(J, M)[0], combine=args.combine)
    batches = [torch.from_numpy(b).to(dev) for b in gen_batches(T)]
    x, gw = make_inputs(T, K_TOP, D_H, 3, dev)
    first, cnt = plan.shard(T, rank) if att else (0, 0)
    xs = x[first:first + cnt].contiguous()
    gws = [gw[first * K_TOP:(first + cnt) * K_TOP].contiguous()] if att else []
    exs = [b[first * K_TOP:(first + cnt) * K_TOP].contiguous() for b in batches]
    if args.gate:  # the attention GPUs ship rows only
        gws = [None] if att else []
        exs = [None] * N_BATCHES
    out = torch.empty(max(cnt, 1), D_H, dtype=torch.bfloat16, device=dev)
    s = torch.cuda.current_stream(dev)
    stream = s.cuda_stream
    # a colocated rank runs its MoE role on a second stream (the two roles
    # share no device state; every kernel kind has its own completion counter),
    # so its combine of step i — which waits for every rank's MoE step i — does
    # not hold back its MoE step i+1
    s_moe = torch.cuda.Stream(dev) if plan.colocated else s
    stream_moe = s_moe.cuda_stream
    # combines on their own stream: a dispatch is not queued behind the previous
    # step's combine (which waits for every rank's partial-sum push); the
    # library keeps the epoch slots safe by events and flags (three slots)
    s_comb = torch.cuda.Stream(dev)
    stream_comb = s_comb.cuda_stream
    epoch = [0]

    # Two steps in flight (the exchange double-buffers by epoch parity): an
    # attention rank dispatches step i+1 before it combines step i, so the MoE
    # GPUs find step i+1's rows already delivered when they finish step i.
    # (a colocated rank interleaves its two roles in that order on one stream)
    # dispatches run `ahead` steps ahead of the MoE step (the library's three
    # epoch slots allow up to 2: combine(e-3) is enqueued before dispatch(e))
    ahead = int(os.environ.get("JANUS_BOX_AHEAD", "1"))

    def run_steps(n, i0=0):
        e0_ = epoch[0]
        if att:
            for j in range(min(ahead, n)):
                box.dispatch(xs, exs[(i0 + j) % N_BATCHES], gws[0], T, e0_ + j + 1, stream)
        for j in range(n):
            if att and j + ahead < n:
                box.dispatch(xs, exs[(i0 + j + ahead) % N_BATCHES], gws[0], T, e0_ + j + ahead + 1,
                             stream)
            if moe:
                box.moe_step(T, e0_ + j + 1, stream_moe)
            if att:
                box.combine(out, T, e0_ + j + 1, stream_comb)
        epoch[0] += n

    run_steps(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    if layer is not None:
        lib.janus_profile(layer.ctx, 1)
    launches0 = box.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(s)
        run_steps(args.steps)
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = box.launches() - launches0
    ffn = [0.0, 0.0, 0.0]
    if layer is not None:
        a_, b_, c_ = C.c_double(), C.c_double(), C.c_int()
        lib.janus_profile_read(layer.ctx, C.byref(a_), C.byref(b_), C.byref(c_))
        lib.janus_profile(layer.ctx, 0)
        ffn = [a_.value / max(c_.value, 1), b_.value / max(c_.value, 1), 1.0]
    if os.environ.get("JANUS_BOX_TRACE"):  # diagnostics: per-call events of the pipelined loop
        box_trace(box, run_steps, s, s_moe, s_comb, att, moe, rank, epoch)
    # dispatch kernel alone (attention ranks): events around the dispatch only,
    # over extra steps after the timed region
    # each phase alone, one step in flight: attention dispatch; MoE step (from
    # its inputs being present); attention combine (after every MoE published)
    disp_ms = moe_ms = comb_ms = 0.0
    dist.barrier()
    nd = 20
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for i in range(nd):
        epoch[0] += 1
        if att:
            d0, d1 = ev(), ev()
            d0.record(s)
            box.dispatch(xs, exs[i % N_BATCHES], gws[0], T, epoch[0], stream)
            d1.record(s)
            torch.cuda.synchronize()
            disp_ms += d0.elapsed_time(d1) / nd
        dist.barrier()
        if moe:
            m0, m1 = ev(), ev()
            m0.record(s_moe)
            box.moe_step(T, epoch[0], stream_moe)
            m1.record(s_moe)
            torch.cuda.synchronize()
            moe_ms += m0.elapsed_time(m1) / nd
        dist.barrier()
        if att:
            c0, c1 = ev(), ev()
            c0.record(s)
            box.combine(out, T, epoch[0], stream)
            c1.record(s)
            torch.cuda.synchronize()
            comb_ms += c0.elapsed_time(c1) / nd
    torch.cuda.synchronize()
    dist.barrier()
    # the scheduler every MoE GPU runs (replicated, on all T*k slots of the step)
    sched_us = layer.sched.time_schedule(batches[0], T, K_TOP, reps=51) if layer is not None else 0.0
    # algorithmic bytes of this MoE GPU's grouped GEMMs per step:
    # its activated replicas' weights + its routed rows in and out, averaged over
    # the batches the timed steps cycled through
    alg_b = alg_f = 0.0
    if layer is not None:
        inst = plan.instance(rank)
        per, perf = [], []
        for b in gen_batches(T):
            a = layer.sched.schedule(J.ActivationBatch(T, K_TOP, b))
            A_loc, rows = int(a.load[inst]), int(a.routed_tokens[inst])
            if SHARED:  # shared expert on this instance's even share of the tokens
                A_loc, rows = A_loc + 1, rows + J.shard_tokens(T, M, inst)[1]
            per.append(A_loc * 3 * D_H * D_E * 2 + rows * (D_H + D_E) * 2 * 2)
            perf.append(6.0 * D_H * D_E * rows)
        alg_b = float(np.mean([per[i % N_BATCHES] for i in range(args.steps)]))
        alg_f = float(np.mean([perf[i % N_BATCHES] for i in range(args.steps)]))
    tvec = torch.tensor([ms, ffn[1], float(launches), disp_ms, moe_ms, comb_ms, sched_us, alg_b, alg_f],
                        device=dev)
    allv = [torch.zeros_like(tvec) for _ in range(ws)]
    dist.all_gather(allv, tvec)
    ms_max = max(float(v[0]) for v in allv)
    ffn_ms = max(float(v[1]) for v in allv)  # slowest MoE GPU's grouped GEMMs
    slow = max(range(ws), key=lambda r: float(allv[r][1]))
    alg_slow, algf_slow = float(allv[slow][7]), float(allv[slow][8])
    launches_all = int(sum(float(v[2]) for v in allv))
    disp_ms = max(float(v[3]) for v in allv)
    moe_ms = max(float(v[4]) for v in allv)
    comb_ms = max(float(v[5]) for v in allv)
    sched_us = max(float(v[6]) for v in allv)

    # e2e through the host API: attention ranks copy their shard in from pinned
    # host memory and their outputs back each step
    if att:
        xh = xs.cpu().pin_memory()
        oh = torch.empty(max(cnt, 1), D_H, dtype=torch.bfloat16).pin_memory()
        xd = torch.empty_like(xs)
        if not args.gate:
            exh = [e.cpu().pin_memory() for e in exs]
            gwh = gws[0].cpu().pin_memory()
            exd, gwd = torch.empty_like(exs[0]), torch.empty_like(gws[0])
    dist.barrier()
    t0 = time.perf_counter()
    e0_ = epoch[0]
    if att:
        # per step: H2D of step i+1's shard (copy stream), dispatch i+1,
        # combine i (compute stream), D2H of step i's output (second copy
        # stream) — every step's bytes cross PCIe, overlapped with the layer
        xd2 = [xd, torch.empty_like(xd)]
        exd2 = [exd, torch.empty_like(exd)] if not args.gate else [None, None]
        gwd2 = [gwd, torch.empty_like(gwd)] if not args.gate else [None, None]
        out2 = [out, torch.empty_like(out)]
        h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_out = [torch.cuda.Event(), torch.cuda.Event()]   # combine wrote out[b]
        ev_read = [torch.cuda.Event(), torch.cuda.Event()]  # D2H read out[b]

        def h2d_dispatch(i):
            # the dispatch goes on the copy stream right behind its inputs'
            # H2D, so the compute stream's combine of the previous step never
            # queues behind a PCIe copy
            b = i & 1
            with torch.cuda.stream(h2d_s):
                # input buffer b: free once dispatch(i-2) ran (earlier on this stream)
                xd2[b].copy_(xh, non_blocking=True)
                if not args.gate:
                    exd2[b].copy_(exh[i % N_BATCHES], non_blocking=True)
                    gwd2[b].copy_(gwh, non_blocking=True)
                if i >= 2:
                    # exchange slot of epoch parity b: free once step i-2's
                    # combine completed (every MoE rank consumed it); the H2D
                    # above already overlaps that step
                    h2d_s.wait_event(ev_out[b])
                box.dispatch(xd2[b], exd2[b], gwd2[b], T, e0_ + i + 1, h2d_s.cuda_stream)

        h2d_dispatch(0)
        for i in range(args.steps):
            if i + 1 < args.steps:
                h2d_dispatch(i + 1)
            if moe:  # colocated rank: its MoE role for step i
                box.moe_step(T, e0_ + i + 1, stream_moe)
            b = i & 1
            if i >= 2:
                s.wait_event(ev_read[b])
            box.combine(out2[b], T, e0_ + i + 1, stream)
            ev_out[b].record(s)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_out[b])
                oh.copy_(out2[b], non_blocking=True)
                ev_read[b].record(d2h_s)
        torch.cuda.synchronize()
    else:
        for i in range(args.steps):
            box.moe_step(T, e0_ + i + 1, stream)
    epoch[0] += args.steps
    torch.cuda.synchronize()
    dist.barrier()
    e2e_s = time.perf_counter() - t0
    tt = torch.tensor([e2e_s], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s = float(tt.item())
    timed_out = box.timed_out()
    if rank == 0:
        box_tok_s = T * args.steps / (ms_max / 1e3)
        value = box_tok_s  # the whole box (all N GPUs); per GPU in tokens_per_s_per_gpu
        sends = plan.bytes_per_step(T, D_H, 0 if args.gate else K_TOP)
        send_bytes = sends[0][0]
        hbm, tf_burst, tf_sus, src = peaks()
        gbs_slow = alg_slow / (ffn_ms / 1e3) / 1e9 if ffn_ms > 0 else 0.0
        tfs_slow = algf_slow / (ffn_ms / 1e3) / 1e12 if ffn_ms > 0 else 0.0
        tf_peak = tf_burst if ms_max / 1e3 < 2.0 or not tf_sus else tf_sus
        hbm_bound = gbs_slow / hbm >= tfs_slow / tf_peak
        roof = ({"bound": "hbm", "achieved": gbs_slow, "peak": hbm, "unit": "GB/s",
                 "frac": gbs_slow / hbm} if hbm_bound else
                {"bound": "tensor", "achieved": tfs_slow, "peak": tf_peak, "unit": "TFLOP/s",
                 "frac": tfs_slow / tf_peak})
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (gen_batch Zipf routing, random-init bf16 weights)",
            "config": {"workload": f"{SHAPE_NAME} on one NVLink box " +
                                   (f"of {M} GPUs each owning a token shard and an MoE instance "
                                    f"(MoE-only box); token dispatch and combine "
                                    if plan.colocated else
                                    f"split {A} attention + {M} MoE GPUs; attention->MoE "
                                    f"dispatch and MoE->attention ") +
                                   "combine by " + ("NVSwitch multicast (NVLS) kernels"
                                                     if box.transport == "nvls" else
                                                     "copy-engine copies (dispatch) and "
                                                     "peer-memory kernels (combine)"
                                                     if box.transport == "ce"
                                                     else "peer-memory (P2P) kernels"),
                       "transport": box.transport,
                       "tokens_per_step": T, "tokens_per_moe_gpu": args.tokens,
                       "shared_expert": "every MoE GPU on its even share of the tokens"
                                        if SHARED else False,
                       "replica_map": shape_map_name(M),
                       "parallelism": f"{M} x (A+E)" if plan.colocated else f"{A}A+{M}E",
                       "gating": "MoE-side: rows only cross NVLink, every MoE GPU runs "
                                 "gate_kernel on the full step" if args.gate else
                                 "attention-side: top-k ids and gate weights shipped with "
                                 "the rows",
                       "l2": "inputs > L2 (weights streamed)"},
            "tokens_per_s_box": box_tok_s, "tokens_per_s_per_moe_gpu": box_tok_s / M,
            "tokens_per_s_per_gpu": box_tok_s / ws,
            "value_is": METRIC_NOTE + " (attention GPUs included in N; they run no "
                        "attention math here)",
            "roofline": {**roof, "kernel": "grouped_gemm_kernel on the slowest MoE GPU",
                         "ffn_us_per_step": ffn_ms * 1e3,
                         "traffic": None, "alg_bytes_per_step": alg_slow,
                         "alg_flops_per_step": algf_slow, "hbm_frac": gbs_slow / hbm,
                         "tensor_frac": tfs_slow / tf_peak,
                         "how": "library CUDA events around both grouped-GEMM launches of "
                                "every step on the MoE GPU with the largest FFN time; bytes "
                                "from that GPU's own schedule of the same batches",
                         "peak_source": f"{src} (MEASURED_PEAKS.json)"},
            "nvlink": {"transport": box.transport,
                       # P2P: the attention GPU stores each row once per MoE GPU;
                       # NVLS: once, the switch fans it out to the M MoE GPUs
                       "dispatch_egress_bytes_per_step_per_attention_gpu":
                           send_bytes // (M if box.transport == "nvls" else 1),
                       "dispatch_bytes_per_step_per_attention_gpu": send_bytes,
                       "combine_bytes_per_step_per_attention_gpu": sends[0][1],
                       "dispatch_us": disp_ms * 1e3,
                       "moe_step_us": moe_ms * 1e3,
                       "combine_us": comb_ms * 1e3,
                       "dispatch_achieved_gbs": send_bytes / (disp_ms / 1e3) / 1e9
                       if disp_ms > 0 else None,
                       "dispatch_egress_gbs": send_bytes // (M if box.transport == "nvls" else 1)
                       / (disp_ms / 1e3) / 1e9 if disp_ms > 0 else None,
                       "peak_gbs": 770.0, "peak_source": "B200_PROFILING.md measured peer copy "
                                                         "per direction (fallback)"},
            "e2e": {"value": T * args.steps / e2e_s, "unit": "tokens/s",
                    "h2d_bytes_per_step": T * (D_H * 2 + (0 if args.gate else K_TOP * 8)),
                    "d2h_bytes_per_step": T * D_H * 2},
            "scheduler": {"us_per_iter": sched_us, "slots": T * K_TOP,
                          "how": "CUDA-graph replay of 20 passes on an MoE GPU, median; the "
                                 "slowest MoE GPU"},
            "gpu_launches": launches_all, "timed_out": timed_out,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-tokens", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--box", default="moe-only", choices=["split", "moe-only"],
                    help="--gpus > 1: the paper's attention/MoE split (1 attention GPU per "
                         "4), or the MoE-only box (every GPU owns tokens and experts)")
    ap.add_argument("--shape", default="c2", choices=sorted(SHAPES),
                    help="expert shape (BASELINE configs); c2 is the headline")
    ap.add_argument("--gate", action="store_true",
                    help="box: MoE-side gating (rows only cross NVLink; every MoE GPU runs "
                         "the router GEMM + top-k on the full step)")
    ap.add_argument("--combine", default="default", choices=["default", "push", "switch"],
                    help="NVLS combine: partial sums pushed point to point (default) or "
                         "summed by the NVSwitch (multimem.ld_reduce)")
    ap.add_argument("--transport", default="default",
                    choices=["default", "auto", "p2p", "nvls", "routed", "ce"],
                    help="box exchange for --gpus > 1 (auto: NVLS multicast when supported; "
                         "routed: rows only to the MoE GPUs their slots are scheduled on; "
                         "ce: the P2P broadcast moved by the copy engines)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    apply_shape(args.shape)
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[0] > 1:
        run_box(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
