"""The attention <-> MoE box exchange through the real C ABI on ONE GPU.

Every rank of an A-attention + M-MoE box (or the MoE-only box) is a context in
this process, connected with raw pointers (janus_xfer_connect_local) instead of
CUDA IPC; the same kernels run — dispatch (broadcast P2P or routed), the MoE
rank's wait + K1-K5 with K5 pushing partial sums into the owners' regions, the
combine flag with the step's status, the owner's wait + reduce.  All calls go
on one stream in causal order (every producer before its consumer's wait), so
no kernel ever waits on one that has not run (B200_PROFILING.md: waiting
kernels must not rely on running concurrently on one GPU).

Each attention shard's output is compared with the fp32 oracle (oracle.c
or_expert_swiglu + the combine sum), not with the repo's own single-GPU layer:
  * vs the oracle with h rounded to bf16 as the device rounds it:
    |dev - ref| <= 2^-6 |ref| + 2^-6 rms(ref);
  * vs the pure fp32 layer: |dev - ref| <= 2^-5 |ref| + 2^-5 rms(ref).
The box's per-MoE-rank partial sums are rounded to bf16 before the owner adds
them (fp32), so the bound is the single-GPU layer's plus one bf16 rounding per
partial.  References: comm.hpp:96-98 (MoE-side aggregation plays the
all-reduce role), test_comm.cpp:35-64 (every MoE node gets the full batch —
the broadcast transports), comm.hpp:20-39 / comm.cpp:155-160 (per-destination
traffic — the routed transport).
"""
import json
import os

import numpy as np
import pytest

from _ffn_ref import assert_close, err_stats, moe_reference, u16

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E, K, D_H, D_E = 16, 4, 256, 128


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2512_13525_b200 as J
    from paper_2512_13525_b200.moe import expert_weights
    cache = {}

    def weights_of(e):
        if e not in cache:
            cache[e] = tuple(u16(w) for w in expert_weights(e, D_H, D_E, 1, "cuda"))
        return cache[e]
    return J, weights_of


def make_box(J, plan, T_max, transport, rmap):
    from paper_2512_13525_b200.dist import JanusBox
    from paper_2512_13525_b200.moe import MoELayer, build_weight_store
    layers = {}
    for r in range(plan.world):
        if plan.is_moe(r):
            layer = MoELayer(rmap, D_H, D_E, T_max, K, instance=plan.instance(r), device=0)
            layer.set_weights(*build_weight_store(layer, seed=1))
            layers[r] = layer
    boxes = JanusBox.local(plan, T_max, D_H, K, layers, transport=transport, rmap=rmap)
    return boxes, layers


def box_map(J, M):
    # two replicas per expert on neighbouring instances (AEBS has choices)
    return J.ReplicaMap.from_hosts(M, E, [sorted({e % M, (e + 1) % M}) for e in range(E)])


def gen_steps(oracle, n, T):
    import torch
    from paper_2512_13525_b200.moe import make_inputs
    _, cdf = oracle.pattern("gaussian", E, sigma=0.2)
    steps = []
    for s in range(1, n + 1):
        Ts = T - 37 * (s % 3)  # ragged shards, varying step size
        ex = torch.from_numpy(oracle.gen_batch(cdf, Ts, K, 7, s)).cuda()
        x, gw = make_inputs(Ts, K, D_H, s, "cuda")
        steps.append((Ts, x, gw, ex))
    return steps


def run_box(plan, boxes, steps, inflight, transport):
    """Enqueue every rank's calls on torch's current stream in causal order."""
    import torch
    s = torch.cuda.current_stream().cuda_stream
    k = K
    outs = {}

    def dispatch(e):
        Ts, x, gw, ex = steps[e - 1]
        att = [r for r in range(plan.world) if plan.is_attention(r)]
        if transport == "routed":  # every shard's routing lands before any dispatch waits on it
            for r in att:
                f, c = plan.shard(Ts, r)
                boxes[r].route(ex[f * k:(f + c) * k].contiguous(),
                               gw[f * k:(f + c) * k].contiguous(), Ts, e, s)
        for r in att:
            f, c = plan.shard(Ts, r)
            boxes[r].dispatch(x[f:f + c].contiguous(), ex[f * k:(f + c) * k].contiguous(),
                              gw[f * k:(f + c) * k].contiguous(), Ts, e, s)

    def moe(e):
        for r in range(plan.world):
            if plan.is_moe(r):
                boxes[r].moe_step(steps[e - 1][0], e, s)

    def combine(e):
        Ts = steps[e - 1][0]
        for r in range(plan.world):
            if plan.is_attention(r):
                f, c = plan.shard(Ts, r)
                outs[(e, r)] = torch.empty(max(c, 1), D_H, dtype=torch.bfloat16, device="cuda")
                boxes[r].combine(outs[(e, r)], Ts, e, s)

    n = len(steps)
    if inflight == 1:
        for e in range(1, n + 1):
            dispatch(e)
            moe(e)
            combine(e)
    else:  # dispatch step e+1 before combining step e (double-buffered slots)
        dispatch(1)
        for e in range(1, n + 1):
            if e < n:
                dispatch(e + 1)
            moe(e)
            combine(e)
    torch.cuda.synchronize()
    return outs


def check_outputs(oracle, weights_of, plan, steps, outs, what):
    stats = []
    for e, (Ts, x, gw, ex) in enumerate(steps, 1):
        xu = u16(x)
        exn = ex.cpu().numpy().reshape(Ts, K)
        w = gw.cpu().numpy().reshape(Ts, K)
        ref_h = moe_reference(oracle, xu, exn, w, weights_of, round_h=True)
        ref_f = moe_reference(oracle, xu, exn, w, weights_of, round_h=False)
        for r in range(plan.world):
            if not plan.is_attention(r):
                continue
            f, c = plan.shard(Ts, r)
            if c == 0:
                continue
            dev = outs[(e, r)][:c].float().cpu().numpy()
            assert_close(dev, ref_h[f:f + c], 2.0 ** -6, 2.0 ** -6, f"{what} step {e} rank {r}")
            assert_close(dev, ref_f[f:f + c], 2.0 ** -5, 2.0 ** -5,
                         f"{what} step {e} rank {r} (pure fp32)")
            stats.append({"step": e, "rank": r, "vs_round_h": err_stats(dev, ref_h[f:f + c])[0],
                          "vs_fp32": err_stats(dev, ref_f[f:f + c])[0]})
    return stats


# ... plus the north_star box split 2A+6E (BASELINE c3) and the 8-GPU MoE-only
# box the 8-GPU bench runs, every rank on this one GPU
CASES = [(1, 1, False), (1, 3, False), (2, 2, False), (2, 2, True), (4, 4, True), (2, 6, False),
         (8, 8, True)]


@pytest.mark.parametrize("transport", ["p2p", "routed", "ce"])
@pytest.mark.parametrize("inflight", [1, 2])
@pytest.mark.parametrize("attn,moe,colocated", CASES)
def test_box_exchange_vs_oracle(env, oracle, attn, moe, colocated, inflight, transport):
    J, weights_of = env
    from paper_2512_13525_b200.dist import BoxPlan
    plan = BoxPlan.moe_only(moe) if colocated else BoxPlan(attn, moe)
    rmap = box_map(J, plan.n_moe)
    T = 300
    boxes, layers = make_box(J, plan, T, transport, rmap)
    for b in boxes:
        b.set_timeout(5.0)
    steps = gen_steps(oracle, 4, T)
    outs = run_box(plan, boxes, steps, inflight, transport)
    for b in boxes:
        assert not b.timed_out()
        b.check()
    what = f"{attn}A+{moe}M{' colocated' if colocated else ''} {transport} inflight={inflight}"
    stats = check_outputs(oracle, weights_of, plan, steps, outs, what)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "box_local_stats.jsonl"), "a") as f:
        f.write(json.dumps({"case": what, "max_err_over_rms": {
            "vs_round_h": max(s["vs_round_h"] for s in stats),
            "vs_fp32": max(s["vs_fp32"] for s in stats)}}) + "\n")


@pytest.mark.parametrize("transport", ["p2p", "routed", "ce"])
def test_unknown_expert_on_moe_rank_raises_on_attention_rank(env, oracle, transport):
    """An unknown expert in one step: every MoE rank's K1 rejects it and
    publishes the status with its combine flag; the attention ranks raise the
    reference's ValidationError (aebs.cpp:22-25) from check(), their rows of
    that step are zeros, and the next step is correct again."""
    import torch
    J, weights_of = env
    from paper_2512_13525_b200.dist import BoxPlan
    plan = BoxPlan(2, 2)
    rmap = box_map(J, 2)
    boxes, _ = make_box(J, plan, 300, transport, rmap)
    for b in boxes:
        b.set_timeout(5.0)
    steps = gen_steps(oracle, 3, 300)
    Ts, x, gw, ex = steps[1]
    ex = ex.clone()
    ex[5 * K + 1] = E + 3  # step 2, token 5: expert 19 has no replica
    steps[1] = (Ts, x, gw, ex)
    outs = run_box(plan, boxes, steps, 2, transport)
    for r in (0, 1):
        with pytest.raises(J.ValidationError, match=r"^unknown-expert: batch references expert 19 "
                                                    r"with no replica in the map$"):
            boxes[r].check()
        boxes[r].check()  # reported once
        f, c = plan.shard(Ts, r)
        assert torch.count_nonzero(outs[(2, r)][:c]).item() == 0
    for r in (2, 3):  # the MoE ranks saw it too
        with pytest.raises(J.ValidationError):
            boxes[r].check()
    good = [steps[0], steps[2]]
    check_outputs(oracle, weights_of, plan, good,
                  {(1, r): outs[(1, r)] for r in (0, 1)} | {(2, r): outs[(3, r)] for r in (0, 1)},
                  f"around a failed step ({transport})")


def test_missing_shard_times_out_and_propagates(env, oracle):
    """A MoE step whose shards never arrive: its bounded wait expires, K1-K5
    skip, the step's status (EPEER) reaches the attention rank, whose rows of
    the step are zeros — no hang."""
    import torch
    J, _ = env
    from paper_2512_13525_b200._lib import EPEER
    from paper_2512_13525_b200.dist import BoxPlan
    from paper_2512_13525_b200.moesim import JanusError
    plan = BoxPlan(1, 1)
    boxes, _ = make_box(J, plan, 64, "p2p", box_map(J, 1))
    for b in boxes:
        b.set_timeout(0.05)
    s = torch.cuda.current_stream().cuda_stream
    boxes[1].moe_step(64, 7, s)  # epoch 7 was never dispatched
    out = torch.ones(64, D_H, dtype=torch.bfloat16, device="cuda")
    boxes[0].combine(out, 64, 7, s)
    torch.cuda.synchronize()
    assert boxes[1].timed_out()
    assert torch.count_nonzero(out).item() == 0
    with pytest.raises(JanusError) as ei:
        boxes[0].check()
    assert ei.value.status == EPEER


def test_routed_layout_bytes(env, oracle):
    """Routed transport: a token row reaches exactly the MoE ranks its slots
    were scheduled on (the oracle's schedule), i.e. NVLink bytes per MoE rank
    = its distinct routed tokens x 2 d_h (StepTraffic, comm.hpp:20-39): the
    receive buffer rows of every other token keep a sentinel."""
    import torch
    J, _ = env
    from oracle import CSRMap
    from paper_2512_13525_b200.dist import BoxPlan
    plan = BoxPlan(1, 3)
    rmap = box_map(J, 3)
    T = 200
    boxes, layers = make_box(J, plan, T, "routed", rmap)
    steps = gen_steps(oracle, 1, T)
    Ts, x, gw, ex = steps[0]
    # sentinel-fill the MoE ranks' receive rows (slot of epoch 1)
    s = torch.cuda.current_stream().cuda_stream
    recv = {r: boxes[r].recv_rows(1, Ts) for r in (1, 2, 3)}
    for r in (1, 2, 3):
        recv[r].fill_(0x2B2B)
    torch.cuda.synchronize()
    boxes[0].dispatch(x, ex, gw, Ts, 1, s)
    torch.cuda.synchronize()
    off, hosts, rid = rmap.csr()
    m = CSRMap(E, 3, rmap.slots_per_instance, off, hosts, rid)
    inst = oracle.schedule(ex.cpu().numpy(), Ts, K, m).instance.reshape(Ts, K)
    xu = u16(x)
    for g, r in enumerate((1, 2, 3)):
        rows = recv[r].cpu().numpy().view(np.uint16)
        want = (inst == g).any(axis=1)
        assert 0 < want.sum() < Ts, g
        assert np.array_equal(rows[want], xu[want]), g
        assert (rows[~want] == 0x2B2B).all(), g
