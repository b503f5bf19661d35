"""The box protocol on CPU with gloo (world sizes 2 and 3): roles, token shards,
the replicated scheduler's sync-free invariant, and the partial-sum combine.

Each process plays one rank of an A-attention + M-MoE box.  The data movement
the GPU kernels do over NVLink (janus_attn_dispatch_async / combine) is
emulated with gloo send/recv, and the MoE compute with the CPU oracle, so the
host-side plan (paper_2512_13525_b200.dist.BoxPlan) and the exchange's
semantics are checked without a GPU:
  * every rank derives the same plan and the shards tile [0, T) (comm.cpp:76-81);
  * every MoE rank computes the identical assignment from the identical batch
    (no count exchange);
  * sum over MoE ranks of the per-instance partials (each rounded to bf16, as
    the push kernel does) == the single-GPU layer within the layer tolerance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RTOL = ATOL = 2.0 ** -6
E, K, D_H, D_E, T = 12, 3, 64, 32, 23


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def weights():
    from oracle import Oracle
    o = Oracle()
    r = np.random.default_rng(11)
    return [tuple(o.f32_to_bf16(r.standard_normal(sh).astype(np.float32) * sc)
                  for sh, sc in (((D_E, D_H), D_H ** -0.5), ((D_E, D_H), D_H ** -0.5),
                                 ((D_H, D_E), D_E ** -0.5)))
            for _ in range(E)]


def worker(rank, world, n_attn, port, q):
    import sys
    for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
        sys.path.insert(0, p)
    from oracle import CSRMap, Oracle
    from paper_2512_13525_b200.dist import BoxPlan

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        orc = Oracle()
        plan = BoxPlan(n_attn, world - n_attn)
        M = plan.n_moe
        views = [None] * world
        dist.all_gather_object(views, (plan.n_attn, plan.n_moe, plan.role(rank),
                                       plan.instance(rank)))
        assert all(v[:2] == (plan.n_attn, plan.n_moe) for v in views)
        shards = [plan.shard(T, a) for a in range(plan.n_attn)]
        assert shards[0][0] == 0 and sum(c for _, c in shards) == T
        assert all(shards[i][0] + shards[i][1] == shards[i + 1][0] for i in range(len(shards) - 1))

        hosts = [sorted({e % M, (e + 1) % M}) for e in range(E)]
        m = CSRMap.from_lists(M, E, hosts)
        _, cdf = orc.pattern("gaussian", E, 0.25)
        ex = orc.gen_batch(cdf, T, K, 5, 1)
        r = np.random.default_rng(3)
        x = orc.f32_to_bf16(r.standard_normal((T, D_H)).astype(np.float32))
        gw = r.random((T, K)).astype(np.float32)
        W = weights()

        if plan.role(rank) == "attention":
            first, cnt = plan.shard(T, rank)
            for g in range(M):  # dispatch: shard rows, routing, gate weights to every MoE rank
                dst = plan.n_attn + g
                dist.send(torch.from_numpy(x[first:first + cnt].astype(np.int32)), dst)
                dist.send(torch.from_numpy(ex[first * K:(first + cnt) * K].copy()), dst)
                dist.send(torch.from_numpy(gw[first:first + cnt].copy()), dst)
            parts = []
            for g in range(M):  # combine: M partials for this shard, fixed instance order
                buf = torch.zeros(cnt, D_H, dtype=torch.float32)
                dist.recv(buf, plan.n_attn + g)
                parts.append(buf.numpy())
            got = np.zeros((cnt, D_H), np.float32)
            for p in parts:
                got += p
            # single-GPU reference: all slots, one fp32 sum
            a = orc.schedule(ex, T, K, m)
            ref = np.zeros((cnt, D_H), np.float32)
            for t in range(first, first + cnt):
                for j in range(K):
                    e = int(ex[t * K + j])
                    y = orc.expert_swiglu(x[t:t + 1], *W[e], round_h=True)[0]
                    ref[t - first] += gw[t, j] * y
            rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2)))
            ok = bool((np.abs(got - ref) <= RTOL * np.abs(ref) + ATOL * rms).all())
            q.put(("attention", rank, ok, a.load.tolist()))
        else:
            g = plan.instance(rank)
            rx = np.zeros((T, D_H), np.uint16)
            rex = np.zeros(T * K, np.int32)
            rgw = np.zeros((T, K), np.float32)
            for a_ in range(plan.n_attn):
                first, cnt = plan.shard(T, a_)
                b = torch.zeros(cnt, D_H, dtype=torch.int32)
                dist.recv(b, a_)
                rx[first:first + cnt] = b.numpy().astype(np.uint16)
                b = torch.zeros(cnt * K, dtype=torch.int32)
                dist.recv(b, a_)
                rex[first * K:(first + cnt) * K] = b.numpy()
                b = torch.zeros(cnt, K, dtype=torch.float32)
                dist.recv(b, a_)
                rgw[first:first + cnt] = b.numpy()
            asg = orc.schedule(rex, T, K, m)  # replicated, identical on every MoE rank
            part = np.zeros((T, D_H), np.float32)
            for t in range(T):
                for j in range(K):
                    s = t * K + j
                    if asg.instance[s] != g:
                        continue
                    e = int(rex[s])
                    part[t] += rgw[t, j] * orc.expert_swiglu(rx[t:t + 1], *W[e], round_h=True)[0]
            from oracle import bf16_to_f32
            part = bf16_to_f32(orc.f32_to_bf16(part))  # pushed as bf16
            for a_ in range(plan.n_attn):
                first, cnt = plan.shard(T, a_)
                dist.send(torch.from_numpy(part[first:first + cnt].copy()), a_)
            q.put(("moe", rank, True, asg.instance.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_attn", [(2, 1), (3, 1), (3, 2)])
def test_box_protocol_gloo(world, n_attn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, n_attn, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    res = [q.get(timeout=5) for _ in range(world)]
    assert all(ok for _, _, ok, _ in res)
    moe = [inst for role, _, _, inst in res if role == "moe"]
    assert all(m_ == moe[0] for m_ in moe)  # sync-free: identical assignments everywhere


@pytest.mark.parametrize("n", [2, 4, 8])  # the N of the driver's scaling run
def test_bench_box_plans(n):
    """The splits `bench.py --gpus n` launches (BoxPlan.for_gpus: 1 attention GPU
    per 4, the paper's 2A+6E box at 8) and the MoE-only box: roles cover every
    rank once, attention shards tile the step exactly (comm.cpp:76-81), and the
    replica map each split needs ships in the package."""
    import paper_2512_13525_b200 as J
    from paper_2512_13525_b200.dist import BoxPlan
    p = BoxPlan.for_gpus(n)
    assert p.n_attn == max(1, n // 4) and p.n_attn + p.n_moe == n == p.world
    assert [p.instance(r) for r in range(n) if p.is_moe(r)] == list(range(p.n_moe))
    assert sum(p.is_attention(r) for r in range(n)) == p.n_attn
    for Tn in (4096 * p.n_moe, 4096 * p.n_moe + 3, 1):
        spans = [p.shard(Tn, a) for a in range(p.n_attn)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == Tn
        assert all(f0 + c0 == f1 for (f0, c0), (f1, _) in zip(spans, spans[1:]))
        assert p.owner(Tn, Tn - 1) == max(a for a, (_, c) in enumerate(spans) if c)
    for M in (p.n_moe, n):  # split box and MoE-only box (BoxPlan.moe_only(n))
        m = J.config_map(f"c2_m{M}") if M > 1 else J.config_map("c2")
        assert m.num_instances == M and m.num_experts == 128
    q = BoxPlan.moe_only(n)
    assert all(q.is_attention(r) and q.is_moe(r) and q.instance(r) == r for r in range(n))
