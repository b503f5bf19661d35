"""Multi-GPU worker for tests/test_gpu_dist.py (launched with torchrun, one rank
per GPU).  Runs several decode steps of an A-attention + M-MoE box through the
C-ABI exchange and checks every attention shard's output against the fp32
oracle (oracle.c or_expert_swiglu + the combine sum, tests/_ffn_ref.py) — with
h rounded as the device rounds it (2^-6 rel + 2^-6 rms) and pure fp32
(2^-5 rel + 2^-5 rms) — and every rank's janus_xfer_check.

  torchrun --nproc-per-node A+M tests/dist_worker.py --attn A --moe M --out DIR
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200.dist import BoxPlan, JanusBox  # noqa: E402
from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs  # noqa: E402
from _ffn_ref import err_stats, moe_reference, u16  # noqa: E402
from oracle import Oracle  # noqa: E402

RTOL = ATOL = 2.0 ** -6          # vs the oracle with h rounded like the device
RTOL32 = ATOL32 = 2.0 ** -5      # vs the pure fp32 oracle


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--attn", type=int, default=1)
    ap.add_argument("--moe", type=int, default=1)
    ap.add_argument("--tokens", type=int, default=300)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nvls", "routed", "ce"])
    ap.add_argument("--combine", default="push", choices=["push", "switch"])
    ap.add_argument("--shared", action="store_true", help="add a shared expert (NVLS only)")
    ap.add_argument("--shared-split", action="store_true",
                    help="the shared expert split evenly over the MoE instances (implies --shared)")
    ap.add_argument("--colocated", action="store_true",
                    help="MoE-only box: every rank owns a shard and is an MoE instance")
    ap.add_argument("--gate", action="store_true",
                    help="MoE-side gating: dispatch rows only, MoE ranks run the router")
    ap.add_argument("--inflight", type=int, default=1, choices=[1, 2, 3],
                    help="2 / 3: dispatch step s+1 / s+2 before combining step s (three epoch slots)")
    ap.add_argument("--split-streams", action="store_true",
                    help="combines on a stream of their own (the slots kept safe by the library)")
    args = ap.parse_args()
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    # JANUS_TEST_GPUS=n: more ranks than GPUs (rank r on GPU r % n; the
    # exchange's protocol at a world the box does not have, e.g. 8 ranks);
    # torch.distributed then runs on gloo (plumbing only: IPC handles, barriers)
    ngpu = int(os.environ.get("JANUS_TEST_GPUS", "0"))
    if ngpu:
        local = local % ngpu
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    plan = BoxPlan.moe_only(args.moe) if args.colocated else BoxPlan(args.attn, args.moe)
    assert dist.get_world_size() == plan.world
    E, k, d_h, d_e, T = 16, 4, 256, 128, args.tokens
    M = plan.n_moe
    hosts = [sorted({e % M, (e + 1) % M}) for e in range(E)]
    rmap = J.ReplicaMap.from_hosts(M, E, hosts)
    dev = torch.device("cuda", local)

    layer = None
    att, moe = plan.is_attention(rank), plan.is_moe(rank)
    if moe:
        layer = MoELayer(rmap, d_h, d_e, T, k, instance=plan.instance(rank), device=local)
        layer.set_weights(*build_weight_store(layer, seed=1))
    args.shared = args.shared or args.shared_split
    if args.shared:
        from paper_2512_13525_b200.moe import expert_weights
        wg, wu, wd = expert_weights(99, d_h, d_e, 5, dev)
        shared_w = (torch.cat([wg, wu]).contiguous(), wd.contiguous())
        if layer is not None:
            layer.set_shared(*shared_w, split=args.shared_split)
    if args.gate:
        from paper_2512_13525_b200.moe import router_weights
        wr = router_weights(E, d_h, 13, dev)
        if layer is not None:
            layer.set_router(wr)
    box = JanusBox(plan, rank, T, d_h, k, layer=layer, device=local, transport=args.transport,
                   rmap=rmap, combine=args.combine)
    orc = Oracle()
    from paper_2512_13525_b200.moe import expert_weights
    wcache = {}

    def weights_of(e):
        if e not in wcache:
            wcache[e] = tuple(u16(w) for w in (expert_weights(99, d_h, d_e, 5, dev) if e == -1
                                               else expert_weights(e, d_h, d_e, 1, dev)))
        return wcache[e]

    stream = torch.cuda.current_stream(dev).cuda_stream
    # --split-streams: as bench.py runs the box — dispatch, MoE step and combine
    # each on a stream of its own
    cstream = torch.cuda.Stream(dev).cuda_stream if args.split_streams else stream
    mstream = torch.cuda.Stream(dev).cuda_stream if args.split_streams else stream
    result = {"rank": rank, "role": plan.role(rank), "steps": [], "transport": box.transport}
    steps = []
    for step in range(1, args.steps + 1):
        Ts = T - 37 * (step % 3)  # vary the step size: ragged shards
        _, cdf = orc.pattern("gaussian", E, sigma=0.2)
        x, gw = make_inputs(Ts, k, d_h, step, dev)
        ex = torch.from_numpy(orc.gen_batch(cdf, Ts, k, 7, step)).to(dev)
        steps.append((Ts, x, gw, ex))

    outs = {}
    for step in range(1, args.steps + 1 if att else 1):  # made before any stream uses them
        first, cnt = plan.shard(steps[step - 1][0], rank)
        outs[step] = torch.empty(cnt, d_h, dtype=torch.bfloat16, device=dev)
    torch.cuda.synchronize()

    def dispatch(step):
        Ts, x, gw, ex = steps[step - 1]
        first, cnt = plan.shard(Ts, rank)
        if args.gate:
            box.dispatch(x[first:first + cnt].contiguous(), None, None, Ts, step, stream)
        else:
            box.dispatch(x[first:first + cnt].contiguous(),
                         ex[first * k:(first + cnt) * k].contiguous(),
                         gw[first * k:(first + cnt) * k].contiguous(), Ts, step, stream)

    def combine(step):
        Ts = steps[step - 1][0]
        first, cnt = plan.shard(Ts, rank)
        box.combine(outs[step], Ts, step, cstream)

    # one stream per rank; a colocated rank interleaves its roles in the same
    # order as the split box's ranks would (dispatch before MoE before combine).
    # More ranks than GPUs: ranks sharing a GPU are separate processes, and no
    # wait kernel may rely on another process's kernel running beside it — so
    # every phase ends with a device sync and a barrier of all ranks, and each
    # wait finds the flags it waits for already published.
    def phase_end():
        if ngpu:
            torch.cuda.synchronize()
            dist.barrier()

    if args.inflight == 1:
        for step in range(1, args.steps + 1):
            if att:
                dispatch(step)
            phase_end()
            if moe:
                box.moe_step(steps[step - 1][0], step, mstream)
            phase_end()
            if att:
                combine(step)
            torch.cuda.synchronize()
    else:  # dispatches inflight - 1 steps ahead of the MoE step
        ahead = args.inflight - 1
        if att:
            for j in range(1, min(ahead, args.steps) + 1):
                dispatch(j)
        phase_end()
        for step in range(1, args.steps + 1):
            if att and step + ahead <= args.steps:
                dispatch(step + ahead)
            phase_end()
            if moe:
                box.moe_step(steps[step - 1][0], step, mstream)
            phase_end()
            if att:
                combine(step)
            phase_end()
        torch.cuda.synchronize()
    for step in range(1, args.steps + 1):
        Ts, x, gw, ex = steps[step - 1]
        if not att:
            result["steps"].append({"T": Ts})
            continue
        first, cnt = plan.shard(Ts, rank)
        xs = u16(x[first:first + cnt])
        keep = np.ones(cnt, bool)
        if args.gate:  # the routing the MoE ranks computed: the gating oracle on the same rows
            exn, wn, lg = orc.gate(xs, u16(wr), k, want_logits=True)
            exn, wn = exn.reshape(cnt, k), wn.reshape(cnt, k)
            srt = -np.sort(-lg, axis=1)  # tokens whose k-th / (k+1)-th logits nearly tie
            keep = srt[:, k - 1] - srt[:, k] > 1e-3  # may select differently (fp32 vs double)
        else:
            exn = ex.cpu().numpy().reshape(Ts, k)[first:first + cnt]
            wn = gw.cpu().numpy().reshape(Ts, k)[first:first + cnt]
        if args.shared:  # the shared expert: one more slot of weight 1 on every token
            exn = np.concatenate([exn, np.full((cnt, 1), -1, np.int32)], axis=1)
            wn = np.concatenate([wn, np.ones((cnt, 1), np.float32)], axis=1)
        o = outs[step][:cnt].float().cpu().numpy()[keep]
        xs, exn, wn = xs[keep], exn[keep], wn[keep]
        bad = n32 = 0
        errs = [0.0, 0.0]
        for i, (rh, tol_r, tol_a) in enumerate(((True, RTOL, ATOL), (False, RTOL32, ATOL32))):
            r = moe_reference(orc, xs, exn, wn, weights_of, round_h=rh)
            rms = float(np.sqrt(np.mean(r.astype(np.float64) ** 2))) or 1.0
            nb = int((np.abs(o - r) > tol_r * np.abs(r) + tol_a * rms).sum())
            bad, n32 = (nb, n32) if rh else (bad, nb)
            errs[i] = err_stats(o, r)[0]
        result["steps"].append({"T": Ts, "shard": [first, cnt], "bad": bad + n32,
                                "max_err_over_rms": errs[0], "max_err_over_rms_fp32": errs[1]})
    result["timed_out"] = box.timed_out()
    try:
        box.check()
        result["check"] = "ok"
    except Exception as ex_:  # noqa: BLE001
        result["check"] = str(ex_)
    os.makedirs(args.out, exist_ok=True)
    with open(os.path.join(args.out, f"dist_{args.attn}a{args.moe}m_{args.transport}{args.combine}_{args.inflight}{'s' if args.shared else ''}{'x' if args.shared_split else ''}{'g' if args.gate else ''}{'c' if args.colocated else ''}{'t' if args.split_streams else ''}_rank{rank}.json"), "w") as f:
        json.dump(result, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
