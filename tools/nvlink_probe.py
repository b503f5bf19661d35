"""NVLink evidence for the box exchange in ONE process driving two GPUs (so ncu
can profile it: no multi-rank command).  Rank 0 = attention on GPU 0, rank 1 =
MoE instance 0 on GPU 1 (1A+1E, c2 expert shape), connected with raw peer
pointers (janus_xfer_connect_local).  Each phase runs alone, in causal order
with a host sync between phases, so no kernel ever waits on one that has not
run:  dispatch (GPU 0 -> GPU 1 rows)  ->  MoE step (GPU 1, K5 pushes partial
sums to GPU 0)  ->  combine (GPU 0).

  python tools/nvlink_probe.py [--transport p2p|routed] [--tokens 4096] [--steps 10]

Also measures the peer-copy peak (cudaMemcpyPeer, 1 GiB, both directions)
and prints one JSON line.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--transport", default="p2p", choices=["p2p", "routed"])
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--no-peak", action="store_true")
    args = ap.parse_args()
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    import paper_2512_13525_b200 as J
    from paper_2512_13525_b200.dist import BoxPlan, JanusBox
    from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs
    from routing import RoutingPattern, gen_batch

    E, k, d_h, d_e, T = 128, 8, 2048, 768, args.tokens
    plan = BoxPlan(1, 1)
    rmap = J.config_map("c2")
    torch.cuda.set_device(1)
    layer = MoELayer(rmap, d_h, d_e, T, k, instance=0, device=1)
    layer.set_weights(*build_weight_store(layer, seed=1))
    boxes = JanusBox.local(plan, T, d_h, k, {1: layer}, devices={0: 0, 1: 1},
                           transport=args.transport, rmap=rmap)
    torch.cuda.set_device(0)
    x, gw = make_inputs(T, k, d_h, 3, "cuda:0")
    ex = torch.from_numpy(gen_batch(RoutingPattern.zipf(E, 1.0), T, k, 0x30, T * 1000).experts).to(
        "cuda:0")
    out = torch.empty(T, d_h, dtype=torch.bfloat16, device="cuda:0")
    s0 = torch.cuda.current_stream(0)
    s1 = torch.cuda.current_stream(1)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t = {"dispatch": [], "moe": [], "combine": []}
    for step in range(1, args.steps + 1):
        torch.cuda.set_device(0)
        a, b = ev(), ev()
        a.record(s0)
        boxes[0].dispatch(x, ex, gw, T, step, s0.cuda_stream)
        b.record(s0)
        torch.cuda.synchronize(0)
        t["dispatch"].append(a.elapsed_time(b))
        torch.cuda.set_device(1)
        a, b = ev(), ev()
        a.record(s1)
        boxes[1].moe_step(T, step, s1.cuda_stream)
        b.record(s1)
        torch.cuda.synchronize(1)
        t["moe"].append(a.elapsed_time(b))
        torch.cuda.set_device(0)
        a, b = ev(), ev()
        a.record(s0)
        boxes[0].combine(out, T, step, s0.cuda_stream)
        b.record(s0)
        torch.cuda.synchronize(0)
        t["combine"].append(a.elapsed_time(b))
    for bx in boxes:
        bx.check()
    med = {kk: float(np.median(v[2:] if len(v) > 3 else v)) for kk, v in t.items()}
    row_bytes = T * d_h * 2
    res = {"transport": args.transport, "tokens": T, "d_hidden": d_h,
           "dispatch_us": med["dispatch"] * 1e3, "moe_step_us": med["moe"] * 1e3,
           "combine_us": med["combine"] * 1e3,
           "dispatch_rows_bytes": row_bytes, "dispatch_gbs": row_bytes / (med["dispatch"] / 1e3) / 1e9,
           "combine_bytes_into_owner": row_bytes,
           "how": "1A+1E on two GPUs of one process; each phase alone after a host sync; "
                  "CUDA events on the launching GPU's stream, median"}
    if not args.no_peak:
        n = 1 << 29  # 1 GiB of bf16
        a0 = torch.empty(n, dtype=torch.bfloat16, device="cuda:0")
        a1 = torch.empty(n, dtype=torch.bfloat16, device="cuda:1")
        for src, dst, name in ((a0, a1, "peer_copy_0to1_gbs"), (a1, a0, "peer_copy_1to0_gbs")):
            torch.cuda.set_device(src.device)
            dst.copy_(src)
            torch.cuda.synchronize(0)
            torch.cuda.synchronize(1)
            best = 0.0
            for _ in range(5):
                e0, e1 = ev(), ev()
                s = torch.cuda.current_stream(src.device)
                e0.record(s)
                dst.copy_(src, non_blocking=True)
                e1.record(s)
                torch.cuda.synchronize(src.device)
                best = max(best, 2 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
            res[name] = best
        res["peer_copy_how"] = "torch copy_ between the GPUs (cudaMemcpyPeer path), 1 GiB, best of 5"
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
