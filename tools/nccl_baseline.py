"""NCCL baseline for the box exchange: the same bytes the
library's dispatch / combine kernels move, moved by plain NCCL collectives over
NVLink, timed on the device (CUDA events, max over ranks).

  torchrun --nproc-per-node N tools/nccl_baseline.py [--box split|moe-only] [--tokens 4096]

split box (BoxPlan.for_gpus: A attention + M MoE ranks), T = tokens x M:
  dispatch  every attention rank broadcasts its shard (rows + top-k ids + gate
            weights) to the box (NCCL broadcast, one per attention rank);
  combine   every owner receives the sum of the box's partial sums for its
            shard (NCCL reduce of bf16 rows, one per attention rank).
MoE-only box (every rank owns a shard and is an MoE instance), T = tokens x N:
  dispatch  all_gather of the shards; combine  reduce_scatter of the partials.
Prints one JSON line (rank 0).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--box", default="split", choices=["split", "moe-only"])
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--d-hidden", type=int, default=2048)
    ap.add_argument("--top-k", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    ws, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2512_13525_b200.dist import BoxPlan
    from paper_2512_13525_b200.moesim import shard_tokens
    plan = BoxPlan.moe_only(ws) if args.box == "moe-only" else BoxPlan.for_gpus(ws)
    A, M, d_h, k = plan.n_attn, plan.n_moe, args.d_hidden, args.top_k
    T = args.tokens * M
    shards = [shard_tokens(T, A, a) for a in range(A)]
    ta_max = max(c for _, c in shards)
    row_b = d_h * 2 + k * 8  # bytes per token shipped: bf16 row + ids + weights
    s = torch.cuda.current_stream(dev)

    if plan.colocated:
        send = torch.randn(ta_max, row_b // 2, device=dev).bfloat16()   # packed shard
        gathered = torch.empty(ws * ta_max, row_b // 2, dtype=torch.bfloat16, device=dev)
        parts = torch.randn(ws * ta_max, d_h, device=dev).bfloat16()
        mine = torch.empty(ta_max, d_h, dtype=torch.bfloat16, device=dev)

        def dispatch():
            dist.all_gather_into_tensor(gathered, send)

        def combine():
            dist.reduce_scatter_tensor(mine, parts, op=dist.ReduceOp.SUM)
        egress_d = (ws - 1) * ta_max * row_b          # each rank sends its shard to N-1 peers
        egress_c = (ws - 1) * ta_max * d_h * 2
    else:
        bufs = [torch.randn(c, row_b // 2, device=dev).bfloat16() for _, c in shards]
        parts = [torch.randn(c, d_h, device=dev).bfloat16() for _, c in shards]

        def dispatch():
            for a in range(A):
                dist.broadcast(bufs[a], src=a)

        def combine():
            for a in range(A):
                dist.reduce(parts[a], dst=a, op=dist.ReduceOp.SUM)
        ta = shards[0][1]
        egress_d = M * ta * row_b                      # what an attention rank must deliver
        egress_c = M * ta * d_h * 2                    # what an owner must receive

    res = {}
    for name, fn in (("dispatch", dispatch), ("combine", combine)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.iters):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = float(t.item())
    if rank == 0:
        print(json.dumps({
            "what": "NCCL collectives moving the box exchange's bytes",
            "box": args.box, "plan": f"{A}A+{M}E" if not plan.colocated else f"{ws} colocated",
            "tokens_per_step": T, "d_hidden": d_h, "top_k": k,
            "nccl": torch.cuda.nccl.version(),
            "dispatch_us": res["dispatch"] * 1e3, "combine_us": res["combine"] * 1e3,
            "dispatch_bytes": egress_d, "combine_bytes": egress_c,
            "dispatch_gbs": egress_d / (res["dispatch"] / 1e3) / 1e9,
            "combine_gbs": egress_c / (res["combine"] / 1e3) / 1e9,
            "how": "CUDA events over 20 back-to-back ops after 5 warm-up, max over ranks"}),
            flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
