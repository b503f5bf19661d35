"""Host <-> device copy bandwidth with every rank copying at once (pinned
buffers, 64 MiB, both directions concurrently on two streams): what the
box's end-to-end path can get from the host when N GPUs share it.

  torchrun --nproc-per-node N tools/pcie_probe.py
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    ws, rank, local = (int(os.environ.get(k, d)) for k, d in
                       (("WORLD_SIZE", "1"), ("RANK", "0"), ("LOCAL_RANK", "0")))
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = 64 << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for mode in ("h2d", "d2h", "both"):
        for it in range(2):  # warm-up, then timed
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            for _ in range(10):
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(s1):
                        d_in.copy_(h_in, non_blocking=True)
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(s2):
                        h_out.copy_(d_out, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
        res[mode + "_gbs_per_direction"] = 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    allr = [None] * ws
    if ws > 1:
        dist.all_gather_object(allr, res)
    else:
        allr = [res]
    if rank == 0:
        print(json.dumps({"ranks": ws, "per_rank": allr}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
