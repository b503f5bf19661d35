"""What bounds the e2e (host-buffer) number: the bench's pipelined host API
against the same copies without the layer, and the layer without copies.
  python tools/e2e_probe.py [--tokens 4096] [--steps 50]"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    T, n = args.tokens, args.steps
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    rmap, _ = bench.shape_map(J, 1)
    layer = MoELayer(rmap, bench.D_H, bench.D_E, T, bench.K_TOP, instance=-1, device=0)
    layer.set_weights(*build_weight_store(layer, seed=1))
    batches = [torch.from_numpy(b).to(dev) for b in bench.gen_batches(T)]
    x, gw = make_inputs(T, bench.K_TOP, bench.D_H, 3, dev)
    out = torch.empty_like(x)
    xh, gh = x.cpu().pin_memory(), gw.cpu().pin_memory()
    bh = [b.cpu().pin_memory() for b in batches]
    oh = torch.empty(T, bench.D_H, dtype=torch.bfloat16).pin_memory()
    res = {"T": T, "steps": n}
    # layer only (graph replay, device buffers)
    for i in range(5):
        layer.forward(x, batches[i % len(batches)], gw, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        layer.forward(x, batches[i % len(batches)], gw, out=out)
    torch.cuda.synchronize()
    res["layer_only_us"] = (time.perf_counter() - t0) / n * 1e6
    # e2e: the bench's pipelined host API
    for i in range(5):
        layer.forward_host_async(xh, bh[i % len(bh)], gh, oh)
    layer.host_sync()
    t0 = time.perf_counter()
    for i in range(n):
        layer.forward_host_async(xh, bh[i % len(bh)], gh, oh)
    layer.host_sync()
    res["e2e_us"] = (time.perf_counter() - t0) / n * 1e6
    # the same copies, no layer: H2D on one stream, D2H on another, 3 buffer sets
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    xs = [torch.empty_like(x) for _ in range(3)]
    bs = [torch.empty_like(batches[0]) for _ in range(3)]
    gs = [torch.empty_like(gw) for _ in range(3)]
    os_ = [torch.empty_like(x) for _ in range(3)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        k = i % 3
        with torch.cuda.stream(h2d):
            xs[k].copy_(xh, non_blocking=True)
            bs[k].copy_(bh[i % len(bh)], non_blocking=True)
            gs[k].copy_(gh, non_blocking=True)
        with torch.cuda.stream(d2h):
            oh.copy_(os_[k], non_blocking=True)
    torch.cuda.synchronize()
    res["copies_only_us"] = (time.perf_counter() - t0) / n * 1e6
    # the same copies split over two streams per direction (two DMA engines each)
    hs = [torch.cuda.Stream() for _ in range(2)]
    ds = [torch.cuda.Stream() for _ in range(2)]
    half = T // 2
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        k = i % 3
        for j in range(2):
            with torch.cuda.stream(hs[j]):
                xs[k][j * half:(j + 1) * half].copy_(xh[j * half:(j + 1) * half], non_blocking=True)
                if j == 0:
                    bs[k].copy_(bh[i % len(bh)], non_blocking=True)
                else:
                    gs[k].copy_(gh, non_blocking=True)
            with torch.cuda.stream(ds[j]):
                oh[j * half:(j + 1) * half].copy_(os_[k][j * half:(j + 1) * half], non_blocking=True)
    torch.cuda.synchronize()
    res["copies_2streams_us"] = (time.perf_counter() - t0) / n * 1e6
    # one direction at a time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        xs[i % 3].copy_(xh, non_blocking=True)
    torch.cuda.synchronize()
    res["h2d_only_us"] = (time.perf_counter() - t0) / n * 1e6
    t0 = time.perf_counter()
    for i in range(n):
        oh.copy_(os_[i % 3], non_blocking=True)
    torch.cuda.synchronize()
    res["d2h_only_us"] = (time.perf_counter() - t0) / n * 1e6
    res["h2d_bytes"] = x.numel() * 2 + batches[0].numel() * 4 + gw.numel() * 4
    res["d2h_bytes"] = out.numel() * 2
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
