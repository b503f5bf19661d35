"""Which part of bench.py's run before its e2e leg slows the host link: the e2e
leg measured fresh, after the clock-sampled timed leg, after the profiled leg.
  python tools/e2e_ab.py"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200._lib import lib  # noqa: E402
from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs  # noqa: E402


def main():
    T, n = 4096, 100
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

    def e2e():
        for i in range(5):
            layer.forward_host_async(xh, bh[i % len(bh)], gh, oh)
        layer.host_sync()
        t0 = time.perf_counter()
        for i in range(n):
            layer.forward_host_async(xh, bh[i % len(bh)], gh, oh)
        layer.host_sync()
        return round((time.perf_counter() - t0) / n * 1e6, 1)

    def steps(k):
        for i in range(k):
            layer.forward(x, batches[i % len(batches)], gw, out=out)
        torch.cuda.synchronize()

    res = {"fresh": [e2e(), e2e()]}
    steps(50)
    res["after_graph_steps"] = e2e()
    with bench.ClockSampler(0):
        steps(200)
    res["after_sampler"] = [e2e(), e2e()]
    time.sleep(2)
    res["after_sampler_2s"] = e2e()
    lib.janus_profile(layer.ctx, 1)
    steps(50)
    lib.janus_profile(layer.ctx, 0)
    res["after_profile"] = [e2e(), e2e()]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
