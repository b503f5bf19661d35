"""Gating kernel timing probe (CUDA-graph replay, so host launch cost is out):
python tools/gate_probe.py [T ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200.moe import MoELayer, make_inputs, router_weights  # noqa: E402

dev = torch.device("cuda", 0)
rm = J.config_map("c2")
for T in [int(a) for a in sys.argv[1:]] or [256, 4096]:
    L = MoELayer(rm, 2048, 768, T, 8, device=0)
    x, _ = make_inputs(T, 8, 2048, 5, dev)
    wr = router_weights(128, 2048, 9, dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            L.gate(x, wr)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                L.gate(x, wr)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"gate T={T}: {a.elapsed_time(b) / 200 * 1e3:.1f} us", flush=True)
