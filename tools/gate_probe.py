"""Gating kernel timing probe: python tools/gate_probe.py [T ...]"""
import sys
import os
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
    for _ in range(3):
        L.gate(x, wr)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        L.gate(x, wr)
    e.record()
    torch.cuda.synchronize()
    print(f"gate T={T}: {s.elapsed_time(e) / 50 * 1e3:.1f} us")
