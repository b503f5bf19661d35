"""One MoE rank's layer on one GPU (instance filter, T tokens routed over M
instances), for ncu launch lists of the box path's MoE side.

  python tools/moe_rank_probe.py --moe 3 --tokens-per-gpu 4096 [--steps 20]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from routing import RoutingPattern, gen_batch  # noqa: E402
import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--moe", type=int, default=3)
ap.add_argument("--tokens-per-gpu", type=int, default=4096)
ap.add_argument("--instance", type=int, default=0)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--gate", action="store_true", help="MoE-side gating (forward_gated)")
a = ap.parse_args()
T = a.tokens_per_gpu * a.moe
dev = torch.device("cuda", 0)
rmap = J.config_map("c2" if a.moe == 1 else f"c2_m{a.moe}")
layer = MoELayer(rmap, 2048, 768, T, 8, instance=a.instance, device=0)
layer.set_weights(*build_weight_store(layer, seed=1))
ex = torch.from_numpy(gen_batch(RoutingPattern.zipf(128, 1.0), T, 8, 0x30, T * 1000).experts).to(dev)
x, gw = make_inputs(T, 8, 2048, 3, dev)
out = torch.empty_like(x)
if a.gate:
    from paper_2512_13525_b200.moe import router_weights
    layer.set_router(router_weights(128, 2048, 13, dev))
fwd = (lambda: layer.forward_gated(x, out=out)) if a.gate else (lambda: layer.forward(x, ex, gw, out=out))
for _ in range(a.steps):
    fwd()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.steps):
    fwd()
e.record()
torch.cuda.synchronize()
print(f"T={T} instance {a.instance}/{a.moe}: {s.elapsed_time(e) / a.steps * 1e3:.1f} us/step (graph)")
