"""A few c2 layer steps (bench's T=4096 workload) — the target of an ncu
capture of the grouped GEMMs:
  ncu -k regex:grouped_gemm --launch-skip 6 --launch-count 2 --set full python tools/ffn_probe.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
rmap, _ = bench.shape_map(J, 1)
layer = MoELayer(rmap, bench.D_H, bench.D_E, T, bench.K_TOP, instance=-1, device=0)
layer.set_weights(*build_weight_store(layer, seed=1))
batches = [torch.from_numpy(b).to(dev) for b in bench.gen_batches(T)]
x, gw = make_inputs(T, bench.K_TOP, bench.D_H, 3, dev)
out = torch.empty_like(x)
for i in range(5):
    layer.forward(x, batches[0], gw, out=out)
torch.cuda.synchronize()
print("ok", T)
