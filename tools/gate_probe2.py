import sys, os, torch
sys.path.insert(0, "/root/repo")
import paper_2512_13525_b200 as J
from paper_2512_13525_b200.moe import MoELayer, make_inputs, router_weights
dev = torch.device("cuda", 0)
for (T, d_h, E) in [(128, 256, 16), (128, 2048, 16), (128, 2048, 128), (128, 256, 128)]:
    rm = J.ReplicaMap.from_hosts(1, E, [[0]] * E)
    L = MoELayer(rm, d_h, 128, T, 4, device=0)
    x, _ = make_inputs(T, 4, d_h, 5, dev)
    wr = router_weights(E, d_h, 9, dev)
    for _ in range(3):
        L.gate(x, wr)
    torch.cuda.synchronize()
