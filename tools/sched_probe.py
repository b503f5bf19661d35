"""A few scheduler passes on one config/T (no graph) — the target of an ncu
capture of the scheduler kernel.  python tools/sched_probe.py [config] [T]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from routing import RoutingPattern, gen_batch  # noqa: E402
import paper_2512_13525_b200 as J  # noqa: E402

PATS = {"c5": (256, 1.2, 0x5A), "c2": (128, 1.0, 0x30), "c3": (128, 1.0, 0x235)}
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
E, s, seed = PATS[name]
rm = J.config_map(name)
sch = J.Scheduler(rm)
b = gen_batch(RoutingPattern.zipf(E, s), T, 8, seed, T)
d = torch.from_numpy(b.experts).cuda()
S, N, R = T * 8, rm.num_instances, int(rm.csr()[0][-1])
z = lambda n, dt=torch.int32: torch.zeros(n, dtype=dt, device="cuda")  # noqa: E731
out = dict(instance=z(S), replica=z(S), expert_instance=z(E), load=z(N),
           routed_tokens=z(N, torch.int64), expert_tokens=z(E, torch.int64), slot_row=z(S),
           row_slot=z(S), group_off=z(R + 1), status=z(2))
for _ in range(8):
    sch.schedule_async(d, T, 8, out)
torch.cuda.synchronize()
a = sch.schedule(b)
print("ok", name, T, a.max_load())
