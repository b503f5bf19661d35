"""Scheduler µs/iter sweep on the GPU (graph-replayed) + in-kernel phase trace,
with the reference CPU schedule()/schedule_reference() timed on the same
batches when oracle/_ref is present.  Prints one JSON line per (config, T).

  python tools/sched_sweep.py [--configs c1_uniform,c2,...] [--tokens 32,256,4096]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from routing import RoutingPattern, gen_batch  # noqa: E402

import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200._lib import lib  # noqa: E402

PATTERNS = {
    "c1_uniform": (lambda: RoutingPattern.uniform(64), 0x5EED),
    "c1_gaussian": (lambda: RoutingPattern.gaussian(64, 0.15), 0x5EED),
    "c2": (lambda: RoutingPattern.zipf(128, 1.0), 0x30),
    "c2_m3": (lambda: RoutingPattern.zipf(128, 1.0), 0x30),
    "c3": (lambda: RoutingPattern.zipf(128, 1.0), 0x235),
    "c4_n2": (lambda: RoutingPattern.zipf(256, 1.0), 0xD5),
    "c4_n4": (lambda: RoutingPattern.zipf(256, 1.0), 0xD5),
    "c4_n8": (lambda: RoutingPattern.zipf(256, 1.0), 0xD5),
    "c5": (lambda: RoutingPattern.zipf(256, 1.2), 0x5A),
}
PHASES = ["load+stage", "pass1", "scan+pin", "greedy", "finish+scan", "pass2"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1_uniform,c2,c3,c4_n8,c5")
    ap.add_argument("--tokens", default="32,64,128,256,512,1024,2048,4096")
    ap.add_argument("--cpu", action="store_true")
    args = ap.parse_args()
    ref = None
    if args.cpu:
        from oracle import CSRMap, Ref
        try:
            ref = Ref()
        except FileNotFoundError:
            ref = None
    for name in args.configs.split(","):
        rm = J.config_map(name)
        pat_fn, seed = PATTERNS[name]
        pat = pat_fn()
        s = J.Scheduler(rm)
        for T in (int(t) for t in args.tokens.split(",")):
            b = gen_batch(pat, T, 8, seed, T)
            d = torch.from_numpy(b.experts).cuda()
            us = s.time_schedule(d, T, 8, reps=51)
            ns = (C.c_int64 * 8)()
            lib.janus_trace_schedule(s.ctx, d.data_ptr(), T, 8, ns)
            a = s.schedule(b)
            rnd = s.schedule_random(b, 7)
            row = {"config": name, "T": T, "gpu_us_per_iter": us,
                   "trace_us": {PHASES[i]: (ns[i + 1] - ns[i]) / 1e3 for i in range(6)},
                   "sm_ghz": (ns[7] / ns[6]) if ns[7] and ns[6] else None,
                   "max_load_aebs": a.max_load(), "max_load_random": rnd.max_load(),
                   "activated": int((a.expert_instance >= 0).sum())}
            if ref is not None:
                m = CSRMap(rm.num_experts, rm.num_instances, rm.slots_per_instance, *rm.csr())
                row["cpu_schedule_us"] = ref.time_schedule(b.experts, T, 8, m, "schedule",
                                                           reps=101)
                row["cpu_schedule_reference_us"] = ref.time_schedule(b.experts, T, 8, m,
                                                                     "reference", reps=101)
            print(json.dumps(row), flush=True)
        s.close()


if __name__ == "__main__":
    main()
