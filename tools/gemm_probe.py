"""Grouped-GEMM efficiency probe: FFN time (library events, no graph) for
synthetic routings that isolate the tensor-bound and weight-bound regimes.

  python tools/gemm_probe.py [--tokens 4096]

  dense8   E=8,   every token -> experts 0..7   (8 groups of T rows: tensor-bound)
  uni128   E=128, uniform top-8                 (128 groups of ~T/16 rows)
  c2       the bench workload (c2 map, Zipf 1.0)
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
from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs  # noqa: E402

D_H, D_E, K = 2048, 768, 8
PEAK_TF, PEAK_BW = 1721.9, 6372.5


def probe(name, rmap, experts, T, steps=50):
    dev = torch.device("cuda", 0)
    layer = MoELayer(rmap, D_H, D_E, T, K, instance=-1, device=0)
    w13, w2 = build_weight_store(layer, seed=1)
    layer.set_weights(w13, w2)
    ex = torch.from_numpy(np.ascontiguousarray(experts, dtype=np.int32)).to(dev)
    x, gw = make_inputs(T, K, D_H, 3, dev)
    out = torch.empty_like(x)
    for _ in range(5):
        layer.forward(x, ex, gw, out=out)
    torch.cuda.synchronize()
    lib.janus_profile(layer.ctx, 1)
    for _ in range(steps):
        layer.forward(x, ex, gw, out=out)
    torch.cuda.synchronize()
    s_ms, f_ms, calls = C.c_double(), C.c_double(), C.c_int()
    lib.janus_profile_read(layer.ctx, C.byref(s_ms), C.byref(f_ms), C.byref(calls))
    lib.janus_profile(layer.ctx, 0)
    ffn_us = f_ms.value / calls.value * 1e3
    A = len(np.unique(experts))
    flops = 6.0 * D_H * D_E * T * K
    wbytes = A * 3 * D_H * D_E * 2
    print(json.dumps({"probe": name, "T": T, "active_experts": A, "ffn_us": round(ffn_us, 1),
                      "tflops": round(flops / ffn_us / 1e6, 1),
                      "tensor_frac": round(flops / ffn_us / 1e6 / PEAK_TF, 3),
                      "weight_GBps": round(wbytes / ffn_us / 1e3, 1),
                      "hbm_frac": round(wbytes / ffn_us / 1e3 / PEAK_BW, 3)}), flush=True)
    del layer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--probes", default="dense8,uni128,c2")
    a = ap.parse_args()
    T = a.tokens
    for name in a.probes.split(","):
        if name == "dense8":
            rmap = J.ReplicaMap.from_hosts(1, 8, [[0]] * 8)
            ex = np.tile(np.arange(8, dtype=np.int32), T)
        elif name == "bal128":  # every expert exactly T*8/128 rows
            rmap = J.ReplicaMap.from_hosts(1, 128, [[0]] * 128)
            ex = ((np.arange(T)[:, None] * 8 + np.arange(8)[None, :]) % 128).astype(np.int32).ravel()
        elif name == "uni128":
            rmap = J.ReplicaMap.from_hosts(1, 128, [[0]] * 128)
            ex = gen_batch(RoutingPattern.uniform(128), T, K, 0x77, 0).experts
        else:
            rmap = J.config_map("c2")
            ex = gen_batch(RoutingPattern.zipf(128, 1.0), T, K, 0x30, T * 1000).experts
        probe(name, rmap, ex, T)


if __name__ == "__main__":
    main()
