"""Latency-model calibration: measure the grouped SwiGLU FFN
on one B200 over a grid of (A activated experts, b routed tokens) and fit the
reference's per-instance model (latency.cpp:17-24)

    t = t_launch + max(A * W_e / beta, F(b) / pi)

where the reference uses W_e = 2 * d_h * d_e * bpp and F(b) = 2 * b * d_h * d_e
(two matrices) and the device computes SwiGLU (three matrices: W_e and F(b)
x 1.5).  Prints one JSON document: the grid, the reference's prediction with
MEASURED_PEAKS (uncalibrated), and the fitted (t_launch, beta, pi) of the
three-matrix form with its residuals.

  python tools/calibrate_latency.py [--d-h 2048 --d-e 768 --out profiles/r2/latency_calibration.json]
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

import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200._lib import lib  # noqa: E402
from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs  # noqa: E402


def measure(layer, A, T, k, dev, reps=20):
    rng = np.random.default_rng(A * 100003 + T)
    ex = np.stack([rng.choice(A, k, replace=False) for _ in range(T)]).astype(np.int32).ravel()
    ext = torch.from_numpy(ex).to(dev)
    x, gw = make_inputs(T, k, layer.d_h, 3, dev)
    out = torch.empty_like(x)
    for _ in range(3):
        layer.forward(x, ext, gw, out=out)
    torch.cuda.synchronize()
    lib.janus_profile(layer.ctx, 1)
    for _ in range(reps):
        layer.forward(x, ext, gw, out=out)
    torch.cuda.synchronize()
    s, f, c = C.c_double(), C.c_double(), C.c_int()
    lib.janus_profile_read(layer.ctx, C.byref(s), C.byref(f), C.byref(c))
    lib.janus_profile(layer.ctx, 0)
    return f.value / c.value * 1e-3, len(np.unique(ex))  # seconds, activated


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d-h", type=int, default=2048)
    ap.add_argument("--d-e", type=int, default=768)
    ap.add_argument("--experts", type=int, default=128)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    E, k, d_h, d_e = a.experts, a.k, a.d_h, a.d_e
    rmap = J.ReplicaMap.from_hosts(1, E, [[0]] * E)
    T_max = 4096
    layer = MoELayer(rmap, d_h, d_e, T_max, k, device=0)
    layer.set_weights(*build_weight_store(layer, seed=1))
    pts = []
    for A in (8, 16, 32, 64, 128):
        for T in (16, 64, 256, 1024, 4096):
            if A < k:
                continue
            t, act = measure(layer, A, T, k, dev)
            pts.append({"A": act, "b": T * k, "T": T, "us": t * 1e6})
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    beta0, pi0 = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
    A = [p["A"] for p in pts]
    b = [p["b"] for p in pts]
    tv = np.array([p["us"] for p in pts]) * 1e-6
    ref = J.reference_latency_model(pi0, beta0, 5e-6)  # the model as shipped, measured peaks
    for p in pts:
        p["ref_model_us"] = 1e6 * J.layer_latency(ref, [J.InstanceLoad(p["A"], p["b"])], d_h, d_e)
    # the calibrated form through the C ABI (janus_latency_fit): SwiGLU
    # accounting (3 weight matrices, 3 matrices of FLOPs per row), p-norm blend
    m, err = J.fit_latency_model(A, b, tv, d_h, d_e)
    for p in pts:
        p["fit_us"] = 1e6 * J.layer_latency(m, [J.InstanceLoad(p["A"], p["b"])], d_h, d_e)
    res = {
        "shape": {"experts": E, "top_k": k, "d_hidden": d_h, "d_expert": d_e},
        "reference_model": {"form": "t_launch + max(A*2*d_h*d_e*bpp/beta, 2*b*d_h*d_e/pi) "
                                    "(latency.cpp:17-24), MEASURED_PEAKS",
                            "mean_abs_rel_err": float(np.mean(np.abs(
                                np.array([p["ref_model_us"] for p in pts]) * 1e-6 - tv) / tv))},
        "fitted_model": {"form": "t_launch + (mem^p + comp^p)^(1/p), mem = A*3*d_h*d_e*2/beta, "
                                 "comp = b*6*d_h*d_e/pi (janus_latency_fit)",
                         "t_launch_s": m.t_launch, "hbm_bandwidth_Bps": m.hbm_bandwidth,
                         "peak_flops": m.peak_flops, "p": m.p, "matrices": m.matrices,
                         "bytes_per_param": m.bytes_per_param, "flop_matrices": m.flop_matrices,
                         "mean_abs_rel_err": err},
        "points": pts,
    }
    txt = json.dumps(res, indent=1)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")


if __name__ == "__main__":
    main()
