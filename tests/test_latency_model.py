"""The calibrated MoE-layer latency model (latency.cpp:17-32).

CPU: with the reference's parameters (two matrices, max form) the C-ABI model
is the reference's moe_layer_latency to the last bit (oracle restatement, and
oracle/_ref where built); the fit recovers a model's own parameters.
GPU: the layer measured over a grid of (activated experts, routed rows) on
this B200 — the fit's mean relative error <= 10 %, and the constants committed
in profiles/r2/latency_calibration.json predict the same grid within 15 %
(box-to-box spread under the power cap)."""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def J():
    import paper_2512_13525_b200 as J
    return J


def _loads(J, load, routed):
    return [J.InstanceLoad(int(a), int(b)) for a, b in zip(load, routed)]


def test_reference_form_is_the_reference(J, oracle):
    from oracle import REF_SO, Ref
    ref = Ref() if os.path.exists(REF_SO) else None
    rng = np.random.default_rng(7)
    for case in range(200):
        N = int(rng.integers(1, 9))
        load = rng.integers(0, 60, N).astype(np.int32)
        routed = rng.integers(0, 40000, N).astype(np.int64)
        d_h, d_e = int(rng.choice([2048, 4096, 7168])), int(rng.choice([768, 1536, 2048]))
        pf, bw, tl = float(rng.choice([989e12, 1401.8e12])), float(rng.choice([3.35e12, 6.3725e12])), 5e-6
        m = J.reference_latency_model(pf, bw, tl)
        got = J.layer_latency(m, _loads(J, load, routed), d_h, d_e)
        assert got == oracle.moe_layer_latency(load, routed, d_h, d_e, 2, pf, bw, tl), case
        assert got == J.moe_layer_latency(_loads(J, load, routed), d_h, d_e, 2, pf, bw, tl)
        if ref is not None:
            assert got == ref.moe_layer_latency(load, routed, d_h, d_e, 2, pf, bw, tl), case


def test_fit_recovers_parameters(J):
    from paper_2512_13525_b200._lib import LatencyModel
    true = LatencyModel(25e-6, 6.1e12, 1.3e15, 3.0, 3, 2, 3)
    A, b = [], []
    for a in (8, 16, 32, 64, 128):
        for T in (16, 64, 256, 1024, 4096):
            A.append(a)
            b.append(T * 8)
    t = [J.layer_latency(true, [J.InstanceLoad(x, y)], 2048, 768) for x, y in zip(A, b)]
    m, err = J.fit_latency_model(A, b, t, 2048, 768)
    assert err < 1e-3
    for f in ("t_launch", "hbm_bandwidth", "peak_flops"):
        assert abs(getattr(m, f) / getattr(true, f) - 1) < 0.02, f


GRID_A = (8, 32, 128)
GRID_T = (16, 256, 4096)


def measure_grid(J, d_h=2048, d_e=768, k=8, reps=10):
    import ctypes as C
    import torch
    from paper_2512_13525_b200._lib import lib
    from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs
    E = 128
    layer = MoELayer(J.ReplicaMap.from_hosts(1, E, [[0]] * E), d_h, d_e, max(GRID_T), k)
    layer.set_weights(*build_weight_store(layer, seed=1))
    A, b, t = [], [], []
    for a in GRID_A:
        for T in GRID_T:
            rng = np.random.default_rng(a * 100003 + T)
            ex = np.stack([rng.choice(a, k, replace=False) for _ in range(T)]).astype(np.int32)
            ext = torch.from_numpy(ex.ravel()).cuda()
            x, gw = make_inputs(T, k, d_h, 3, "cuda")
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
            A.append(len(np.unique(ex)))
            b.append(T * k)
            t.append(f.value / c.value * 1e-3)
    return A, b, t


@pytest.mark.gpu
def test_calibrated_model_predicts_measured_layer(J):
    from paper_2512_13525_b200._lib import LatencyModel
    A, b, t = measure_grid(J)
    m, err = J.fit_latency_model(A, b, t, 2048, 768)
    assert err <= 0.10, (err, list(zip(A, b, t)))
    cal = json.load(open(os.path.join(ROOT, "profiles", "r2", "latency_calibration.json")))
    c = cal["fitted_model"]
    committed = LatencyModel(c["t_launch_s"], c["hbm_bandwidth_Bps"], c["peak_flops"], c["p"],
                             c["matrices"], c["bytes_per_param"], c["flop_matrices"])
    pred = [J.layer_latency(committed, [J.InstanceLoad(x, y)], 2048, 768) for x, y in zip(A, b)]
    rel = np.abs(np.array(pred) - np.array(t)) / np.array(t)
    assert rel.mean() <= 0.15, list(zip(A, b, t, pred))
