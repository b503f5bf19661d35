"""fp32 references of the MoE layer's output for the GPU parity tests (test
infrastructure: the oracle's SwiGLU expert FFN and combine, oracle/oracle.c).

Two references, both from the same bf16 inputs and weights:
  * ``round_h=False`` — the pure fp32 layer: h and y stay fp32, out in fp32;
  * ``round_h=True``  — h rounded to bf16 where the device rounds it (between its
    gate/up and down GEMMs).
"""
import numpy as np


def u16(t):
    import torch
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def moe_reference(oracle, x_u16, ex, w, weights_of, round_h, mask=None, nthreads=8):
    """out[t] = sum_j w[t,j] * swiglu_{ex[t,j]}(x[t]) in fp32 for every token.

    ex, w: [T, k]; weights_of(e) -> (wg [d_e,d_h], wu [d_e,d_h], wd [d_h,d_e])
    as bf16 bit patterns; mask [T, k] bool (optional): only those slots count."""
    T, k = ex.shape
    d_h = x_u16.shape[1]
    out = np.zeros((T, d_h), np.float32)
    by_e = {}
    for t in range(T):
        for j in range(k):
            if mask is None or mask[t, j]:
                by_e.setdefault(int(ex[t, j]), []).append((t, j))
    for e, lst in sorted(by_e.items()):
        wg, wu, wd = weights_of(e)
        rows = np.stack([x_u16[t] for t, _ in lst])
        y = oracle.expert_swiglu(rows, wg, wu, wd, round_h=round_h, nthreads=nthreads)
        for r, (t, j) in enumerate(lst):
            out[t] += w[t, j] * y[r]
    return out


def err_stats(dev, ref):
    """(max |dev - ref| / rms(ref), rms(ref))."""
    rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2))) or 1.0
    return float(np.abs(dev - ref).max() / rms), rms


def assert_close(dev, ref, rtol, atol, what=""):
    """|dev - ref| <= rtol * |ref| + atol * rms(ref) per element."""
    rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2))) or 1.0
    err = np.abs(dev - ref)
    bad = err > rtol * np.abs(ref) + atol * rms
    assert not bad.any(), (f"{what}: {bad.sum()} / {bad.size} outside tolerance; max err "
                           f"{err.max():.4g}, rms(ref) {rms:.4g}")
    return float(err.max() / rms)
