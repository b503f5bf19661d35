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


def bf16_round(a):
    """fp32 -> nearest-even bf16 -> fp32 (numpy)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def moe_reference_device_exact(oracle, x_u16, ex, w, weights_of, nthreads=8):
    """The device's rounding points, restated: h rounded to bf16 (between the
    GEMMs), y rounded to bf16 (the down GEMM's output rows), the combine
    out[t] = fma(w_j, y_j, acc) over j ascending in fp32 (K5, ffn.cu), out
    rounded to bf16.  Returns (out as the fp32 values of bf16 numbers,
    sum_j |w_j y_j| per element)."""
    T, k = ex.shape
    d_h = x_u16.shape[1]
    y = np.zeros((T, k, d_h), np.float32)
    by_e = {}
    for t in range(T):
        for j in range(k):
            by_e.setdefault(int(ex[t, j]), []).append((t, j))
    for e, lst in sorted(by_e.items()):
        wg, wu, wd = weights_of(e)
        rows = np.stack([x_u16[t] for t, _ in lst])
        ye = bf16_round(oracle.expert_swiglu(rows, wg, wu, wd, round_h=True, nthreads=nthreads))
        for r, (t, j) in enumerate(lst):
            y[t, j] = ye[r]
    acc = np.zeros((T, d_h), np.float32)
    mag = np.zeros((T, d_h), np.float64)
    for j in range(k):  # fma: the f32 product is exact in f64; one rounding to f32
        p = w[:, j:j + 1].astype(np.float64) * y[:, j].astype(np.float64)
        acc = (acc.astype(np.float64) + p).astype(np.float32)
        mag += np.abs(p)
    return bf16_round(acc), mag


def ulp_stats(dev, ref, mag):
    """dev, ref: fp32 values of bf16 numbers; mag = sum_j |w_j y_j| (the
    combine's magnitude).  (fraction bit-identical, max |dev - ref| in bf16
    ulps of mag) — a 1-ulp flip of some y_j's rounding moves out by at most
    w_j ulp(y_j) <= ulp(mag), whatever cancellation the sum has."""
    same = float(np.mean(dev.view(np.uint32) == ref.view(np.uint32)))
    e = np.floor(np.log2(np.maximum(np.abs(mag), 1e-30)))
    ulp = np.exp2(e - 7)
    return same, float(np.max(np.abs(dev - ref) / ulp))
