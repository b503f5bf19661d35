"""Tile timeline of the two grouped GEMMs (K4) of one c2 layer step, from the
kernel's own %globaltimer stamps (JANUS_GEMM_TRACE=1, csrc/gemm.cu): per tile
the draw, MMA start, accumulator-ready and epilogue-done times, the SM and the
(group, rows, m-block).  Prints where the step's time goes — per-tile
efficiency against the pair's fair share of HBM and tensor throughput, SM-pair
idle time at each kernel's tail, the gap between the kernels, and how many
tensor-bound vs weight-streaming tiles run at once.

  JANUS_GEMM_TRACE=1 python tools/gemm_timeline.py [--tokens 4096] [--out gpurun_out/timeline.npz]
"""
import argparse
import ctypes
import json
import os
import sys
from collections import Counter

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TRACE_TILES = 1 << 14
TW = 16  # trace words per tile


def analyse(tr, K, name, hbm, tf, pairs):
    """Summary of one GEMM's tiles.  Ideal tile times use the pair's fair share
    of the measured peaks (HBM / pairs, bf16 / pairs); a weight block is read
    from DRAM once per group (its n-tiles share it in L2), token rows from L2."""
    used = tr[:, 0] > 0
    tr = tr[used].astype(np.int64)
    draw, mma, acc, epi = (tr[:, i] for i in range(4))
    meta = tr[:, 4]
    sm, q = meta & 0xFFFF, (meta >> 16) & 0xFFFF
    rows, m = (meta >> 32) & 0xFFFF, (meta >> 48) & 0xFFFF
    t0, end = draw.min(), epi.max()
    span = (end - t0) / 1e3
    cnt = Counter(zip(q.tolist(), m.tolist()))
    nt = np.array([cnt[(a, b)] for a, b in zip(q.tolist(), m.tolist())])
    grows = Counter()
    for a, r, b in zip(q.tolist(), rows.tolist(), m.tolist()):
        if b == 0:
            grows[a] += r
    G = np.array([grows[a] for a in q.tolist()])
    t_mem = (256.0 * K * 2 / nt) / (hbm * 1e9 / pairs) * 1e6
    t_tc = 2.0 * 256 * rows * K / (tf * 1e12 / pairs) * 1e6
    dur = (acc - mma) / 1e3
    classes = []
    for lo, hi in ((0, 128), (128, 256), (256, 512), (512, 1024), (1024, 1 << 30)):
        s = (G >= lo) & (G < hi)
        if s.any():
            classes.append(dict(group_rows=[lo, hi], tiles=int(s.sum()),
                                groups=len(set(q[s].tolist())),
                                tile_us_median=float(np.median(dur[s])),
                                pair_us=float(dur[s].sum() / pairs),
                                weight_stream_us=float(t_mem[s].sum() / pairs),
                                tensor_us=float(t_tc[s].sum() / pairs),
                                weight_gbs_per_pair_median=float(np.median(
                                    (256.0 * K * 2 / dur[s] / 1e3)[G[s] < 256]))
                                if (G[s] < 256).any() else None))
    idle = []
    for pr in set((sm >> 1).tolist()):
        i = np.nonzero((sm >> 1) == pr)[0]
        o = i[np.argsort(mma[i])]
        idle.append(((mma[o[1:]] - acc[o[:-1]]).clip(0)).sum() / 1e3)
    last = Counter()
    for pr, e in zip((sm >> 1).tolist(), epi.tolist()):
        last[pr] = max(last[pr], e)
    tail = np.array([(end - v) / 1e3 for v in last.values()])
    ts = np.linspace(t0, end, 12)
    hot = G >= 256
    tq, issued = tr[:, 5], tr[:, 7]
    wait = (tr[:, 6] & 0xFFFFFFFF) / 1e3
    tq_wait = (tr[:, 6] >> 32) / 1e3
    # the issuer's time per tile: tile-queue wait, accumulator (epilogue) wait,
    # stage (data) waits, the rest = issuing
    acc_wait = (mma - tq) / 1e3 - tq_wait
    issue_span = (issued - mma) / 1e3
    prod = {"A_acquire": float(tr[:, 8].sum() / 1e3 / pairs), "A_loop": float(tr[:, 9].sum() / 1e3 / pairs),
            "B_acquire": float(tr[:, 10].sum() / 1e3 / pairs), "B_loop": float(tr[:, 11].sum() / 1e3 / pairs)}
    res = {"gemm": name, "tiles": int(len(tr)), "span_us": span, "producer_pair_us": prod,
           "issuer_pair_us": {"tile_queue_wait": float(tq_wait.sum() / pairs),
                              "acc_free_wait": float(acc_wait.sum() / pairs),
                              "stage_wait": float(wait.sum() / pairs),
                              "issuing": float((issue_span - wait).sum() / pairs)},
           "pair_busy_frac": float(dur.sum() / pairs / span),
           "weight_stream_us_total": float(t_mem.sum() / pairs),
           "tensor_us_total": float(t_tc.sum() / pairs),
           "classes": classes,
           "pair_idle_between_tiles_us_mean": float(np.mean(idle)),
           "tail_idle_us_mean": float(tail.mean()), "tail_idle_us_max": float(tail.max()),
           "active_hot_group_tiles": [int(np.sum(hot & (mma <= t) & (acc > t))) for t in ts],
           "active_cold_group_tiles": [int(np.sum(~hot & (mma <= t) & (acc > t))) for t in ts]}
    return res, (t0, end)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gemm_timeline.npz"))
    args = ap.parse_args()
    assert os.environ.get("JANUS_GEMM_TRACE") == "1", "run with JANUS_GEMM_TRACE=1"
    import torch

    import bench
    import paper_2512_13525_b200 as J
    from paper_2512_13525_b200._lib import lib
    from paper_2512_13525_b200.moe import MoELayer, build_weight_store, make_inputs

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    T = args.tokens
    rmap, _ = bench.shape_map(J, 1)
    layer = MoELayer(rmap, bench.D_H, bench.D_E, T, bench.K_TOP, instance=-1, device=0)
    layer.set_weights(*build_weight_store(layer, seed=1))
    batches = [torch.from_numpy(b).to(dev) for b in bench.gen_batches(T)]
    x, gw = make_inputs(T, bench.K_TOP, bench.D_H, 3, dev)
    out = torch.empty_like(x)
    for i in range(6):
        layer.forward(x, batches[i % len(batches)], gw, out=out)
    torch.cuda.synchronize()
    fn = lib.janus_debug_ffn_trace
    buf = np.zeros(2 * TRACE_TILES * TW, dtype=np.uint64)
    assert fn(buf.ctypes.data, buf.size) == 0  # read + clear the warm-up steps' stamps
    # one more step, after an L2 flush, then read its timeline
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush.zero_()
    layer.forward(x, batches[0], gw, out=out)
    torch.cuda.synchronize()
    assert fn(buf.ctypes.data, buf.size) == 0
    buf = buf.reshape(2, TRACE_TILES, TW)
    hbm, tf, _, _ = bench.peaks()
    pairs = torch.cuda.get_device_properties(0).multi_processor_count // 2
    nt = TRACE_TILES - 512  # the rest: stage log of CTA 0
    r1, (a0, a1) = analyse(buf[0][:nt], bench.D_H, "gate_up", hbm, tf, pairs)
    r2, (b0, b1) = analyse(buf[1][:nt], bench.D_E, "down", hbm, tf, pairs)
    res = {"T": T, "step_gemm_span_us": (b1 - a0) / 1e3, "gap_us": (b0 - a1) / 1e3,
           "overlap_note": "gap < 0: the down GEMM's first draw precedes gate/up's last epilogue (PDL)",
           "gemms": [r1, r2]}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.savez_compressed(args.out, trace=buf)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
