"""Summarise CTA 0's per-stage log from a gemm_timeline npz: per token-row
count, the producers' issue lag, the TMA latency (issue -> data seen by the
MMA) and the stage period.   python tools/stage_log.py gpurun_out/tl_x.npz"""
import sys

import numpy as np

TRACE_TILES, TW = 1 << 14, 16
for f in sys.argv[1:]:
    d = np.load(f)["trace"]
    print(f)
    for g, name in enumerate(["gate_up", "down"]):
        sl = d[g][TRACE_TILES - 512:].reshape(-1)[:2048 * 4].reshape(2048, 4).astype(np.int64)
        n = int((sl[:, 0] > 0).sum())
        sl = sl[:n]
        half = sl[:, 3]
        t0 = sl[:, 0].min()
        A, B, F = ((sl[:, i] - t0) / 1e3 for i in range(3))
        print(" ", name, "stages", n)
        for hv in sorted(set(half.tolist())):
            idx = np.nonzero(half == hv)[0]
            idx = idx[idx >= 6]
            if len(idx) < 5:
                continue
            med = lambda x: float(np.median(x))  # noqa: E731
            print("    half %3d n=%4d  B-A %.3f  A-F(n-6) %.3f  B-F(n-6) %.3f  F-max(A,B) %.3f  "
                  "period %.3f" % (hv, len(idx), med(B[idx] - A[idx]), med(A[idx] - F[idx - 6]),
                                   med(B[idx] - F[idx - 6]),
                                   med(F[idx] - np.maximum(A[idx], B[idx])),
                                   med(F[idx] - F[idx - 1])))
