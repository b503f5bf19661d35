"""Summarise gpurun_out logs: python tools/show.py TAG"""
import json
import sys

tag = sys.argv[1]
for l in open(f"gpurun_out/{tag}_sweep.log"):
    try:
        r = json.loads(l)
    except Exception:
        print(l[:300].rstrip())
        continue
    t = r["trace_us"]
    print(f"{r['config']:12s} T={r['T']:5d} gpu={r['gpu_us_per_iter']:6.2f}us ml {r['max_load_aebs']}/"
          f"{r['max_load_random']} trace", " ".join(f"{v:5.2f}" for v in t.values()))
for T in (256, 4096):
    try:
        lines = open(f"gpurun_out/{tag}_bench{T}.log").read().strip().splitlines()
        r = json.loads(lines[-1])
        rf = r["roofline"]
        print(f"T={T}: {r['value']:.4g} tok/s, step {r['ms_per_step']*1e3:.1f} us, ffn "
              f"{rf['ffn_us_per_step']:.1f} us ({rf['bound']} {rf['frac']:.3f}, hbm {rf['hbm_frac']:.3f},"
              f" tensor {rf['tensor_frac']:.3f}), e2e {r['e2e']['value']:.4g}, sched "
              f"{r['scheduler']['us_per_iter']:.2f} us, clocks {r['clocks']}")
    except Exception as ex:
        print(T, "bench:", ex, open(f"gpurun_out/{tag}_bench{T}.log").read()[-1500:])
