#!/bin/bash
# scheduler A/B (JANUS_LIB=old/new .so), interleaved; bit-exact tests of the new one
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/sched_ab; mkdir -p $O; rm -f $O/*.jsonl
timeout 900 python -m pytest tests/test_gpu_schedule.py -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for r in 1 2; do for v in old new; do
  JANUS_LIB=$PWD/abtmp/$v.so timeout 300 python tools/sched_sweep.py --configs c2,c5 --tokens 512,1024,2048,4096 >> $O/$v.jsonl 2>> $O/err.txt
done; done
python - <<'PY'
import json
for v in ("old","new"):
    rows=[json.loads(l) for l in open(f"gpurun_out/sched_ab/{v}.jsonl")]
    for r in rows: print(v, r["config"], r["T"], round(r["gpu_us_per_iter"],2), {k: round(x,2) for k,x in r["trace_us"].items()})
PY
