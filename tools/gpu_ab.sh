# usage: bash tools/gpu_ab.sh TAG VAR "v1 v2 ..."  — pytest -m gpu once, then bench T=256/4096 per env value
TAG=$1; VAR=$2; VALS=$3
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 || { echo smoke failed; tail -5 gpurun_out/${TAG}_smoke.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/${TAG}_pytest.log
for v in $VALS; do
  for T in 256 4096; do
    env $VAR=$v timeout -s KILL 300 python bench.py --tokens $T --steps 300 --no-cpu > gpurun_out/${TAG}_${v}_t$T.log 2>&1
    python - "$v" "$T" gpurun_out/${TAG}_${v}_t$T.log <<'PY'
import json, sys
v, T, f = sys.argv[1:]
try:
    r = json.loads(open(f).read().strip().splitlines()[-1]); rf = r["roofline"]
    print(f"{v} T={T}: step {r['ms_per_step']*1e3:.1f} us ffn {rf['ffn_us_per_step']:.1f} us nograph {rf['ms_per_step_without_graph']*1e3:.1f} sm_mhz {r['clocks']['sm_mhz']}")
except Exception as e:
    print(v, T, "failed", e, open(f).read()[-400:])
PY
  done
done
