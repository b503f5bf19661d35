# K4 tile timeline + a short bench per library build (LIBS: alternative builds to compare)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for lib in ${LIBS:-paper_2512_13525_b200/libjanus_b200.so}; do
  cp "$lib" /tmp/cur.so && cp /tmp/cur.so paper_2512_13525_b200/libjanus_b200.so
  echo "== $lib"
  if [ -n "$PARITY" ]; then timeout 600 python -m pytest -x -q tests/test_gpu_moe.py tests/test_gpu_fuzz.py 2>&1 | tail -2; fi
  JANUS_GEMM_TRACE=1 timeout 300 python tools/gemm_timeline.py --out gpurun_out/tl_$(basename $lib .so).npz 2>&1 | tail -3 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('gemm span %.1f gap %.2f'%(d['step_gemm_span_us'], d['gap_us']))
        for g in d['gemms']: print(' ', g['gemm'], 'span %.1f'%g['span_us'], {k:round(v,1) for k,v in g['issuer_pair_us'].items()}, {k:round(v,1) for k,v in g['producer_pair_us'].items()}, 'tail %.1f'%g['tail_idle_us_mean'])
    else: print(l.rstrip())"
  for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('  value %.3fM ffn_us %.1f hbm %.3f'%(d['value']/1e6, r['ffn_us_per_step'], r['hbm_frac']), d['clocks']['sm_mhz'])"; done
done
