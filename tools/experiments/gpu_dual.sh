#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export JANUS_GEMM_DUAL=1
for thr in 1 64 96 100000; do
  JANUS_DUAL_THR=$thr timeout 240 python bench.py --steps 30 --warmup 5 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('thr $thr', 'value %.3fM'%(d['value']/1e6), 'ffn_us %.1f'%r['ffn_us_per_step'], 'hbm %.3f tensor %.3f'%(r['hbm_frac'], r['tensor_frac']), d['clocks']['sm_mhz'])"
done
