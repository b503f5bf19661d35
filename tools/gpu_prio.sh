#!/bin/bash
# box: MoE stream priority (highest vs default), N = 4 and 2, interleaved
# (JANUS_MOE_PRIO was a temporary bench.py knob: s_moe = torch.cuda.Stream(dev, priority=-1); removed after this measurement)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/prio; mkdir -p $O
run() {
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $2 --steps 50 --warmup 5 --no-cpu > $O/b.json 2>$O/b.err
  tail -1 $O/b.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 n=$2', 'value %.3fM'%(d['value']/1e6), 'ms %.1f'%(d['ms_per_step']*1e3))" || tail -3 $O/b.err
}
for r in 1 2; do for p in 0 1; do JANUS_MOE_PRIO=$p run "prio $p" 4; done; done
for p in 0 1; do JANUS_MOE_PRIO=$p run "prio $p" 2; done
