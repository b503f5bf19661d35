#!/bin/bash
# 4-GPU box: the attention-side reduce grid now that the combine runs off the MoE stream
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/sweepr; mkdir -p $O
run() {
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-4} --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus ${NG:-4} --steps 50 --warmup 5 --no-cpu > $O/b.json 2>$O/b.err
  tail -1 $O/b.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'value %.3fM'%(d['value']/1e6), 'ms %.1f'%(d['ms_per_step']*1e3))" || tail -3 $O/b.err
}
for rc in 74 148 296 592; do JANUS_REDUCE_CTAS=$rc run "reduce $rc"; done
run "default"
for rc in 148 296; do JANUS_REDUCE_CTAS=$rc run "reduce $rc"; done
run "default"
