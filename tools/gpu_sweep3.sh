#!/bin/bash
# 4-GPU box after the three slots: push blocks and dispatch-grid sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/sweep3; mkdir -p $O
run() {
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 50 --warmup 5 --no-cpu > $O/b.json 2>$O/b.err
  tail -1 $O/b.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'value %.3fM'%(d['value']/1e6), 'ms %.1f'%(d['ms_per_step']*1e3))" || tail -3 $O/b.err
}
for pb in 296 444 592 888; do JANUS_PUSH_BLOCKS=$pb run "push $pb"; done
for dc in 24 49 74 148; do JANUS_DISPATCH_CTAS=$dc run "disp $dc"; done
run "default"
