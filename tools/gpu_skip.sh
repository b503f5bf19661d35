# (a measurement with an experiment build, exp_libs/skip.so, whose push kernel returned at once when JANUS_SKIP_PUSH=1; that build and knob are not in the tree)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp exp_libs/skip.so paper_2512_13525_b200/libjanus_b200.so
for sp in "" 1; do
  JANUS_SKIP_PUSH=$sp timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2965${#sp} bench.py --gpus 4 --steps 50 --warmup 5 --no-cpu > /tmp/b.json 2>/tmp/b.err
  tail -1 /tmp/b.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); n=d['nvlink']; print('skip=$sp', 'value %.3fM'%(d['value']/1e6), 'ms %.1f'%(d['ms_per_step']*1e3), 'disp %.1f moe %.1f comb %.1f'%(n['dispatch_us'],n['moe_step_us'],n['combine_us']), 'ffn %.1f'%d['roofline']['ffn_us_per_step'])"
done
