cd "${GRAFT_REPO_ROOT:-/root/repo}"
NG=${NG:-4}
for pb in ${PBS:-148 296 592 0}; do
  JANUS_PUSH_BLOCKS=$pb timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29700 + pb % 97)) bench.py --gpus $NG --steps 50 --warmup 5 --no-cpu > /tmp/b.json 2>/tmp/b.err
  tail -1 /tmp/b.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); n=d['nvlink']; print('pb $pb', 'value %.3fM'%(d['value']/1e6), 'ms %.1f'%(d['ms_per_step']*1e3), 'disp %.1f moe %.1f comb %.1f'%(n['dispatch_us'],n['moe_step_us'],n['combine_us']), 'ffn %.1f'%d['roofline']['ffn_us_per_step'])" || tail -3 /tmp/b.err
done
