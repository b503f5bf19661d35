# copy-engine vs routed vs p2p dispatch on an N-GPU MoE-only box (N = $NG, default 2)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
NG=${NG:-2}
mkdir -p gpurun_out/ce
timeout 900 python -m pytest -x -q tests/test_gpu_dist.py -k "ce" 2>&1 | tail -3
for tr in ${TRS:-routed ce}; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG --steps 50 --warmup 5 --transport $tr > gpurun_out/ce/bench_n${NG}_$tr.json 2> gpurun_out/ce/bench_n${NG}_$tr.err
  tail -1 gpurun_out/ce/bench_n${NG}_$tr.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); n=d['nvlink']; print('$tr', 'value %.3fM'%(d['value']/1e6), 'ms %.1f'%(d['ms_per_step']*1e3), 'disp %.1f moe %.1f comb %.1f'%(n['dispatch_us'],n['moe_step_us'],n['combine_us']), 'ffn %.1f'%d['roofline']['ffn_us_per_step'])"
done
