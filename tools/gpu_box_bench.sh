# usage: bash tools/gpu_box_bench.sh TAG N [TRANSPORTS] — bench --gpus N per transport
N=${2:-4}; TRS=${3:-"p2p nvls"}
for tr in $TRS; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 100 --warmup 5 --transport $tr > gpurun_out/${1}_bench${N}_$tr.log 2>&1
  tail -n 1 gpurun_out/${1}_bench${N}_$tr.log | python -c "
import json,sys
r=json.loads(sys.stdin.read()); n=r['nvlink']
print(r['config']['transport'], 'tok/s %.4g'%r['value'], 'step %.1f us'%(r['ms_per_step']*1e3), 'disp %.1f moe %.1f comb %.1f ffn %.1f'%(n['dispatch_us'], n['moe_step_us'], n['combine_us'], r['roofline']['ffn_us_per_step']), 'e2e %.4g'%r['e2e']['value'])" || tail -5 gpurun_out/${1}_bench${N}_$tr.log
done
