# usage: bash tools/gpu_box_gate.sh TAG N — box bench (NVLS) with attention-side routing vs MoE-side gating
N=${2:-4}
for g in "" "--gate"; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --steps 100 --warmup 5 --transport nvls $g > gpurun_out/${1}_box${N}${g}.log 2>&1
  tail -n 1 gpurun_out/${1}_box${N}${g}.log | python -c "
import json,sys
r=json.loads(sys.stdin.read()); n=r['nvlink']
print('gate' if '$g' else 'routed', 'tok/s %.4g'%r['value'], 'step %.1f us'%(r['ms_per_step']*1e3), 'disp %.1f moe %.1f comb %.1f ffn %.1f'%(n['dispatch_us'], n['moe_step_us'], n['combine_us'], r['roofline']['ffn_us_per_step']), 'e2e %.4g'%r['e2e']['value'], 'launches', r['gpu_launches'])" || tail -5 gpurun_out/${1}_box${N}${g}.log
done
