# usage: bash tools/gpu_box_shapes.sh TAG — c3 on the 1A+3E split box, c4 (DS-V3 + shared) on MoE-only boxes of 2 and 4
run() {  # name nproc args...
  local name=$1 n=$2; shift 2
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n --steps 30 --warmup 3 --transport nvls "$@" > gpurun_out/${TAG}_$name.log 2>&1
  tail -n 1 gpurun_out/${TAG}_$name.log | python -c "
import json,sys
r=json.loads(sys.stdin.read()); n=r['nvlink']
print('$name', 'tok/s %.4g'%r['value'], 'step %.1f us'%(r['ms_per_step']*1e3), 'disp %.1f moe %.1f comb %.1f ffn %.1f'%(n['dispatch_us'], n['moe_step_us'], n['combine_us'], r['roofline']['ffn_us_per_step']), 'e2e %.4g'%r['e2e']['value'], r['clocks'])" || tail -5 gpurun_out/${TAG}_$name.log
}
TAG=$1
run c3_split4 4 --shape c3
run c4_moeonly2 2 --shape c4 --box moe-only
run c4_moeonly4 4 --shape c4 --box moe-only
