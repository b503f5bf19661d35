# final code: the other BASELINE shapes on one GPU and on boxes of 2 / 4 (c3 split 1A+3E,
# c4 = DeepSeek-V3 + shared expert on MoE-only boxes; c4 needs a broadcast transport)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2shapes
mkdir -p $O
one() { local name=$1; shift; timeout 900 python bench.py --no-cpu "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; tail -1 $O/$name.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('  value %.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'ffn_us %.1f'%r['ffn_us_per_step'], 'hbm %.3f tensor %.3f'%(r['hbm_frac'], r['tensor_frac']))"; }
box() { local name=$1 n=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 30 --warmup 3 --no-cpu "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; tail -1 $O/$name.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); n=d['nvlink']; print('  value %.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'disp %.1f moe %.1f comb %.1f ffn %.1f'%(n['dispatch_us'], n['moe_step_us'], n['combine_us'], d['roofline']['ffn_us_per_step']), d['config'].get('transport'))"; }
one c3_t4096 --shape c3 --steps 20 --warmup 3
one c4_t256 --shape c4 --tokens 256 --steps 10 --warmup 3
one c4_t4096 --shape c4 --steps 10 --warmup 3
box c3_split4 4 --shape c3 --box split
box c3_moeonly4 4 --shape c3
box c4_moeonly2 2 --shape c4 --box moe-only --transport ce
box c4_moeonly4 4 --shape c4 --box moe-only --transport ce
