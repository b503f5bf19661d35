# round 2 end-of-round evidence on a 4-GPU box: every multi-GPU test, the
# default bench at N = 2 and 4 (MoE-only box, routed transport)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2final4
mkdir -p $O
if [ -z "$SKIP_TESTS" ]; then timeout 2400 python -m pytest tests/test_gpu_dist.py tests/test_gpu_box_local.py -q > $O/pytest_dist4.log 2>&1; echo "dist rc=$?"; tail -2 $O/pytest_dist4.log; fi
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900+n)) bench.py --gpus $n --steps 50 --warmup 5 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo "bench n=$n rc=$?"
  tail -1 $O/bench_n$n.json | cut -c1-200
done
