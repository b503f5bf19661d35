#!/bin/bash
# three epoch slots + split streams: every multi-GPU test, then the box benches
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/slots3; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_dist.py tests/test_gpu_box_local.py -q > $O/pytest_all.log 2>&1; echo "all rc=$?"; tail -2 $O/pytest_all.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900+n)) bench.py --gpus $n --steps 50 --warmup 5 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo "bench n=$n rc=$?"
  tail -1 $O/bench_n$n.json | cut -c1-200
done
