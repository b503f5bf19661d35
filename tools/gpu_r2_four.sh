#!/bin/bash
# round 2, four GPUs: every box test, bench N=4 over the transports and box kinds, NCCL baselines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2four
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -q > $O/pytest_dist4.log 2>&1; echo "dist rc=$?"; tail -3 $O/pytest_dist4.log
P=29700
for box in split moe-only; do
  for tr in auto p2p routed; do
    P=$((P+1))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 100 --warmup 10 --no-cpu --box $box --transport $tr > $O/bench_n4_${box}_$tr.json 2> $O/bench_n4_${box}_$tr.err; echo "bench $box $tr rc=$?"
  done
  P=$((P+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/nccl_baseline.py --box $box > $O/nccl_n4_$box.json 2> $O/nccl_n4_$box.err; echo "nccl $box rc=$?"
done
