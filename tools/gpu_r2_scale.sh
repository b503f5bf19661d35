#!/bin/bash
# bench defaults at N = 2 and 4 (run with --gpus 4), plus the split box at 4; routed/colocated box tests
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2scale
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -q -k "routed or colocated" > $O/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -2 $O/pytest_dist.log
P=29900
for n in 2 4; do
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 100 --warmup 10 > $O/bench_n${n}.json 2> $O/bench_n${n}.err; echo "bench n$n rc=$?"
done
P=$((P+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 100 --warmup 10 --box split --no-cpu > $O/bench_n4_split.json 2> $O/bench_n4_split.err; echo "bench n4 split rc=$?"
