#!/bin/bash
# bench defaults at N = 2 and 4 (run with --gpus 4), plus the split box at 4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2scale
mkdir -p $O
P=29900
for n in 2 4; do
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 100 --warmup 10 > $O/bench_n${n}.json 2> $O/bench_n${n}.err; echo "bench n$n rc=$?"
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 100 --warmup 10 --box split --no-cpu > $O/bench_n${n}_split.json 2> $O/bench_n${n}_split.err; echo "bench n$n split rc=$?"
done
