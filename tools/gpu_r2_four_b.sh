#!/bin/bash
# round 2, four GPUs: bench N=4 after the push-combine / two-stream changes + the new nvls tests
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2four_b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -q -k "switch or colocated or nvls-2-1-3" > $O/pytest_dist4.log 2>&1; echo "dist rc=$?"; tail -3 $O/pytest_dist4.log
P=29800
for box in split moe-only; do
  for tr in auto routed; do
    for cb in push switch; do
      [ "$tr" = routed ] && [ "$cb" = switch ] && continue
      P=$((P+1))
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 100 --warmup 10 --no-cpu --box $box --transport $tr --combine $cb > $O/bench_n4_${box}_${tr}_$cb.json 2> $O/bench_n4_${box}_${tr}_$cb.err; echo "bench $box $tr $cb rc=$?"
    done
  done
done
