#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv -lms 100 > gpurun_out/sched_clocks.csv 2>&1 &
SMI=$!
timeout 600 python tools/sched_sweep.py --configs c2,c5 --tokens 32,256,1024 --cpu > gpurun_out/sched_small.jsonl 2> gpurun_out/sched_small.err
kill $SMI
tools/micro/greedy_bench > gpurun_out/greedy_bench.txt 2>&1
