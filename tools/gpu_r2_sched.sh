#!/bin/bash
# scheduler: parity (schedule + fuzz) and the graph-replayed sweep, small-CTA vs cluster kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_fuzz.py -k "sched or schedule" -x -q > gpurun_out/pytest_sched.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sched.log
timeout 600 python tools/sched_sweep.py --configs c1_uniform,c2,c3,c5 --tokens 32,64,128,256,512,1024 --cpu > gpurun_out/sched_small.jsonl 2> gpurun_out/sched_small.err
echo "sweep rc=$?"
JANUS_SCHED_CLUSTER=1 timeout 600 python tools/sched_sweep.py --configs c5 --tokens 32,64,128,256 > gpurun_out/sched_cluster.jsonl 2>&1
echo "sweep2 rc=$?"
