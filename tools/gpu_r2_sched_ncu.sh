#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_fuzz.py -k "sched or schedule" -x -q 2>&1 | tail -2
JANUS_TRACE_DEBUG=1 python tools/sched_sweep.py --configs c2,c5 --tokens 32,256 2>&1 | tail -8
python tools/sched_probe.py c5 256 > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --sampling-interval 0 --clock-control none --import-source on -k regex:aebs_small -s 3 -c 1 \
    -o gpurun_out/sched_small_c5_t256 -f python tools/sched_probe.py c5 256 > gpurun_out/ncu_sched.log 2>&1
echo "ncu rc=$?"
