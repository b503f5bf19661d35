#!/bin/bash
# one ncu --set full capture of gate_kernel at T = 4096 (after the same command ran clean)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/gate
timeout 300 python tools/gate_probe.py 4096 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gate_kernel" -s 3 -c 1 -o gpurun_out/gate/full_t4096 -f python tools/gate_probe.py 4096 > gpurun_out/gate/ncu.log 2>&1; echo ncu $?
