#!/bin/bash
# gate kernel: parity tests + graph-replay timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/gate; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gate.py tests/test_gpu_moe.py -q -k "gate or gated" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 300 python tools/gate_probe.py 128 256 1024 2048 4096 8192 > $O/probe.txt 2>&1; cat $O/probe.txt
