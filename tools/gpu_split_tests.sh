#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/splitt; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -k "split_streams or oversubscribed or colocated" > $O/pytest.log 2>&1; echo "rc=$?"; tail -2 $O/pytest.log
