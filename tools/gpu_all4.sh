#!/bin/bash
# the whole -m gpu suite on a 4-GPU box (the 1-GPU tests and every multi-GPU test)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/all4; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?"; tail -2 $O/pytest.log
