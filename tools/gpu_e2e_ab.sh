#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/e2eab; mkdir -p $O
timeout 300 python tools/e2e_ab.py > $O/ab.json 2> $O/ab.err; tail -2 $O/ab.err; cat $O/ab.json
