#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2san
mkdir -p $O profiles/r2
timeout 600 python tools/calibrate_latency.py --out profiles/r2/latency_calibration.json > $O/calib.log 2>&1; echo "calib rc=$?"
mkdir -p gpurun_out/profiles/r2 && cp profiles/r2/latency_calibration.json gpurun_out/profiles/r2/
timeout 600 python -m pytest tests/test_latency_model.py -q > $O/latency_test.log 2>&1; echo "latency test rc=$?"; tail -2 $O/latency_test.log
timeout 600 python tools/sanitize_probe.py > $O/probe_plain.log 2>&1 && \
timeout 1800 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_probe.py > $O/memcheck.log 2>&1
echo "memcheck rc=$?"; tail -5 $O/memcheck.log
