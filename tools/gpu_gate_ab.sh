#!/bin/bash
# gate kernel A/B (JANUS_LIB=old/new .so), interleaved, graph replay; parity of the new one
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/gate_ab; mkdir -p $O; rm -f $O/probe.txt
timeout 900 python -m pytest tests/test_gpu_gate.py tests/test_gpu_moe.py -q -k "gate or gated" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for r in 1 2; do for v in old new; do
  echo "== $v" >> $O/probe.txt
  JANUS_LIB=$PWD/abtmp/$v.so timeout 300 python tools/gate_probe.py 256 1024 2048 4096 8192 >> $O/probe.txt 2>&1
done; done
cat $O/probe.txt
