# quick correctness gate: smoke with a short timeout, then the GPU suites
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${1}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${1}_smoke.log
if grep -q "rc=0" gpurun_out/${1}_smoke.log; then bash tools/gpu_check.sh $1; fi
