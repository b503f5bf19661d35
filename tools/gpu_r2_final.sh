#!/bin/bash
# round 2 end-of-round evidence on one B200: the -m gpu suite, smoke, bench (both arms),
# the ncu launch list of the bench (one ncu per call; the --set full captures are tools/gpu_ncu_*.sh)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 500 --warmup 10 --no-cpu > $O/bench_500.json 2> $O/bench_500.err; echo "bench500 rc=$?"
timeout 900 python bench.py --tokens 256 --steps 200 --warmup 10 --no-cpu > $O/bench_t256.json 2> $O/bench_t256.err; echo "bench256 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"aebs|permute_kernel|grouped_gemm|combine_kernel" -c 40 --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1
echo "ncu rc=$?"

