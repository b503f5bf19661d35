nvidia-smi -L > gpurun_out/r1_smi.log 2>&1
timeout -s KILL 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout -s KILL 600 python -m pytest tests/test_gpu_schedule.py -x -q > gpurun_out/r1_sched.log 2>&1; echo "rc=$?" >> gpurun_out/r1_sched.log
timeout -s KILL 600 python -m pytest tests/test_gpu_moe.py -x -q > gpurun_out/r1_moe.log 2>&1; echo "rc=$?" >> gpurun_out/r1_moe.log
timeout -s KILL 300 python bench.py --tokens 256 --steps 200 --no-cpu > gpurun_out/r1_bench256.log 2>&1; echo "rc=$?" >> gpurun_out/r1_bench256.log
timeout -s KILL 300 python bench.py --tokens 4096 --steps 100 --no-cpu > gpurun_out/r1_bench4096.log 2>&1; echo "rc=$?" >> gpurun_out/r1_bench4096.log
tail -n 4 gpurun_out/r1_*.log
