timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest.log
timeout -s KILL 300 python tools/sched_sweep.py --cpu > gpurun_out/r2_sweep.log 2>&1
timeout -s KILL 300 python bench.py --tokens 256 --steps 500 > gpurun_out/r2_bench256.log 2>&1
timeout -s KILL 300 python bench.py --tokens 4096 --steps 200 --no-cpu > gpurun_out/r2_bench4096.log 2>&1
tail -n 3 gpurun_out/r2_pytest.log
