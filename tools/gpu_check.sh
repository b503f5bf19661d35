# usage: bash tools/gpu_check.sh TAG   — gpu tests + scheduler sweep + bench at T=256/4096
TAG=${1:-chk}
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout -s KILL 300 python tools/sched_sweep.py --tokens 32,256,1024,4096 > gpurun_out/${TAG}_sweep.log 2>&1
timeout -s KILL 300 python bench.py --tokens 256 --steps 500 --no-cpu > gpurun_out/${TAG}_bench256.log 2>&1
timeout -s KILL 300 python bench.py --tokens 4096 --steps 200 --no-cpu > gpurun_out/${TAG}_bench4096.log 2>&1
tail -n 2 gpurun_out/${TAG}_pytest.log
