# 4-GPU box: correctness (1A+3E, 2A+2E) + bench --gpus 4 and 2
timeout -s KILL 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/${1}_dist_pytest.log 2>&1; echo rc=$? >> gpurun_out/${1}_dist_pytest.log
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 100 --warmup 5 > gpurun_out/${1}_bench4.log 2>&1
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/${1}_bench2.log 2>&1
tail -n 3 gpurun_out/${1}_dist_pytest.log
