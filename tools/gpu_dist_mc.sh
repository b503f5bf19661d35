# N-GPU box: dist tests (both transports) + bench per transport
N=${2:-2}
timeout -s KILL 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/${1}_dist_pytest.log 2>&1; echo rc=$? >> gpurun_out/${1}_dist_pytest.log
tail -n 3 gpurun_out/${1}_dist_pytest.log
for tr in p2p nvls; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 100 --warmup 5 --transport $tr > gpurun_out/${1}_bench${N}_$tr.log 2>&1
  tail -n 1 gpurun_out/${1}_bench${N}_$tr.log | cut -c1-400
done
