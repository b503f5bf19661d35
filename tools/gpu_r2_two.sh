#!/bin/bash
# round 2, two GPUs: box tests (1A+1E, MoE-only 2), the NVLink probe (+ ncu NVLink sections), bench N=2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2two
O=gpurun_out/r2two
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -q -k "1-1 or 2-nvls" > $O/pytest_dist2.log 2>&1; echo "dist rc=$?"; tail -3 $O/pytest_dist2.log
for tr in p2p routed; do
  timeout 300 python tools/nvlink_probe.py --transport $tr > $O/nvlink_probe_$tr.json 2> $O/nvlink_probe_$tr.err; echo "probe $tr rc=$?"
done
for tr in auto p2p routed; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu --transport $tr > $O/bench_n2_$tr.json 2> $O/bench_n2_$tr.err; echo "bench $tr rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 tools/nccl_baseline.py > $O/nccl_n2.json 2> $O/nccl_n2.err; echo "nccl rc=$?"
ncu --list-sections > $O/ncu_sections.txt 2>&1
ncu --query-metrics > $O/ncu_metrics.txt 2>&1
grep -i nvl $O/ncu_metrics.txt | head -50 > $O/ncu_nvl_metrics.txt
python tools/nvlink_probe.py --transport p2p --steps 3 --no-peak > $O/probe_plain.log 2>&1 && \
ncu --section Nvlink --section Nvlink_Tables --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"dispatch|combine|reduce" -c 12 -o $O/nvlink_p2p -f python tools/nvlink_probe.py --transport p2p --steps 3 --no-peak > $O/ncu_nvlink.log 2>&1
echo "ncu rc=$?"
