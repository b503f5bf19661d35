#!/bin/bash
# box pipeline trace (JANUS_BOX_TRACE): per-call events of the pipelined loop at N = 4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/boxtrace; mkdir -p $O; rm -f gpurun_out/boxtrace_rank*.json
N=${N:-4}
JANUS_BOX_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29931 bench.py --gpus $N --steps 50 --warmup 5 > $O/bench_n$N.json 2> $O/bench_n$N.err; echo "bench rc=$?"
mv gpurun_out/boxtrace_rank*.json $O/ 2>/dev/null
tail -1 $O/bench_n$N.json | cut -c1-200
