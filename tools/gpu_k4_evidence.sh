# K4 evidence for profiles/r2/k4: tile timeline of the shipped kernel, CTA 0's
# stage log summary, the TMA microbenchmark.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/k4
JANUS_GEMM_TRACE=1 timeout 300 python tools/gemm_timeline.py --out gpurun_out/k4/timeline.npz > gpurun_out/k4/timeline.json 2> gpurun_out/k4/timeline.err
python tools/stage_log.py gpurun_out/k4/timeline.npz > gpurun_out/k4/stage_log.txt
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2512_13525_b200/csrc \
   tma_issue.cu -o tma_issue -lcuda && timeout 120 ./tma_issue && timeout 200 ./tma_issue --stream) > gpurun_out/k4/tma_issue.jsonl 2>&1
tail -c 600 gpurun_out/k4/timeline.json; wc -l gpurun_out/k4/tma_issue.jsonl
