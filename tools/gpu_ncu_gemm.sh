# ncu --set full on the gate/up GEMM only: bash tools/gpu_ncu_gemm.sh TAG TOKENS
TAG=$1; T=$2
CMD="python bench.py --tokens $T --steps 10 --warmup 3 --no-cpu"
timeout -s KILL 300 $CMD > gpurun_out/${TAG}_plain_t$T.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm" -s 6 -c 2 -o gpurun_out/${TAG}_gemm_t$T $CMD > gpurun_out/${TAG}_gemm_t$T.log 2>&1
echo "rc=$?"
