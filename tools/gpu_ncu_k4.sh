cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp exp_libs/base.so paper_2512_13525_b200/libjanus_b200.so
mkdir -p gpurun_out
timeout 300 python tools/ffn_probe.py || exit 1
timeout 900 ncu -k regex:grouped_gemm --launch-skip 6 --launch-count 2 --set full --clock-control none --import-source on -o gpurun_out/k4_full -f python tools/ffn_probe.py > gpurun_out/k4_full.log 2>&1
tail -3 gpurun_out/k4_full.log
