cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/small
timeout 300 python tools/ffn_probe.py 4096 || exit 1
timeout 600 ncu --set full --clock-control none -k regex:"permute_kernel|combine_kernel|aebs" -s 3 -c 3 -o gpurun_out/small/t4096 -f python tools/ffn_probe.py 4096 > gpurun_out/small/ncu4096.log 2>&1; echo ncu $?
