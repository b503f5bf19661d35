# usage: bash tools/gpu_profile.sh TAG TOKENS  — plain run, ncu launch list, ncu --set full
TAG=${1:-r1}; T=${2:-4096}
CMD="python bench.py --tokens $T --steps 20 --warmup 3 --no-cpu"
timeout -s KILL 300 $CMD > gpurun_out/${TAG}_plain_t$T.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"aebs|grouped|permute|combine" -c 400 --csv --log-file gpurun_out/${TAG}_launches_t$T.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"aebs|grouped|permute|combine" -s 15 -c 5 -o gpurun_out/${TAG}_full_t$T $CMD > gpurun_out/${TAG}_full_t$T.log 2>&1
echo "full rc=$?"
