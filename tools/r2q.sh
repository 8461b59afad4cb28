set -u
OUT=gpurun_out
CMDC="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu"
$CMDC > $OUT/plain_c5_r2q.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tropical_tma -s 2 -c 1 -o $OUT/prof_c5_r2q $CMDC > $OUT/ncu_c5_r2q.log 2>&1
echo "ncu c5 rc=$?"
