set -u
OUT=gpurun_out
./tools/peaks_minplus > $OUT/minplus_r2n.json 2>&1; echo "mb rc=$?"; cat $OUT/minplus_r2n.json
ncu --set full --clock-control none --import-source on -k regex:"mix<9" -c 1 -o $OUT/prof_mix9_r2n ./tools/peaks_minplus > $OUT/ncu_mix9.log 2>&1; echo "ncu mix9 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"tile<8, 8" -c 1 -o $OUT/prof_tile88_r2n ./tools/peaks_minplus > $OUT/ncu_tile88.log 2>&1; echo "ncu tile rc=$?"
CMDC="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu"
$CMDC > $OUT/plain_c5_r2n.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tropical_tma -s 2 -c 1 -o $OUT/prof_c5_r2n $CMDC > $OUT/ncu_c5_r2n.log 2>&1
echo "ncu c5 rc=$?"
