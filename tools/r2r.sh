set -u
OUT=gpurun_out
python bench.py > $OUT/bench_r2r.log 2>&1; echo "bench rc=$?"
bash tools/profile_all.sh r02
CMDF="python bench.py --steps 3 --warmup 3 --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $OUT/launches_full_r02.csv $CMDF > $OUT/ncu_launches_full_r02.log 2>&1; echo "full launch list rc=$?"
python tools/ncu_summary.py r02 c2=$OUT/prof_c2_r02.ncu-rep c4=$OUT/prof_c4_r02.ncu-rep c5=$OUT/prof_c5_r02.ncu-rep c3=$OUT/prof_c3_r02.ncu-rep c1=$OUT/prof_c1_r02.ncu-rep > $OUT/summary_r02.log 2>&1; echo "summary rc=$?"
cp profiles/r02_ncu_summary.md profiles/ncu_traffic.json $OUT/ 2>/dev/null
