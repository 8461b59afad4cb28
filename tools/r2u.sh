set -u
OUT=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2u.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_r2u.log
python bench.py > $OUT/bench_r2u.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref_r2u.log 2>&1; echo "ref rc=$?"; tail -1 $OUT/bench_ref_r2u.log | cut -c1-300
timeout 300 python tools/cold_call.py c4 > $OUT/cold_call_r2u.json 2>&1; cat $OUT/cold_call_r2u.json
