set -u
OUT=gpurun_out
timeout 300 python tools/e2e_host_probe.py c3 > $OUT/p5.jsonl 2> $OUT/p5.err; echo "e2e probe rc=$?"; cat $OUT/p5.jsonl
timeout 300 python tools/cold_call.py c4 > $OUT/cold_call_r2k.json 2> $OUT/cold_call_r2k.err; echo "cold rc=$?"; cat $OUT/cold_call_r2k.json
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2k.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_r2k.log
python bench.py > $OUT/bench_r2k.log 2>&1; echo "bench rc=$?"
