set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_abi.py tests/test_gpu_integration.py -x -q > $OUT/pytest_r2b_host.log 2>&1; echo "host tests rc=$?"; tail -5 $OUT/pytest_r2b_host.log
timeout 300 python tools/cold_call.py c4 > $OUT/cold_call_r2b.json 2> $OUT/cold_call_r2b.err; echo "cold rc=$?"; cat $OUT/cold_call_r2b.json; tail -3 $OUT/cold_call_r2b.err
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2b.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_r2b.log
python bench.py --no-cpu > $OUT/bench_r2b.log 2>&1; echo "bench rc=$?"; tail -c 300 $OUT/bench_r2b.log
