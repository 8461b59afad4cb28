set -u
OUT=gpurun_out
./tools/host_probe > $OUT/host_probe.json 2> $OUT/host_probe.err; echo "probe rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2a.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_r2a.log
python bench.py > $OUT/bench_r2a.log 2>&1; echo "bench rc=$?"; tail -c 600 $OUT/bench_r2a.log
