set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_abi.py tests/test_gpu_integration.py -x -q > $OUT/pytest_r2d_host.log 2>&1; echo "host tests rc=$?"; tail -5 $OUT/pytest_r2d_host.log
MOA_HOST_TRACE=1 timeout 600 python tools/e2e_host_probe.py c4 > $OUT/e2e_host_probe_r2d.jsonl 2> $OUT/e2e_host_probe_r2d.err; echo "probe rc=$?"
cat $OUT/e2e_host_probe_r2d.jsonl
timeout 300 python tools/cold_call.py c4 > $OUT/cold_call_r2d.json 2> $OUT/cold_call_r2d.err; echo "cold rc=$?"; cat $OUT/cold_call_r2d.json
