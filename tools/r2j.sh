set -u
OUT=gpurun_out
./tools/host_probe > $OUT/host_probe_r2j.json 2>&1; echo "probe rc=$?"
timeout 600 python -m pytest tests/test_gpu_host_abi.py tests/test_gpu_integration.py -x -q > $OUT/pytest_r2j_host.log 2>&1; echo "host tests rc=$?"; tail -1 $OUT/pytest_r2j_host.log
MOA_HOST_TRACE=1 timeout 300 python tools/e2e_host_probe.py c4 c5 c3 > $OUT/p4.jsonl 2> $OUT/p4.err; echo "e2e probe rc=$?"; cat $OUT/p4.jsonl
