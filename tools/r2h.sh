set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_abi.py tests/test_gpu_integration.py -x -q > $OUT/pytest_r2h_host.log 2>&1; echo "host tests rc=$?"; tail -2 $OUT/pytest_r2h_host.log
MOA_HOST_TRACE=1 timeout 300 python tools/e2e_host_probe.py c4 c5 c3 > $OUT/p3.jsonl 2> $OUT/p3.err; echo "probe rc=$?"; cat $OUT/p3.jsonl
timeout 300 python tools/e2e_trace.py c4 $OUT/trace_c4_pageable.json pageable > $OUT/trace_c4_pageable.txt 2>&1; echo rc=$?
