set -u
OUT=gpurun_out
timeout 300 python tools/e2e_trace.py c4 $OUT/trace_c4_pageable.json pageable > $OUT/trace_c4_pageable.txt 2>&1; echo rc=$?
tail -3 $OUT/trace_c4_pageable.txt
