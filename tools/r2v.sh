set -u
OUT=gpurun_out
MOA_BENCH_VERBOSE=1 MOA_HOST_TRACE=1 python bench.py --legs c5 --no-cpu --steps 3 > $OUT/bench_c5_trace.log 2> $OUT/bench_c5_trace.err; echo "rc=$?"
grep -E "e2e per-step|moa_host\] setup=0.00[0-9] blk|cleanup" $OUT/bench_c5_trace.err | tail -40 | cut -c1-220
python -c "
import json; d=json.loads(open('$OUT/bench_c5_trace.log').read().strip().splitlines()[-1]); v=d['inner']['c5']; print(v['e2e'], v['e2e_api'])"
