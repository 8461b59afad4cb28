set -u
OUT=gpurun_out
MOA_BENCH_VERBOSE=1 MOA_HOST_TRACE=1 python bench.py --legs c4 --no-cpu --steps 3 > $OUT/bench_c4_trace2.log 2> $OUT/bench_c4_trace2.err; echo "rc=$?"
grep -E "e2e per-step|execute_host" $OUT/bench_c4_trace2.err | tail -20
MOA_HOST_TRACE=1 python tools/cold_call.py c4 2>&1 | grep -E "execute_host|first" | tail -12
