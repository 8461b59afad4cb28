set -u
OUT=gpurun_out
MOA_BENCH_VERBOSE=1 MOA_HOST_TRACE=1 python bench.py --legs c4 --no-cpu --steps 3 > $OUT/bench_c4_trace.log 2> $OUT/bench_c4_trace.err; echo "rc=$?"
grep -E "e2e per-step|end=" $OUT/bench_c4_trace.err | tail -30
