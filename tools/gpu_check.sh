#!/bin/bash
# tests + bench + optional ncu of one kernel.  Usage: bash tools/gpu_check.sh TAG [ncu-config] [kernel-regex]
set -u
TAG=${1:-x}; NC=${2:-}; KR=${3:-}
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_$TAG.log
python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 $OUT/bench_$TAG.log
if [ -n "$NC" ]; then
  CMD="python bench.py --config $NC --steps 1 --warmup 3 --no-cpu"
  $CMD > $OUT/plain_${NC}_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$KR -s 1 -c 1 -o $OUT/prof_${NC}_$TAG $CMD > $OUT/ncu_${NC}_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
