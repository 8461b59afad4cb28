#!/bin/bash
# ncu --set full of single routes from tools/route_sweep.py (under gpurun):
#   bash tools/profile_routes.sh TAG float64:add:min [float64:divide:add ...]
set -u
TAG=$1; shift
OUT=gpurun_out
for R in "$@"; do
  N=${R//:/_}
  CMD="python tools/route_sweep.py --n 2048 --only $R --out $OUT/route_$N.jsonl"
  $CMD > $OUT/plain_$N.log 2>&1 || { echo "plain $R failed"; continue; }
  ncu --set full --clock-control none --import-source on -k regex:semiring_kernel -s 1 -c 1 \
      -o $OUT/prof_${N}_$TAG $CMD > $OUT/ncu_${N}_$TAG.log 2>&1
  echo "ncu $R rc=$?"
done
