#!/bin/bash
# ncu evidence for every route: launch list of the default bench command and one
# --set full capture of each dominant kernel.  Usage (under gpurun): bash tools/profile_all.sh TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-inner --no-cpu"
$CMD > $OUT/plain_c2_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file $OUT/launches_c2_$TAG.csv $CMD > $OUT/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:outer_vec -s 2 -c 1 \
    -o $OUT/prof_c2_$TAG $CMD > $OUT/ncu_c2_$TAG.log 2>&1
echo "ncu c2 rc=$?"
for C in c4 c5 c3 c1; do
  CMDC="python bench.py --config $C --steps 1 --warmup 3 --no-cpu"
  $CMDC > $OUT/plain_${C}_$TAG.log 2>&1 || { echo "plain $C failed"; continue; }
  # c5 launches the VIMNMX3 and FMNMX3 specialisations per product (the second
  # exits at once): skip the first product's two to land on the working one
  case $C in c5) K=tropical; S=2;; *) K=dmma; S=1;; esac
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c 1 \
      -o $OUT/prof_${C}_$TAG $CMDC > $OUT/ncu_${C}_$TAG.log 2>&1
  echo "ncu $C rc=$?"
done
