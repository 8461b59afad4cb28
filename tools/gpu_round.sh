#!/bin/bash
# One GPU session: bench (plain), then ncu launch list + full captures of the
# top kernel of each route.  Usage (under gpurun): bash tools/gpu_round.sh TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
NCU=${NCU:-ncu}
python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?" >> $OUT/bench_$TAG.log
tail -1 $OUT/bench_$TAG.log
# launch list for the default workload (cold-cache, serialised; compare shares)
CMD="python bench.py --steps 3 --warmup 3 --no-inner --no-cpu"
$CMD > $OUT/plain_c2.log 2>&1 && \
  $NCU --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
       --log-file $OUT/launches_c2_$TAG.csv $CMD > $OUT/ncu_launches_c2.log 2>&1
echo "launches rc=$?"
# full capture: outer kernel
$NCU --set full --clock-control none --import-source on -k regex:outer_vec -s 2 -c 1 \
     -o $OUT/prof_outer_$TAG $CMD > $OUT/ncu_outer.log 2>&1
echo "ncu outer rc=$?"
for C in c4 c5 c3; do
  CMDC="python bench.py --config $C --steps 1 --warmup 3 --no-cpu"
  $CMDC > $OUT/plain_$C.log 2>&1 || { echo "plain $C failed"; continue; }
  case $C in c5) K=semiring;; *) K=dmma;; esac
  $NCU --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
       -o $OUT/prof_${C}_$TAG $CMDC > $OUT/ncu_$C.log 2>&1
  echo "ncu $C rc=$?"
done
