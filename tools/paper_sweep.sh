#!/bin/bash
# The paper's experiment (§II.B) through the harness CLI on the GPU,
# with the reference harness's own defaults (rows = threads, ell = 128,
# n = 2..256) for the MoA inner/outer products and the GEMM comparator at 1, 2
# and 4 row partitions, plus a large inner sweep (rows 4096, ell 1024,
# n = 2..4096); then the paper's derived metrics (mean, total size, ratio to
# one partition).  Usage (under gpurun): bash tools/paper_sweep.sh OUTDIR
set -eu
OUT=${1:-gpurun_out/paper}
mkdir -p "$OUT"
run() {  # tag mode threads extra-args...
  local tag=$1 mode=$2 t=$3; shift 3
  python -m paper_0907_0792_b200 bench --mode $mode --threads $t --repeats 5 \
    --out "$OUT/raw_${tag}_${mode}_t$t.csv" "$@"
}
for mode in moa-inner moa-outer gemm-baseline; do
  for t in 1 2 4; do run paper $mode $t; done
  for t in 1 2 4; do
    python -m paper_0907_0792_b200 metrics --raw "$OUT/raw_paper_${mode}_t$t.csv" \
      --baseline-raw "$OUT/raw_paper_${mode}_t1.csv" --out "$OUT/metrics_paper_${mode}_t$t.csv"
  done
done
for mode in moa-inner gemm-baseline; do
  for t in 1 4; do run large $mode $t --rows 4096 --ell 1024 --n-min 1 --n-max 12; done
done
ls "$OUT"
