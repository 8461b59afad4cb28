set -u
OUT=gpurun_out
for cfg in "16 4 16" "8 6 16" "32 4 16" "16 8 16" "16 4 8" "4 16 16"; do
  set -- $cfg
  echo "== slot=$1MiB slots=$2 threads=$3"
  MOA_HOST_SLOT_MB=$1 MOA_HOST_SLOTS=$2 MOA_HOST_COPY_THREADS=$3 MOA_HOST_TRACE=1 timeout 300 python tools/e2e_host_probe.py c4 > $OUT/p.jsonl 2> $OUT/p.err
  grep '"c4"' $OUT/p.jsonl | grep page
  grep moa_stage $OUT/p.err | grep h2d | sort | uniq -c | sort -rn | head -3
  grep moa_stage $OUT/p.err | grep "h2d 2048.0\|h2d 384\|d2h" | tail -4
done
