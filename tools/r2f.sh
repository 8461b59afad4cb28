set -u
OUT=gpurun_out
./tools/host_probe > $OUT/host_probe_r2f.json 2>&1; echo "probe rc=$?"
lscpu | grep -E "NUMA|Socket|Model name|Thread|Core" > $OUT/lscpu.txt; cat $OUT/lscpu.txt
numactl -H 2>/dev/null | head -5
MOA_HOST_TRACE=1 timeout 300 python tools/e2e_host_probe.py c4 > $OUT/p2.jsonl 2> $OUT/p2.err
grep '"c4"' $OUT/p2.jsonl
