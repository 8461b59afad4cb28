set -u
OUT=gpurun_out
MOA_HOST_TRACE=1 timeout 600 python tools/e2e_host_probe.py c4 > $OUT/e2e_host_probe_r2c.jsonl 2> $OUT/e2e_host_probe_r2c.err; echo "probe rc=$?"
cat $OUT/e2e_host_probe_r2c.jsonl
