set -u
OUT=gpurun_out
MOA_HOST_TRACE=1 timeout 300 python tools/repeat_probe.py c4 12 2> $OUT/rep_c4.err; grep -c . $OUT/rep_c4.err
grep end= $OUT/rep_c4.err | awk '{print $NF}' | tr '\n' ' '; echo
MOA_HOST_POOL_KEEP_BYTES=17179869184 timeout 300 python tools/repeat_probe.py c4 12
timeout 300 python tools/repeat_probe.py c5 8
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv
