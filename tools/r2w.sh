set -u
OUT=gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,temperature.gpu --format=csv,noheader -lms 100 > $OUT/smi_r2w.csv &
SMI=$!
timeout 600 python tools/repeat_probe.py c5 16 > $OUT/rep_c5.json 2>&1
timeout 600 python tools/repeat_probe.py c4 12 > $OUT/rep_c4.json 2>&1
kill $SMI
cat $OUT/rep_c5.json $OUT/rep_c4.json
nvidia-smi -q -d POWER | grep -i -E "limit|draw" | head -8
