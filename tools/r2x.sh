set -u
OUT=gpurun_out
python tools/c5_repeat_device.py
timeout 600 python tools/repeat_probe.py c5 16
timeout 600 python tools/repeat_probe.py c4 6
