set -u
OUT=gpurun_out
python bench.py --config c1 --steps 20 --warmup 3 --no-cpu > $OUT/plain_c1.log 2>&1; echo plain rc=$?
ncu --set full --clock-control none --import-source on -k regex:dmma -s 3 -c 1 -o $OUT/prof_c1 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > $OUT/ncu_c1.log 2>&1; echo ncu rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-cpu > $OUT/gloo2.log 2>&1; echo gloo2 rc=$?
