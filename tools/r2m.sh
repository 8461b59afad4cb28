set -u
OUT=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2m.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_r2m.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo > $OUT/bench_n2_gloo.log 2> $OUT/bench_n2_gloo.err; echo "n2 rc=$?"; tail -c 400 $OUT/bench_n2_gloo.log
