CMDC="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu"
$CMDC > gpurun_out/plain_c5_r01z2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tropical -s 2 -c 1 -o gpurun_out/prof_c5_r01z $CMDC > gpurun_out/ncu_c5_r01z.log 2>&1
echo "ncu c5 rc=$?"
tail -3 gpurun_out/ncu_c5_r01z.log
