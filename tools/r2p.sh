set -u
OUT=gpurun_out
timeout 600 python tools/acc_stress.py 60 > $OUT/acc_stress_r2p.log 2>&1; echo "acc rc=$?"; cat $OUT/acc_stress_r2p.log
timeout 900 python tools/determinism_stress.py 40 > $OUT/det_stress_r2p.log 2>&1; echo "det rc=$?"; tail -12 $OUT/det_stress_r2p.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2p.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_r2p.log
