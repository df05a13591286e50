# Randomised stress of the current build (against numpy under the same order).
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
timeout 400 python scripts/stress.py --seconds ${S1:-240} --seed ${SEED:-7} --max-n 30000000 > gpurun_out/stress.log 2>&1; echo "stress rc=$?"; tail -2 gpurun_out/stress.log
timeout 420 python scripts/stress_big.py > gpurun_out/stress_big.log 2>&1; echo "stress_big rc=$?"; tail -2 gpurun_out/stress_big.log
