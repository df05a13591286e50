# Big-path iteration: build, big-path parity subset, 200M timings of the duplicate configs.
make -j8 > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "dense or large_big or many_big or telemetry or twodups or big_threshold or edge" > gpurun_out/pytest_big.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_big.log
LS_DEBUG_STAGE=512 LS_GRAPH=0 python scripts/prof_sort.py --dist telemetry --n 200000000 --reps 2 2>&1 | grep prof | tail -1
for d in ${DISTS:-telemetry twodups zipf uniform_u64}; do timeout 300 python scripts/prof_sort.py --dist $d --n 200000000 --reps 3 2>&1 | tail -1; done
