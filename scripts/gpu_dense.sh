make -j8 > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "dense or large_big or many_big or telemetry or twodups or big_threshold" > gpurun_out/pytest_dense.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_dense.log
for d in telemetry twodups zipf uniform_u64; do timeout 300 python scripts/prof_sort.py --dist $d --n 200000000 --reps 3 2>&1 | tail -1; done
