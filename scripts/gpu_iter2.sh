# Fast iteration: build, a parity subset, 200M phase timings (median of reps).
make -j8 > gpurun_out/make.log 2>&1 || { echo "make failed"; tail -20 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and not slow" ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -6
if [ $rc -ne 0 ] && [ -z "$FORCE" ]; then exit 1; fi
for d in ${DISTS:-normal twodups telemetry zipf uniform_u64}; do timeout 300 python scripts/prof_sort.py --dist $d --n ${N:-200000000} --reps 4 2>&1 | tail -1; done
