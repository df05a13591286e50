timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for s in ${STAGES:-0 1 3 4 5 6}; do echo "stage $s"; LS_DEBUG_STAGE=$s timeout 300 python scripts/prof_sort.py --dist ${DIST:-normal} --n 200000000 --reps 2 2>&1 | tail -1; done
