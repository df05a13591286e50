timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log | grep -v "^$"
for d in ${DISTS:-normal zipf twodups telemetry}; do timeout 300 python scripts/prof_sort.py --dist $d --n 200000000 --reps 3 2>&1 | tail -1; done
