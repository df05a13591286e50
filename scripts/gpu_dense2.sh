make -j8 > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "dense" > gpurun_out/pytest_dense.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_dense.log
LS_DEBUG_STAGE=512 LS_GRAPH=0 python scripts/prof_sort.py --dist telemetry --n 200000000 --reps 2 2>&1 | tail -4
