set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for d in normal lognormal exponential mixgauss zipf twodups telemetry rootdups uniform_u64; do timeout 300 python scripts/prof_sort.py --dist $d --n 200000000 --reps 3 2>&1 | tail -1; done
timeout 300 python scripts/prof_sort.py --dist telemetry --n 20000000 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bucketsort|k_big" -s 8 -c 4 -o gpurun_out/prof_r2 python scripts/prof_sort.py --dist telemetry --n 20000000 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/ncu_full.log
