set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
for d in normal zipf twodups telemetry rootdups; do timeout 300 python scripts/prof_sort.py --dist $d --n 200000000 --reps 3 2>&1 | tail -1; done
timeout 300 python scripts/prof_sort.py --n 50000000 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_sort.py --n 50000000 > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_count0|k_scatter0|k_bucketsort|k_count1|k_scatter1" -s 5 -c 5 -o gpurun_out/prof_r1 python scripts/prof_sort.py --n 50000000 > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_full.log
