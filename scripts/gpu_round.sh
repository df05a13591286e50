# One GPU pass: smoke, GPU parity tests, per-distribution phase timings, bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
for d in ${DISTS:-normal lognormal exponential mixgauss uniform zipf rootdups twodups telemetry uniform_u64}; do timeout 300 python scripts/prof_sort.py --dist $d --n 200000000 --reps 3 2>&1 | tail -1; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench.log
