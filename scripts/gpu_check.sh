# Candidate check: GPU suite, randomised stress, phase timings at four sizes.
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python scripts/stress.py --seconds ${S1:-200} --seed ${SEED:-11} --max-n 30000000 > gpurun_out/stress.log 2>&1; echo "stress rc=$?"; tail -2 gpurun_out/stress.log
for n in 1000000 10000000 100000000 200000000; do echo "n=$n $(python scripts/prof_sort.py --n $n --reps 4 --dist normal | tail -1)"; done
