# Quick check after a kernel change: build, phase times at 200M for a few
# distributions, then (optionally) the GPU test suite.
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
for d in ${DISTS:-normal zipf telemetry}; do
  timeout 120 python scripts/prof_sort.py --n ${N:-200000000} --reps 3 --dist $d ${FLAGS:+--flags $FLAGS} 2>&1 | tail -1
done
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest tests/ -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -8
fi
