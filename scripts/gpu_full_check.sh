# Full GPU suite (incl. slow 200M tests), smoke, bench line + ncu evidence.
make -j8 > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_full.log
bash scripts/gpu_bench_evidence.sh > gpurun_out/evidence.log 2>&1; echo "evidence rc=$?"
cat gpurun_out/bench.json | cut -c1-300
