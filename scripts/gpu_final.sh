# Round-end pass: build, smoke, full GPU suite, then every piece of round evidence.
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_full.log
bash scripts/gpu_round_evidence.sh > gpurun_out/evidence.log 2>&1; echo "evidence rc=$?"
cut -c1-400 gpurun_out/bench.json
