# Same-box A/B (ab/libls_A.so = HEAD against the working tree's libls.so), after the GPU suite on the candidate.
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
timeout 1200 python -m pytest tests/ -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash scripts/ab.sh > gpurun_out/ab.log 2>&1; cat gpurun_out/ab.log
