./scripts/probe/cluster_occ
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "multi" > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -3 gpurun_out/pytest_multi.log
