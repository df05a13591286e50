# Everything the round's evidence needs, in one call.
bash scripts/gpu_full_check.sh
bash scripts/gpu_configs.sh
timeout 900 python scripts/sweep.py > gpurun_out/sweeps.jsonl 2> gpurun_out/sweeps.err; echo "sweep rc=$?"
