# Everything the round's evidence needs, in one call.
bash scripts/gpu_bench_evidence.sh
bash scripts/gpu_configs.sh
timeout 900 python scripts/sweep.py > gpurun_out/sweeps.jsonl 2> gpurun_out/sweeps.err; echo "sweep rc=$?"
timeout 300 python scripts/graph_latency.py > gpurun_out/graph_latency.jsonl 2> gpurun_out/graph_latency.err; echo "graph rc=$?"
