# One bench line per BASELINE workload (single GPU), for the record.
make -j8 > /dev/null 2>&1
for wl in c1_uniform01 c2_normal c2_lognormal c2_exponential c2_mixgauss c3_zipf c3_rootdups c3_twodups c4_telemetry ref_uniform01 ref_uniform_u64; do
  timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1
done > gpurun_out/configs.jsonl
timeout 600 python bench.py --force-multi --steps 3 --warmup 3 --no-e2e 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
wc -l gpurun_out/configs.jsonl
