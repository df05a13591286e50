# Round evidence: bench line, ncu launch list of the same command, one full capture of the hot kernels.
set -x
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
BENCH="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-configs"
$BENCH > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
P="python scripts/prof_sort.py --dist normal --n 200000000 --reps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_count0|k_scatter0|k_count1|k_scatter1|k_warpsort|k_bucketsort" -s 7 -c 8 -o gpurun_out/prof_full $P > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
