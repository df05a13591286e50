# Launch list of the bench command + one `ncu --set full` capture of each hot kernel.
set -x
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
BENCH="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$BENCH > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
P="python scripts/prof_sort.py --dist normal --n 200000000 --reps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_count0|k_scatter0|k_count1|k_scatter1|k_bucketsort" -s 5 -c 5 -o gpurun_out/prof_r1_normal $P > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
