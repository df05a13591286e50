# Round 2: ncu --set full of the four uniform-path kernels (200M Normal, second sort)
# and of the big path on config 4 (telemetry), plus the launch list of the bench command.
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
P="python scripts/prof_sort.py --dist normal --n 200000000 --reps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter0r|k_count1|k_scatter1|k_warpsort" -s 4 -c 4 -f -o gpurun_out/r2_uni $P > gpurun_out/ncu_uni.log 2>&1
echo "ncu uni rc=$?"; tail -2 gpurun_out/ncu_uni.log
