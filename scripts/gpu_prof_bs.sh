timeout 300 python scripts/prof_sort.py --dist normal --n 50000000 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bucketsort|k_scatter1" -s 2 -c 2 -o gpurun_out/prof_r3 python scripts/prof_sort.py --dist normal --n 50000000 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/ncu_full.log
