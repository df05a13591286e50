# One `ncu --set full` capture of the hot kernels of one sort (second repetition).
set -x
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
P="python scripts/prof_sort.py --dist ${DIST:-normal} --n ${N:-200000000} --reps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_count0|k_scatter0|k_count1|k_scatter1|k_bucketsort}" -s ${SKIP:-5} -c ${CNT:-5} -o gpurun_out/${OUT:-prof} $P > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
