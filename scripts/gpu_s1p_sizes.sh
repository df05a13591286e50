make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
for r in 1 2; do for n in 100000 1000000 4000000 10000000 30000000 100000000; do for v in 0 1; do
  echo "S1P=$v n=$n $(LS_SCATTER1P=$v python scripts/prof_sort.py --n $n --reps 5 --dist ${D:-normal} | tail -1)"
done; done; done
