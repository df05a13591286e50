# usage: DISTS="normal twodups" bash scripts/gpu_launch_dist.sh  (per-kernel launch list for prof_sort runs)
make -j8 > gpurun_out/make.log 2>&1 || exit 1
for d in ${DISTS:-normal twodups}; do
  P="python scripts/prof_sort.py --dist $d --n ${N:-200000000} --reps 2"
  timeout 300 $P > gpurun_out/pl_$d.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$d.csv $P > /dev/null 2>&1
  echo "$d rc=$?"
done
