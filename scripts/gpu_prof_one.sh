# ncu --set full of one kernel (regex $K) in a 200M sort of $DIST (second call).
make -j8 > gpurun_out/make.log 2>&1 || { echo "make failed"; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:${K}" -s ${SKIP:-1} -c 1 -f -o gpurun_out/${OUT:-prof} python scripts/prof_sort.py --dist ${DIST:-normal} --n ${N:-200000000} --reps 2 > gpurun_out/ncu_one.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_one.log
