make -j8 > gpurun_out/make.log 2>&1 || exit 1
LS_DEBUG_STAGE=512 LS_GRAPH=0 python scripts/prof_sort.py --dist telemetry --n 200000000 --reps 2 > gpurun_out/bigprof.log 2>&1
tail -8 gpurun_out/bigprof.log
