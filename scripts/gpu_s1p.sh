# k_scatter1p (LS_SCATTER1P=1) against k_scatter1: GPU suite with it on, then interleaved phase timings.
make -j8 > gpurun_out/make.log 2>&1; echo "make rc=$?"
LS_SCATTER1P=1 timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_s1p.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_s1p.log
for r in 1 2; do for d in ${DISTS:-normal twodups telemetry zipf}; do for v in 0 1; do
  echo "S1P=$v $d $(LS_SCATTER1P=$v python scripts/prof_sort.py --n 200000000 --reps 3 --dist $d | tail -1)"
done; done; done
for v in 0 1; do echo "S1P=$v 1M $(LS_SCATTER1P=$v python scripts/prof_sort.py --n 1000000 --reps 4 --dist normal | tail -1)"; done
for v in 0 1; do echo "S1P=$v 1B $(LS_SCATTER1P=$v python scripts/prof_sort.py --n 1000000000 --reps 3 --dist normal | tail -1)"; done
