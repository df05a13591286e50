# usage: KREGEX=... DIST=... N=... bash scripts/gpu_prof_k.sh   (ncu --set full on one kernel family)
timeout 300 python scripts/prof_sort.py --dist ${DIST:-normal} --n ${N:-50000000} > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_bucketsort}" -s ${SKIP:-1} -c ${CNT:-1} -o gpurun_out/${OUT:-prof_k} python scripts/prof_sort.py --dist ${DIST:-normal} --n ${N:-50000000} > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
