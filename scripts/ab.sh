# A/B of two prebuilt libraries on the same box: /root/repo/ab/libls_A.so (baseline)
# against the in-tree libls.so (candidate), interleaved, DISTS x ROUNDS.
for r in $(seq 1 ${ROUNDS:-3}); do
  for d in ${DISTS:-normal}; do
    echo "A $d $(LS_LIBPATH=$PWD/ab/libls_A.so python scripts/prof_sort.py --n ${N:-200000000} --reps 3 --dist $d | tail -1)"
    echo "B $d $(python scripts/prof_sort.py --n ${N:-200000000} --reps 3 --dist $d | tail -1)"
  done
done
