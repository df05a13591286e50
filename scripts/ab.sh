# A/B of two prebuilt libraries on the same box: /root/repo/ab/libls_A.so (baseline)
# against the in-tree libls.so (candidate), DISTS x ROUNDS, the order of A and
# B alternating between rounds (no warm-box bias toward either).
for r in $(seq 1 ${ROUNDS:-3}); do
  for d in ${DISTS:-normal}; do
    a="A $d $(LS_LIBPATH=$PWD/ab/libls_A.so python scripts/prof_sort.py --n ${N:-200000000} --reps 3 --dist $d | tail -1)"
    if [ $((r % 2)) -eq 1 ]; then echo "$a"; fi
    echo "B $d $(python scripts/prof_sort.py --n ${N:-200000000} --reps 3 --dist $d | tail -1)"
    if [ $((r % 2)) -eq 0 ]; then echo "$a"; fi
  done
done
