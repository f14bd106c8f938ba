# sequential-schedule (chain kernel) A/B: libsbp.so vs ${ALT_LIB}
out=gpurun_out/ab_seq.txt
rm -f $out
for c in "C4 sum" "C2 max" "C3 max" "C5_T9 sum"; do
  for l in libsbp.so ${ALT_LIB:-libsbp_prev.so}; do
    echo "$c $l $(env SBP_LIB=$l python tools/kbench_seq.py $c 5)" >> $out
  done
done
cat $out
