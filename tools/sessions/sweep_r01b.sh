# rolled (one band copy, symmetric potentials) vs unrolled, per config
for c in C4:sum C3:max C5_T2:sum C5_T9:sum C5_T17:sum C5_T33:sum C5_T9:max C5_T33:max; do
  n=${c%%:*}; d=${c##*:}
  for rr in 1 99; do
    SBP_ROLL_MIN_R=$rr python tools/kbench.py $n $d 10 >> gpurun_out/sweep_b.jsonl 2>>gpurun_out/sweep_b.err
    echo "roll_min_r=$rr" >> gpurun_out/sweep_b.jsonl
  done
done
for c in C5_T9:sum C5_T9:max C3:sum C4:sum; do
  n=${c%%:*}; d=${c##*:}
  python tools/kbench.py $n $d 3 standard >> gpurun_out/sweep_b.jsonl 2>>gpurun_out/sweep_b.err
  echo "dense" >> gpurun_out/sweep_b.jsonl
done
