set -x
for pf in 1 0; do for vl in 8 16; do
  SBP_PREFETCH=$pf SBP_BAND_VL=$vl python tools/kbench.py C4 sum 30 >> gpurun_out/sweep.jsonl 2>>gpurun_out/sweep.err; echo "pf=$pf vl=$vl" >> gpurun_out/sweep.jsonl
done; done
for c in C3:max C5_T2:sum C5_T9:sum C5_T33:sum C5_T9:max C5_T33:max C2:sum; do
  n=${c%%:*}; d=${c##*:}
  for vl in 8 16; do SBP_BAND_VL=$vl python tools/kbench.py $n $d 10 >> gpurun_out/sweep.jsonl 2>>gpurun_out/sweep.err; echo "vl=$vl" >> gpurun_out/sweep.jsonl; done
done
