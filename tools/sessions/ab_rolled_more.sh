# rolled vs default variants on the other configs with compiled rolled radii
out=gpurun_out/ab_rolled_more.txt
rm -f $out
for c in C5_T5:max C5_T5:sum C5_T9:sum C5_T9:max; do
  n=${c%%:*}; d=${c##*:}
  for v in "X=0" "SBP_ROLL_MIN_R=1,SBP_STAGED=0" "SBP_ROLL_MIN_R=99,SBP_STAGED=0"; do
    env ${v//,/ } python tools/kbench.py $n $d 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $c $v', d['kernel_name'], round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $out
  done
done
cat $out
