# current build (libsbp.so) vs the previous one (libsbp_prev.so): cold + sustained
out=gpurun_out/ab_prev.txt
rm -f $out
LIBS="libsbp.so ${ALT_LIB:-libsbp_prev.so}"
for c in C4:sum C3:max C5_T9:sum C5_T17:sum C5_T33:sum C2:sum; do
  n=${c%%:*}; d=${c##*:}
  for l in $LIBS; do
    env SBP_LIB=$l python tools/kbench.py $n $d 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $c $l', d['kernel_name'], round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $out
  done
done
for rep in 1 2; do
  for l in $LIBS; do
    env SBP_LIB=$l python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('sustained C4 $l', r['kernel'], round(r['ms_per_iteration'],4), round(r['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> $out
  done
done
cat $out
