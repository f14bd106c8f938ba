# session 14: CREDUX.MAX.F32 for the warp-wide max of the Ms = 256 max-sum tap kernels (A/B)
OUT=gpurun_out/s14_redux.txt; rm -f $OUT
for lib in libsbp.so libsbp_redux.so; do
  for c in C5_T9 C5_T17 C5_T33; do
    SBP_LIB=$lib timeout 300 python tools/lib_hash.py $c max 5 24 40 | python -c "import sys,json; d=json.load(sys.stdin); print('hash $lib', d['config'], d['kernel'], d['sha'])" >> $OUT 2>&1
  done
done
for rep in 1 2; do
  for lib in libsbp.so libsbp_redux.so; do
    for c in C5_T2 C5_T5 C5_T9 C5_T17 C5_T33; do
      SBP_LIB=$lib timeout 300 python tools/kbench.py $c max 20 | python -c "import sys,json; d=json.load(sys.stdin); print('$lib', d['config'], d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4))" >> $OUT 2>&1
    done
  done
done
cat $OUT
