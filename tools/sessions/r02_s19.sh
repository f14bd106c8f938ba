# session 19: staged VL=16 kernel (C5 T=5 sum), 3 vs 4 blocks per SM: cold (20 it) and sustained (600 it);
# the new 4-block tap defaults (C4, C5 T=9) re-timed the same way
OUT=gpurun_out/s19_blocks.txt; rm -f $OUT
for rep in 1 2; do
  for lib in libsbp.so libsbp_stg4.so; do
    for n in 20 600; do
      SBP_LIB=$lib timeout 300 python tools/kbench.py C5_T5 sum $n | python -c "import sys,json; d=json.load(sys.stdin); print('$lib it=$n', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $OUT 2>&1
    done
  done
done
for c in "C4 300" "C5_T9 600" "C5_T2 600" "C5_T17 600" "C5_T33 400"; do set -- $c
  timeout 300 python tools/kbench.py $1 sum $2 | python -c "import sys,json; d=json.load(sys.stdin); print('default it=$2', d['config'], d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $OUT 2>&1
done
cat $OUT
