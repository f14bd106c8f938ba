# session 18: C5 T=9 sum tap v1 VL=16, 3 vs 4 blocks per SM: cold (20 it) and sustained (600 it) A/B
OUT=gpurun_out/s18_t9_blocks.txt; rm -f $OUT
for rep in 1 2; do
  for lib in libsbp.so libsbp_t9b4.so; do
    for n in 20 600; do
      SBP_LIB=$lib timeout 300 python tools/kbench.py C5_T9 sum $n | python -c "import sys,json; d=json.load(sys.stdin); print('$lib it=$n', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $OUT 2>&1
    done
  done
done
cat $OUT
