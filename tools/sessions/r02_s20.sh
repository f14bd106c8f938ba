# session 20: C3 max staged VL=8 kernel: natural 119 registers (4 blocks) vs bounded to 5 blocks (95 registers): cold + sustained
OUT=gpurun_out/s20_c3_blocks.txt; rm -f $OUT
for rep in 1 2; do
  for lib in libsbp.so libsbp_c3b5.so; do
    for n in 100 2000; do
      SBP_LIB=$lib timeout 300 python tools/kbench.py C3 max $n | python -c "import sys,json; d=json.load(sys.stdin); print('$lib it=$n', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $OUT 2>&1
    done
  done
done
for lib in libsbp.so libsbp_c3b5.so; do SBP_LIB=$lib timeout 300 python tools/lib_hash.py C3 max 5 64 96 | python -c "import sys,json; d=json.load(sys.stdin); print('hash $lib', d['kernel'], d['sha'])" >> $OUT 2>&1; done
cat $OUT
