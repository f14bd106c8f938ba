# session 17: C4 tap kernel, 3 vs 4 blocks per SM (146 vs 128 registers, no spills): cold + sustained A/B
OUT=gpurun_out/s17_tap_blocks.txt; rm -f $OUT
for lib in libsbp.so libsbp_b4.so; do
  SBP_LIB=$lib timeout 300 python tools/lib_hash.py C4 sum 3 96 128 | python -c "import sys,json; d=json.load(sys.stdin); print('hash $lib', d['kernel'], d['sha'])" >> $OUT 2>&1
  SBP_LIB=$lib timeout 300 python tools/kbench.py C4 sum 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $lib', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $OUT 2>&1
done
for rep in 1 2 3; do
  for lib in libsbp.so libsbp_b4.so; do
    SBP_LIB=$lib timeout 600 python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sustained $lib', d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), round(d['value']/1e9,3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> $OUT 2>&1
  done
done
cat $OUT
