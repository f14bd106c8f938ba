# session 22: C4 tap kernel, 4 vs 5 blocks per SM (128 registers vs 96 + 164 B of spills): sustained A/B
OUT=gpurun_out/s22_tap_b5.txt; rm -f $OUT
for rep in 1 2 3; do
  for lib in libsbp.so libsbp_b5.so; do
    SBP_LIB=$lib timeout 600 python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sustained $lib', d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), round(d['value']/1e9,3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> $OUT 2>&1
  done
done
cat $OUT
