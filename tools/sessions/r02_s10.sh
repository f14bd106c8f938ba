# round-2 session 10: C4 (R = 7) on the shared-memory-tap kernels (R lifted to 8): cold + sustained A/B
mkdir -p gpurun_out
OUT=gpurun_out/s10_c4_tap.txt
rm -f $OUT
VARS="X=0 SBP_TAP=1,SBP_TAP_LIFT=1 SBP_TAP=1,SBP_TAP_LIFT=1,SBP_TAP_ROLLED=1 SBP_TAP=1,SBP_TAP_LIFT=1,SBP_TAP_VL=8 SBP_TAP=1,SBP_TAP_LIFT=1,SBP_TAP_VL=8,SBP_TAP_ROLLED=1 SBP_TAP=1,SBP_TAP_LIFT=1,SBP_TAP_VL=8,SBP_TAP_STAGED=5 SBP_TAP=1,SBP_TAP_LIFT=1,SBP_TAP_VL=8,SBP_TAP_STAGED=3 SBP_TAP=1,SBP_TAP_LIFT=1,SBP_TAP_VL=8,SBP_TAP_STAGED=0"
for v in $VARS; do
  env ${v//,/ } timeout 300 python tools/lib_hash.py C4 sum 3 96 128 | python -c "import sys,json; d=json.load(sys.stdin); print('hash $v', d['kernel'], d['sha'])" >> $OUT 2>&1
done
for v in $VARS; do
  env ${v//,/ } timeout 300 python tools/kbench.py C4 sum 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $v', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $OUT 2>&1
done
for rep in 1 2; do
  for v in $VARS; do
    env ${v//,/ } timeout 600 python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sustained $v', d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), round(d['value']/1e9,3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> $OUT 2>&1
  done
done
cat $OUT
