# C4 band-kernel variants with the packed build: cold (kbench) and sustained (bench --kernel-only)
out=gpurun_out/ab_c4_variants.txt
rm -f $out
VARS="X=0 SBP_ROLL_MIN_R=99 SBP_BAND_VL=8 SBP_ROLL_MIN_R=99,SBP_BAND_VL=8 SBP_STAGED=1,SBP_ROLL_MIN_R=99 SBP_STAGED=2,SBP_ROLL_MIN_R=99"
for v in $VARS; do
  env ${v//,/ } python tools/kbench.py C4 sum 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $v', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4))" >> $out
done
for rep in 1 2; do
  for v in $VARS; do
    env ${v//,/ } python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('sustained $v', r['kernel'], round(r['ms_per_iteration'],4), round(r['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> $out
  done
done
cat $out
