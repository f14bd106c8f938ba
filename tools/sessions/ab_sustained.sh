# Sustained + cold A/B of band-kernel variants on the bench workload (C4).
# Variants: register-loaded VL=8 / VL=16, TMA-staged VL=8 (2 buffers) / VL=16 (1 buffer).
rm -f gpurun_out/ab_sustained.txt
VARS="SBP_STAGED=0,SBP_BAND_VL=8 SBP_STAGED=0,SBP_BAND_VL=16 SBP_STAGED=1 SBP_STAGED=2"
for rep in 1 2; do
  for v in $VARS; do
    env ${v//,/ } python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), round(d['value']/1e9,3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> gpurun_out/ab_sustained.txt
  done
done
for v in $VARS; do
  env ${v//,/ } python tools/kbench.py C4 sum 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $v', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4))" >> gpurun_out/ab_sustained.txt
done
cat gpurun_out/ab_sustained.txt
