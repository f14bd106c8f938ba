# A/B of the band kernel lane width on C4 (alternating, 50 iterations each)
rm -f gpurun_out/ab_vl.txt
for rep in 1 2 3; do
  for vl in 8 16; do
    SBP_BAND_VL=$vl python tools/kbench.py C4 sum 50 | python -c "import sys,json; d=json.load(sys.stdin); print('vl=$vl', round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> gpurun_out/ab_vl.txt
  done
done
