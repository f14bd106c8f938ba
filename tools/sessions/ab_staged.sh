# A/B of band-kernel variants per config (kbench, 30 iterations, cold-ish single launches)
rm -f gpurun_out/ab_staged.txt
for c in C2:sum C2:max C3:max C5_T2:sum C5_T5:sum C5_T9:sum C5_T17:sum C5_T5:max; do
  n=${c%%:*}; d=${c##*:}
  for v in "SBP_STAGED=0,SBP_BAND_VL=8" "SBP_STAGED=0,SBP_BAND_VL=16" "SBP_STAGED=1" "SBP_STAGED=2" "DEFAULT=1"; do
    env ${v//,/ } python tools/kbench.py $n $d 30 | python -c "import sys,json; d=json.load(sys.stdin); print('$c $v', d['kernel_name'], round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> gpurun_out/ab_staged.txt
  done
done
cat gpurun_out/ab_staged.txt
