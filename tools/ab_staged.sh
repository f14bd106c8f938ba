# A/B: TMA-staged band kernel vs register-loaded, C4 sum / C3 max / C5 T9 sum (50 iterations)
rm -f gpurun_out/ab_staged.txt
for rep in 1 2; do
  for c in C4:sum C3:max C5_T9:sum C5_T2:sum; do
    n=${c%%:*}; d=${c##*:}
    for stg in 0 1; do
      for vl in 8 16; do
        if [ "$vl" = "16" ] && [ "$d" = "max" ]; then continue; fi
        SBP_STAGED=$stg SBP_BAND_VL=$vl python tools/kbench.py $n $d 50 | python -c "import sys,json; d=json.load(sys.stdin); print('$c staged=$stg vl=$vl', round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> gpurun_out/ab_staged.txt
      done
    done
  done
done
