# session 21: direction-loop variants of the tap2 kernels on the final build (redux maxima, 4-block bounds)
OUT=gpurun_out/s21_rolled.txt; rm -f $OUT
for c in "C5_T17 max" "C5_T33 max" "C5_T9 max" "C5_T17 sum" "C5_T33 sum"; do set -- $c
  for r in default 0 1 2; do
    if [ $r = default ]; then E="X=0"; else E="SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=2 SBP_TAP_ROLLED=$r"; fi
    env $E timeout 300 python tools/kbench.py $1 $2 200 | python -c "import sys,json; d=json.load(sys.stdin); print('$1 $2 rolled=$r', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4))" >> $OUT 2>&1
  done
done
cat $OUT
