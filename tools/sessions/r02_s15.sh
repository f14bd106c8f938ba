# session 15: redux max in the band / staged / tap2 max-sum kernels (Ms = 256, R <= 16): timings, hashes, full GPU suite
OUT=gpurun_out/s15_redux.txt; rm -f $OUT
for c in C5_T9 C5_T17 C5_T33; do
  timeout 300 python tools/lib_hash.py $c max 5 24 40 | python -c "import sys,json; d=json.load(sys.stdin); print('hash', d['config'], d['kernel'], d['sha'])" >> $OUT 2>&1
done
for rep in 1 2; do
  for c in C3 C5_T2 C5_T5 C5_T9 C5_T17 C5_T33; do
    timeout 300 python tools/kbench.py $c max 20 | python -c "import sys,json; d=json.load(sys.stdin); print(d['config'], d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4))" >> $OUT 2>&1
  done
done
cat $OUT
timeout 2400 python -m pytest tests -m gpu -q -rf --maxfail=30 --timeout 900 -p no:cacheprovider > gpurun_out/s15_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s15_pytest.log
tail -4 gpurun_out/s15_pytest.log
