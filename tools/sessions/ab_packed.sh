# Packed-FP32 (FFMA2/FADD2/FMUL2) band kernels vs the scalar build.
#  1. bitwise: every build and variant must give the same messages + labels
#  2. C4 sustained (bench --kernel-only) and cold (kbench) per build/variant
#  3. other configs, cold, default variant per build
# Builds: libsbp.so (packed, label-pair x weight-pair form), libsbp_f1.so
# (packed, broadcast-weight form; that form has since been removed, so this
# script is the record of the round-1 run, profiles/r01_ab_packed.txt),
# libsbp_scalar.so (scalar FP32 ops):
#   make -C paper_1010_0012_b200/csrc BUILD=_build_scalar EXTRA=-DSBP_SCALAR_F32 LIB=../libsbp_scalar.so
out=gpurun_out/ab_packed.txt
rm -f $out
LIBS="libsbp.so libsbp_f1.so libsbp_scalar.so"
for c in "C2 sum 20" "C2 max 20" "C3 max 10" "C5_T9 sum 5" "C4 sum 5" "C2 max 3 288 384 sequential"; do
  for l in $LIBS; do
    for v in "X=0" "SBP_STAGED=0" "SBP_ROLL_MIN_R=1,SBP_STAGED=0"; do
      echo "hash $c $l $v $(env SBP_LIB=$l ${v//,/ } python tools/lib_hash.py $c)" >> $out
    done
  done
done
for rep in 1 2; do
  for l in $LIBS; do
    for v in "X=0" "SBP_ROLL_MIN_R=1"; do
      env SBP_LIB=$l ${v//,/ } python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sustained C4 $l $v', d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> $out
    done
  done
done
for l in $LIBS; do
  for v in "X=0" "SBP_ROLL_MIN_R=1"; do
    env SBP_LIB=$l ${v//,/ } python tools/kbench.py C4 sum 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold C4 $l $v', d.get('kernel_name'), round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $out
  done
done
for c in C2:sum C2:max C3:max C5_T2:sum C5_T5:sum C5_T9:sum C5_T17:sum C5_T33:sum C5_T5:max C5_T17:max; do
  n=${c%%:*}; d=${c##*:}
  for l in $LIBS; do
    for v in "X=0" "SBP_STAGED=0"; do
      env SBP_LIB=$l ${v//,/ } python tools/kbench.py $n $d 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $c $l $v', d['kernel_name'], round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $out
    done
  done
done
cat $out
