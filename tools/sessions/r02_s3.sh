# round-2 session 3: GPU tests, tap2 A/B, ncu of the wide-band kernels, memcheck
mkdir -p gpurun_out
ab() {  # ab <tag> <cfg> <dom> [ENV=VAL ...]
  tag=$1; cfg=$2; dom=$3; shift 3
  env "$@" timeout 300 python tools/kbench.py $cfg $dom 20 | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/s3_ab.jsonl 2>>gpurun_out/s3_ab.err
}
for c in C5_T9 C5_T17 C5_T33; do
  for d in sum max; do
    ab default $c $d
    ab tap2 $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=2 SBP_TAP_ROLLED=0
    ab tap2_roll $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=2 SBP_TAP_ROLLED=1
  done
done
for c in "C5_T33 sum" "C5_T33 max" "C5_T17 max"; do
  set -- $c
  SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=2 SBP_TAP_ROLLED=1 NCU_KERNEL=tap2 NCU_SKIP=4 timeout 600 bash tools/ncu_one.sh s3_$1_$2 python tools/kbench.py $1 $2 3
done
timeout 2400 python -m pytest tests -m gpu -q --maxfail=20 --timeout 900 -p no:cacheprovider > gpurun_out/s3_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s3_pytest.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/s3_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/s3_memcheck.log
