# round-2 session 2: GPU tests, pipe microbenchmarks, tap-kernel A/B on C5 wide bands
mkdir -p gpurun_out
./tools/pipes > gpurun_out/s2_pipes.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/s2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2_pytest.log
ab() {  # ab <tag> <cfg> <dom> [ENV=VAL ...]
  tag=$1; cfg=$2; dom=$3; shift 3
  env "$@" timeout 300 python tools/kbench.py $cfg $dom 20 | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/s2_ab.jsonl 2>>gpurun_out/s2_ab.err
}
for c in C5_T9 C5_T17 C5_T33; do
  for d in sum max; do
    ab default $c $d
    ab tap $c $d SBP_TAP=1
    ab tap_stg $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=1
    ab tap_reg8 $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=0
    ab tap_roll $c $d SBP_TAP=1 SBP_TAP_ROLLED=1
    ab tap_unroll $c $d SBP_TAP=1 SBP_TAP_ROLLED=0
  done
done
ab default C4 sum
ab default C3 max
