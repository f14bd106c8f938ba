# round-2 session 4: full GPU tests, tap2+TMA A/B, strip host cost, bench line
mkdir -p gpurun_out
ab() {  # ab <tag> <cfg> <dom> [ENV=VAL ...]
  tag=$1; cfg=$2; dom=$3; shift 3
  env "$@" timeout 300 python tools/kbench.py $cfg $dom 20 | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/s4_ab.jsonl 2>>gpurun_out/s4_ab.err
}
for c in C5_T9 C5_T17 C5_T33; do
  for d in sum max; do
    ab default $c $d
    ab tap2 $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=2 SBP_TAP_ROLLED=1
    ab tap2stg $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=3 SBP_TAP_ROLLED=0
    ab tap2stg_roll $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=3 SBP_TAP_ROLLED=1
    ab tap16 $c $d SBP_TAP=1 SBP_TAP_VL=16
  done
done
timeout 300 python tools/strip_host_cost.py 2 4 8 > gpurun_out/s4_strip_host.jsonl 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --maxfail=30 --timeout 900 -p no:cacheprovider > gpurun_out/s4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4_pytest.log
timeout 900 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
echo "bench rc=$?" >> gpurun_out/s4_bench.err
