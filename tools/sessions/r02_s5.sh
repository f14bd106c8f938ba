# round-2 session 5: band instruction-stream ceiling, strip host cost, sub-row tap layouts A/B
mkdir -p gpurun_out
./tools/band_ceiling > gpurun_out/s5_ceiling.jsonl 2>&1
./tools/pipes > gpurun_out/s5_pipes.jsonl 2>&1
timeout 300 python tools/strip_host_cost.py 2 4 8 > gpurun_out/s5_strip_host.jsonl 2>&1
ab() {
  tag=$1; cfg=$2; dom=$3; shift 3
  env "$@" timeout 300 python tools/kbench.py $cfg $dom 20 | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/s5_ab.jsonl 2>>gpurun_out/s5_ab.err
}
for c in C5_T9 C5_T17 C5_T33; do
  for d in sum max; do
    ab default $c $d
    ab tap8 $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=0 SBP_TAP_ROLLED=0
    ab tap8r $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=0 SBP_TAP_ROLLED=1
    ab tap16 $c $d SBP_TAP=1 SBP_TAP_VL=16
    ab tap2 $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=2 SBP_TAP_ROLLED=0
    ab tap2r $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=2 SBP_TAP_ROLLED=1
    ab tap2s $c $d SBP_TAP=1 SBP_TAP_VL=8 SBP_TAP_STAGED=3 SBP_TAP_ROLLED=0
  done
done
