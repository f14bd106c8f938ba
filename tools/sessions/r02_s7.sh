# round-2 session 7: tap2 L2-prefetch / half-rolled A/B
mkdir -p gpurun_out
ab() {
  tag=$1; cfg=$2; dom=$3; shift 3
  env "$@" timeout 300 python tools/kbench.py $cfg $dom 20 | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/s7_ab.jsonl 2>>gpurun_out/s7_ab.err
}
for c in C5_T9 C5_T17 C5_T33; do
  for d in sum max; do
    ab default $c $d
    ab pf $c $d SBP_TAP_STAGED=4
    ab roll2 $c $d SBP_TAP_ROLLED=2
    ab pf_roll2 $c $d SBP_TAP_STAGED=4 SBP_TAP_ROLLED=2
    ab pf_roll1 $c $d SBP_TAP_STAGED=4 SBP_TAP_ROLLED=1
  done
done
for c in C4 C3; do ab default $c $( [ $c = C4 ] && echo sum || echo max ); done
