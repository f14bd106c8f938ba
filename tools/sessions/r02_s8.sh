# round-2 session 8: tap2 register double-buffering A/B
mkdir -p gpurun_out
ab() {
  tag=$1; cfg=$2; dom=$3; shift 3
  env "$@" timeout 300 python tools/kbench.py $cfg $dom 20 | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/s8_ab.jsonl 2>>gpurun_out/s8_ab.err
}
for c in C5_T9 C5_T17 C5_T33; do
  for d in sum max; do
    ab default $c $d
    ab regpf $c $d SBP_TAP_STAGED=5
    ab regpf_r2 $c $d SBP_TAP_STAGED=5 SBP_TAP_ROLLED=2
    ab regpf_r1 $c $d SBP_TAP_STAGED=5 SBP_TAP_ROLLED=1
    ab regpf_r0 $c $d SBP_TAP_STAGED=5 SBP_TAP_ROLLED=0
  done
done
