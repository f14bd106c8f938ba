# Temporal blocking (sbp_iterate_fused) A/B: levels per launch, wavefront lag,
# work-unit rounds; kbench (ms per iteration, median of 20) and the
# sustained bench (--kernel-only).  Results: gpurun_out/ab_fused.txt
out=gpurun_out/ab_fused.txt
rm -f $out
kb() {  # env, config, domain
  env $1 python tools/kbench.py $2 $3 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $2:$3 $1', d['kernel_name'], round(d['median_ms'],4), round(d['min_ms'],4), round(d['hbm_frac'],4))" >> $out 2>&1
}
for v in SBP_FUSE=1 SBP_FUSE=2 SBP_FUSE=3 SBP_FUSE=4 "SBP_FUSE=2 SBP_FUSE_LAG=3" "SBP_FUSE=2 SBP_FUSE_LAG=6" "SBP_FUSE=2 SBP_FUSE_ROUNDS=2" "SBP_FUSE=2 SBP_FUSE_ROLLED=0" "SBP_FUSE=1 SBP_ROLL_MIN_R=99"; do
  kb "$v" C4 sum
done
for c in C3:max C5_T9:sum C5_T5:max C5_T2:sum C5_T17:sum; do
  for v in SBP_FUSE=1 SBP_FUSE=2 SBP_FUSE=3; do kb "$v" ${c%%:*} ${c##*:}; done
done
for v in SBP_FUSE=1 SBP_FUSE=2 SBP_FUSE=3 SBP_FUSE=4; do
  env $v python bench.py --kernel-only --steps 5 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('sustained C4 $v', r['kernel'], round(r['ms_per_iteration'],4), round(r['kernel_ms'],4), round(r['frac'],4), round(d['value']/1e9,3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" >> $out 2>&1
done
cat $out
