# fused kernel A/B (after the 32-bit unit walk): C4 ms/iteration + ncu counters
out=gpurun_out/ab_fused2.txt
rm -f $out
kb() {
  env $1 python tools/kbench.py $2 $3 20 | python -c "import sys,json; d=json.load(sys.stdin); print('cold $2:$3 $1', d['kernel_name'], round(d['median_ms'],4), round(d['min_ms'],4))" >> $out 2>&1
}
for v in SBP_FUSE=1 "SBP_FUSE=2 SBP_FUSE_ROUNDS=1" "SBP_FUSE=2 SBP_FUSE_ROUNDS=2" "SBP_FUSE=2 SBP_FUSE_ROUNDS=3" "SBP_FUSE=3 SBP_FUSE_ROUNDS=2" "SBP_FUSE=2 SBP_FUSE_ROUNDS=2 SBP_FUSE_ROLLED=0"; do
  kb "$v" C4 sum
done
for v in SBP_FUSE=1 "SBP_FUSE=2 SBP_FUSE_ROUNDS=2"; do kb "$v" C3 max; kb "$v" C5_T2 sum; done
for v in "SBP_FUSE=1" "SBP_FUSE=2 SBP_FUSE_ROUNDS=2"; do
  echo "# ncu $v" >> $out
  env $v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:band_ -s 3 -c 1 --csv python tools/kbench.py C4 sum 4 2>/dev/null | grep -v "^==" | grep '^"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
cat $out
