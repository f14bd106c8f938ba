# ncu evidence for the fused (temporally blocked) kernel on C4.
export SBP_FUSE=2
NCU_KERNEL=band_fused NCU_SKIP=2 bash tools/ncu_one.sh fused2 python tools/kbench.py C4 sum 4
rm -f gpurun_out/ncu_fused_metrics.csv
for v in "SBP_FUSE=2" "SBP_FUSE=3 SBP_FUSE_ROUNDS=2" "SBP_FUSE=2 SBP_FUSE_ROUNDS=4" "SBP_FUSE=1"; do
  echo "# $v" >> gpurun_out/ncu_fused_metrics.csv
  env $v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:band_ -s 2 -c 1 --csv python tools/kbench.py C4 sum 4 2>/dev/null | grep -v "^==" >> gpurun_out/ncu_fused_metrics.csv
done
