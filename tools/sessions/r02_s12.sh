# session 12: is the CTA-pair tensor-core kernel robust?  stress + ncu section by section
mkdir -p gpurun_out
OUT=gpurun_out/s12.txt; rm -f $OUT
timeout 300 python tools/kbench.py C5_T9 sum 1500 standard >> $OUT 2>&1; echo "stress rc=$?" >> $OUT
SBP_MAX_BLOCKS=3 timeout 300 python tools/kbench.py C5_T9 sum 20 standard >> $OUT 2>&1; echo "cap3 rc=$?" >> $OUT
for sec in SpeedOfLight MemoryWorkloadAnalysis WarpStateStats SourceCounters InstructionStats LaunchStats Occupancy SchedulerStats ComputeWorkloadAnalysis; do
  timeout 300 ncu --section $sec --clock-control none -k regex:dense_tc -s 3 -c 1 python tools/kbench.py C5_T9 sum 3 standard > gpurun_out/s12_ncu_$sec.log 2>&1
  echo "ncu $sec rc=$? $(grep -c LaunchFailed gpurun_out/s12_ncu_$sec.log)" >> $OUT
done
cat $OUT
