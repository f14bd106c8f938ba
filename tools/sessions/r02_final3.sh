# Round-2 final evidence (after the tap C4 default, the tensor-core dense kernel and the redux maxima):
# smoke, bench (default) + reference arm, C4 launch list, ncu --set full of the C4 message kernel and the
# tensor-core dense kernel (the CTA-pair kernel without the two SASS-patching sections, which break it under
# ncu: profiles/r02_ncu_tc/s12.txt), sequential-schedule timing, full-size parity report.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f3_smoke.log
timeout 1500 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo "bench rc=$?" >> gpurun_out/f3_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f3_bench_ref.json 2> gpurun_out/f3_bench_ref.err
timeout 600 python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/f3_bench_k.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f3_launches_c4.csv \
      python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/f3_ncu_launch.log 2>&1
NCU_KERNEL=band_iter NCU_SKIP=5 timeout 900 bash tools/ncu_one.sh f3_c4 python bench.py --steps 1 --warmup 1 --kernel-only
NCU_KERNEL=dense_tc NCU_SKIP=3 timeout 500 bash tools/ncu_one.sh f3_tc_c4 python tools/kbench.py C4 sum 3 standard
timeout 600 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats \
    --section ComputeWorkloadAnalysis --section Occupancy --section LaunchStats --clock-control none -k regex:dense_tc -s 3 -c 1 \
    -o /tmp/prof_f3_tc_c5 python tools/kbench.py C5_T9 sum 3 standard > gpurun_out/ncu_f3_tc_c5.log 2>&1
ncu -i /tmp/prof_f3_tc_c5.ncu-rep --page details > gpurun_out/details_f3_tc_c5.txt 2>/dev/null
ncu -i /tmp/prof_f3_tc_c5.ncu-rep --page raw --csv > gpurun_out/raw_f3_tc_c5.csv 2>/dev/null
for c in "C5_T5 max" "C5_T17 max"; do set -- $c; NCU_KERNEL=band_iter NCU_SKIP=4 timeout 600 bash tools/ncu_one.sh f3_$1_$2 python tools/kbench.py $1 $2 3; done
timeout 600 python tools/kbench_seq.py C4 sum 5 > gpurun_out/f3_seq_c4.json 2>&1
for v in 1 2 0; do for c in C4 C5_T9; do SBP_DENSE_TC=$v timeout 300 python tools/kbench.py $c sum 20 standard; done; done > gpurun_out/f3_dense_arms.jsonl 2>&1
tail -3 gpurun_out/f3_smoke.log; tail -c 400 gpurun_out/f3_bench.err; cat gpurun_out/f3_bench_ref.json | head -c 600; echo; cat gpurun_out/f3_seq_c4.json; cat gpurun_out/f3_dense_arms.jsonl
