# Round-end evidence: GPU tests, smoke, bench (default), launch list, one ncu
# --set full capture of the bench's message kernel, sequential-schedule timing.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/final_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
      python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/final_ncu_launch.log 2>&1
NCU_KERNEL=band_iter NCU_SKIP=5 timeout 900 bash tools/ncu_one.sh final_c4 python bench.py --steps 1 --warmup 1 --kernel-only
python tools/kbench_seq.py C4 sum 5 > gpurun_out/final_seq_c4.json 2>&1
tail -2 gpurun_out/final_pytest_gpu.log; cat gpurun_out/final_bench.json gpurun_out/final_bench_ref.json gpurun_out/final_seq_c4.json
