# round-2 session 9: verification checkpoint -- tests, smoke, full-size parity report, bench (both arms), ncu C4
mkdir -p gpurun_out/r02_final
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/r02_final/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_final/smoke.log
timeout 900 python tools/fullsize_report.py > gpurun_out/r02_final/fullsize_parity.jsonl 2> gpurun_out/r02_final/fullsize_parity.err
timeout 900 python bench.py > gpurun_out/r02_final/bench.json 2> gpurun_out/r02_final/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_final/bench_reference.json 2> gpurun_out/r02_final/bench_reference.err
timeout 600 python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/r02_final/bench_k.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_final/launches_c4.csv python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/r02_final/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_iter -s 3 -c 1 -o /tmp/c4full python bench.py --steps 1 --warmup 1 --kernel-only > gpurun_out/r02_final/ncu_full.log 2>&1
ncu -i /tmp/c4full.ncu-rep --page details > gpurun_out/r02_final/ncu_c4_details.txt 2>/dev/null
ncu -i /tmp/c4full.ncu-rep --page raw --csv > gpurun_out/r02_final/ncu_c4_raw.csv 2>/dev/null
