# round-2 session 6: GPU tests with the tap defaults, bench line, ncu of the new defaults + C4 launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --maxfail=30 --timeout 900 -p no:cacheprovider > gpurun_out/s6_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s6_pytest.log
timeout 900 python bench.py > gpurun_out/s6_bench.json 2> gpurun_out/s6_bench.err
echo "bench rc=$?" >> gpurun_out/s6_bench.err
timeout 600 python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/s6_bench_k.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s6_launches_c4.csv python bench.py --steps 2 --warmup 1 --kernel-only > gpurun_out/s6_ncu_launch.log 2>&1
for c in "C5_T33 sum" "C5_T33 max" "C5_T17 max" "C5_T17 sum"; do
  set -- $c
  NCU_KERNEL=tap NCU_SKIP=4 timeout 600 bash tools/ncu_one.sh s6_$1_$2 python tools/kbench.py $1 $2 3
done
