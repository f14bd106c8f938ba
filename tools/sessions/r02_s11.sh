# round-2 session 11: full GPU suite with the tap C4 default and the tensor-core dense kernel; ncu of the TC kernel
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --maxfail=30 --timeout 900 -p no:cacheprovider > gpurun_out/s11_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s11_pytest.log
tail -5 gpurun_out/s11_pytest.log
NCU_KERNEL=dense_tc NCU_SKIP=3 timeout 500 bash tools/ncu_one.sh s11_tc_c4 python tools/kbench.py C4 sum 3 standard
NCU_KERNEL=dense_tc NCU_SKIP=3 timeout 500 bash tools/ncu_one.sh s11_tc_c5 python tools/kbench.py C5_T9 sum 3 standard
NCU_KERNEL=band_iter_tap NCU_SKIP=3 timeout 500 bash tools/ncu_one.sh s11_c4_tap python tools/kbench.py C4 sum 3
