# round-2 session 1: pipe microbenchmarks, C5 wide-band kernel timings, ncu --set full captures
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/s1_smi.txt
./tools/pipes > gpurun_out/s1_pipes.jsonl 2>&1
for cfg in "C5_T17 max" "C5_T33 sum" "C5_T33 max" "C5_T17 sum"; do
  set -- $cfg
  timeout 300 python tools/kbench.py $1 $2 20 >> gpurun_out/s1_kbench.jsonl 2>&1
done
for cfg in "C5_T17 max" "C5_T33 sum" "C5_T33 max"; do
  set -- $cfg
  NCU_SKIP=4 timeout 600 bash tools/ncu_one.sh s1_$1_$2 python tools/kbench.py $1 $2 3
done
ls -la gpurun_out
