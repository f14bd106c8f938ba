# sequential-schedule chain kernel lane width A/B (sum, Ms >= 128)
out=gpurun_out/ab_chain_vl.txt
rm -f $out
for c in "C4 sum" "C5_T9 sum" "C5_T5 sum"; do
  for v in 8 16; do
    echo "$c VL=$v $(SBP_CHAIN_VL=$v python tools/kbench_seq.py $c 5)" >> $out
  done
  for v in 8 16; do
    echo "$c VL=$v hash $(SBP_CHAIN_VL=$v python tools/lib_hash.py ${c% *} ${c#* } 2 96 160 sequential | cut -c1-200)" >> $out
  done
done
cat $out
