# ncu evidence for the fused (temporally blocked) kernel on C4.
export SBP_FUSE=${SBP_FUSE:-2}
NCU_KERNEL=band_fused NCU_SKIP=2 bash tools/ncu_one.sh fused_w python tools/kbench.py C4 sum 4
grep -E "Duration|DRAM Throughput|Issue Slots Busy|Warp Cycles Per Issued|Achieved Occupancy" gpurun_out/details_fused_w.txt
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/raw_fused_w.csv")))
for h, v in zip(rows[0], rows[2]):
    if ("pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")) or h in (
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
            "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct"):
        print(h, v)
PY
