"""Key metrics of an ncu --set full report (one kernel), for profiles/ summaries.

usage: python tools/ncu_summary.py REPORT
"""
import csv, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum",
        "lts__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for w in want:
    for i, h in enumerate(hdr):
        if h == w or (w.endswith("pct_of_peak_sustained_active") and h.startswith(w.split(".avg")[0]) and h.endswith("pct_of_peak_sustained_active")):
            print(f"{h}: {vals[i]} {units[i]}")
            break
# tensor pipe metrics present in the report
for i, h in enumerate(hdr):
    if "tensor" in h and "pct" in h and vals[i] not in ("", "0"):
        print(f"{h}: {vals[i]} {units[i]}")
