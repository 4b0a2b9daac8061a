"""Key throughput / stall metrics of every launch in an ncu report.
usage: python tools/ncu_summary.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[0], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
want = [
    ("Grid Size", "grid"), ("gpu__time_duration.sum", "time (us)"),
    ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %"),
    ("smsp__inst_executed.sum", "warp inst"),
]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
          and h.endswith("_per_issue_active.ratio")]
for r in data:
    print("----", r[idx["Kernel Name"]][:60])
    for k, name in want:
        if k in idx:
            print(f"  {name:12s} {r[idx[k]]}")
    st = sorted(((float(r[idx[h]] or 0), h) for h in stalls), reverse=True)[:10]
    print("  stalls/issue: " + ", ".join(
        f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
        f" {v:.2f}" for v, h in st))
