"""Top CUDA source lines by executed warp instructions of one ncu launch.
usage: python tools/ncu_inst_lines.py REPORT.ncu-rep [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
agg, src, fname, hdr = {}, {}, None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        ci = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(row) <= ci:
        continue
    try:
        ln, v = int(row[0]), int(row[ci] or 0)
    except ValueError:
        continue
    agg[(fname, ln)] = agg.get((fname, ln), 0) + v
    src.setdefault((fname, ln), row[1].strip()[:95])
tot = sum(agg.values()) or 1
print(f"total warp instructions {tot}")
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100.0 * v / tot:5.1f}% {f}:{ln:4d}  {src[(f, ln)]}")
