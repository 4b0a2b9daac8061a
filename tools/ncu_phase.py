"""Executed warp instructions and stall samples of one ncu launch, split by
source-line ranges of tmg_sweep.cu (phase markers given as start lines)."""
import csv
import io
import subprocess
import sys

rep, skip = sys.argv[1], int(sys.argv[2])
marks = [(n, int(l)) for n, l in (a.split("=") for a in sys.argv[3:])]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
inst, samp = {}, {}
fname = hdr = None
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
        ln, v, s = int(row[0]), int(row[ci] or 0), int(row[4] or 0)
    except ValueError:
        continue
    if fname != "tmg_sweep.cu":
        key = "(inlined helpers)"
    else:
        key = "prologue"
        for name, start in marks:
            if ln >= start:
                key = name
    inst[key] = inst.get(key, 0) + v
    samp[key] = samp.get(key, 0) + s
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
for k in inst:
    print(f"{k:20s} inst {100 * inst[k] / ti:5.1f}%   stall samples {100 * samp[k] / ts:5.1f}%")
