"""Summarise an ncu --csv launch list (time + DRAM bytes per launch):
launch_table.py FILE.csv [--by-kernel]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = {}
for r in rows[1:]:
    d.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
agg = {}
for (i, k), m in sorted(d.items()):
    name = k.split("(")[0].replace("void ", "").split("::")[-1]
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    b = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e9
    if "--by-kernel" in sys.argv:
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1; a[1] += t; a[2] += b
    else:
        print(f"{i:4d} {t:9.1f} us {b:8.3f} GB {b / max(t, 1e-9) * 1e6:7.0f} GB/s  {name}")
if agg:
    tot = sum(a[1] for a in agg.values())
    for name, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{t:9.1f} us {100 * t / tot:5.1f}% {c:4d} launches {b:8.3f} GB {b / max(t, 1e-9) * 1e6:7.0f} GB/s  {name}")
    print(f"total {tot:.1f} us")
