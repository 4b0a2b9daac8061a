"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"][:80]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}%  n={n:4d}  {k}")
print(f"total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")
