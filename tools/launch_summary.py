"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.
usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
            scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(d.get("Metric Unit", "ns"), 1e-6)
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total ms':>10} {'ms/launch':>10} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1]:10.2f} {v[1] / v[0]:10.3f} {100 * v[1] / tot:5.1f}%  {k}")
