"""Per-SASS-instruction summary of one kernel of an ncu report (instructions executed, stall samples).
usage: python tools/ncu_sass.py REPORT.ncu-rep KERNEL_REGEX [TOP] [--order]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
order = "--order" in sys.argv
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
for r in rows:
    if len(r) > 2 and r[0] == "Address":
        if hdr is not None:
            break  # first kernel instance only
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        recs.append((d["Address"], d["Source"].strip(), float(d["Instructions Executed"] or 0),
                     float(d["Warp Stall Sampling (All Samples)"] or 0), float(d["Avg. Threads Executed"] or 0)))
    except ValueError:
        pass
ti = sum(x[2] for x in recs) or 1
ts = sum(x[3] for x in recs) or 1
print(f"total warp-instructions {ti:.4e}, stall samples {ts:.0f}")
sel = recs if order else sorted(recs, key=lambda x: -x[2])[:top]
for a, s, i, st, th in sel:
    if order and i / ti < 0.002:
        continue
    print(f"{a[-5:]} {100*i/ti:5.2f}% stall {100*st/ts:5.2f}% thr {th:4.1f}  {s[:70]}")
