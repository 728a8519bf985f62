"""Basic-block summary of one kernel of an ncu report: consecutive SASS instructions with the
same execution count grouped; blocks sorted by their share of executed instructions.
usage: python tools/ncu_blocks.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, recs = None, []
for r in rows:
    if len(r) > 2 and r[0] == "Address":
        if hdr:
            break
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs.append((int(d["Address"], 16), d["Source"].strip(), float(d["Instructions Executed"] or 0),
                     float(d["Warp Stall Sampling (All Samples)"] or 0)))
base = recs[0][0]
ti = sum(x[2] for x in recs) or 1
ts = sum(x[3] for x in recs) or 1
blocks = []
for a, s, i, st in recs:
    if blocks and abs(blocks[-1][2] - i) < 1 and i > 0:
        b = blocks[-1]
        b[1] += 1
        b[3] += i
        b[4] += st
        b[5].append(s)
    else:
        blocks.append([a - base, 1, i, i, st, [s]])
print(f"total warp-instructions {ti:.4e}")
for b in sorted(blocks, key=lambda b: -b[3])[:top]:
    ops = " | ".join((x.split()[1] if x.startswith("@") else x.split()[0]) for x in b[5][:12])
    print(f"{b[0]:#07x} n={b[1]:3d} exec={b[2] / 1e6:8.2f}M inst {100 * b[3] / ti:5.1f}% stall {100 * b[4] / ts:5.1f}%  {ops}")
