"""Summarise an ncu report's source page per CUDA source line (instructions, stall samples).
usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr, recs = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or len(r) != len(hdr):
        continue
    def col(name, idx=0):
        js = [i for i, h in enumerate(hdr) if h == name]
        return r[js[idx]]
    try:
        inst = float(col("Instructions Executed"))
        stall = float(col("Warp Stall Sampling (All Samples)"))
    except ValueError:
        continue
    recs.append((cur_file, int(r[0]), r[1].strip(), inst, stall))
ti = sum(x[3] for x in recs) or 1
ts = sum(x[4] for x in recs) or 1
print(f"total warp-instructions {ti:.3e}, stall samples {ts:.0f}")
for f, ln, src, inst, stall in sorted(recs, key=lambda x: -(x[3] / ti + x[4] / ts))[:top]:
    print(f"{f}:{ln:<5d} inst {100*inst/ti:5.1f}%  stall {100*stall/ts:5.1f}%  {src[:90]}")
