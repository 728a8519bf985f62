"""Per-kernel summary of an ncu --set full report (raw page) as JSON + a text table.
usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [--title TEXT]
The JSON is what bench.py reads for roofline.traffic (DRAM bytes per launch of a kernel)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

rep, out = sys.argv[1], sys.argv[2]
title = sys.argv[sys.argv.index("--title") + 1] if "--title" in sys.argv else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3}


def val(d, name):
    v = d[col[name]].replace(",", "")
    try:
        return float(v) * scale.get(units[col[name]], 1.0)
    except ValueError:
        return None


agg = defaultdict(list)
for d in data:
    k = d[col["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
    k = k.replace("unnamed>::", "")
    agg[k].append({
        "time_ms": val(d, "gpu__time_duration.sum"),
        "dram_read_bytes": val(d, "dram__bytes_read.sum"),
        "dram_write_bytes": val(d, "dram__bytes_write.sum"),
        "dram_throughput_pct": val(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_throughput_pct": val(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": val(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "thread_inst_per_inst": val(d, "smsp__thread_inst_executed_per_inst_executed.ratio"),
        "registers": val(d, "launch__registers_per_thread"),
        "warp_instructions": val(d, "smsp__inst_executed.sum"),
    })
res = {}
ADD = ("time_ms", "dram_read_bytes", "dram_write_bytes", "warp_instructions")
for k, lst in agg.items():
    # the capture holds one call (cudaProfilerStart/Stop in tools/prof_run.py): additive metrics are
    # summed over the call's launches of the kernel (K5 runs in waves), the rest time-weighted
    tw = sum(x["time_ms"] or 0 for x in lst) or 1.0
    r = {}
    for m in lst[0]:
        v = [x for x in lst if x[m] is not None]
        if m in ADD:
            r[m] = sum(x[m] for x in v)
        elif m == "registers":
            r[m] = max((x[m] for x in v), default=None)
        else:
            r[m] = sum(x[m] * (x["time_ms"] or 0) for x in v) / tw
    r["launches_captured"] = len(lst)
    r["traffic_bytes_per_launch"] = (r["dram_read_bytes"] or 0) + (r["dram_write_bytes"] or 0)  # per call
    res[k] = r
json.dump({"title": title, "report": rep, "kernels": res}, open(out, "w"), indent=1)
print(f"# {title}")
print(f"{'kernel':28s} {'ms':>8s} {'DRAM GB':>8s} {'DRAM%':>6s} {'SM%':>6s} {'warps%':>7s} {'issue%':>7s} {'thr/inst':>8s} {'winst':>10s}")
for k, r in sorted(res.items(), key=lambda x: -x[1]["time_ms"]):
    print(f"{k[:28]:28s} {r['time_ms']:8.3f} {r['traffic_bytes_per_launch'] / 1e9:8.3f} {r['dram_throughput_pct']:6.1f} "
          f"{r['sm_throughput_pct']:6.1f} {r['warps_active_pct']:7.1f} {r['issue_active_pct']:7.1f} "
          f"{r['thread_inst_per_inst']:8.2f} {r['warp_instructions']:10.3g}")
