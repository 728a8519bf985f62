"""Object-count scaling benchmark (the paper's speed experiment, PAPER.md:225-230,357,
Fig. 9c): a synthetic 400^3 volume with 15 503 objects of 27 .. ~130 000 voxels (synth.make_count_volume, the
stand-in for the paper's uCT scan), 10 log-spaced object counts 1 .. 2000, 40 draws without replacement per count;
the labels not drawn are set to 0 and the unchanged hot path runs on the volume.

Per count: device time of fastrs_sphericity_roundness (CUDA events on the call stream, labels resident, median and
min over the draws) and, for counts <= 162 on the first draws, the CPU oracle's time on the same masked volume and
the largest relative difference GPU vs oracle (sphericity, roundness of the drawn labels).  Masking runs in torch
(plumbing) outside the timed region.
usage: python tools/count_scaling.py [--draws 40] [--oracle-draws 2] > profiles/r01_count_scaling.jsonl"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2504_05808_b200 as F  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--draws", type=int, default=40)
p.add_argument("--oracle-draws", type=int, default=2)
p.add_argument("--oracle-max-count", type=int, default=162)
a = p.parse_args()

lab, info = synth.make_count_volume()
ml = info["max_label"]
present = np.unique(lab)
present = present[present > 0]
dev = torch.device("cuda:0")
t = torch.from_numpy(lab).to(dev)
ws = F.workspace(F.workspace_bytes(t.shape, 3, ml), dev)
out = {}
stream = torch.cuda.current_stream(dev)
for _ in range(3):  # warm-up on the full volume
    F.sphericity_roundness(t, max_label=ml, ws=ws, out=out)
torch.cuda.synchronize()
full_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
full_ev[0].record(stream)
F.sphericity_roundness(t, max_label=ml, ws=ws, out=out)
full_ev[1].record(stream)
torch.cuda.synchronize()
print(json.dumps({"volume": "count-volume 400^3", "objects": int(present.size), "fill": info["fill"],
                  "sha256": info["sha256"], "all_objects_ms": round(full_ev[0].elapsed_time(full_ev[1]), 4)}),
      flush=True)

counts = sorted(set(int(round(x)) for x in np.logspace(0, np.log10(2000), 10)))
rng = np.random.default_rng(9)
cores = len(os.sched_getaffinity(0))
for n in counts:
    ms, ora_s, worst = [], [], 0.0
    for d in range(a.draws):
        sel = np.sort(rng.choice(present, n, replace=False))
        sel_t = torch.from_numpy(sel.astype(np.int32)).to(dev)
        sub = torch.where(torch.isin(t, sel_t), t, torch.zeros_like(t))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = F.sphericity_roundness(sub, max_label=ml, ws=ws, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        if n <= a.oracle_max_count and d < a.oracle_draws:
            sub_np = sub.cpu().numpy()
            mask = np.zeros(ml, np.uint8)
            mask[sel - 1] = 1
            t0 = time.perf_counter()
            want = oracle.sphericity_roundness(sub_np, max_label=ml, label_mask=mask, nthreads=cores)
            ora_s.append(time.perf_counter() - t0)
            for k in ("sphericity", "roundness"):
                g = res[k].cpu().numpy()[sel - 1]
                w = want[k][sel - 1]
                worst = max(worst, float(np.max(np.abs(g - w) / np.abs(w))))
    rec = {"objects": n, "draws": a.draws, "gpu_ms_median": round(float(np.median(ms)), 4),
           "gpu_ms_min": round(float(np.min(ms)), 4), "gvox_per_s_median": round(64e6 / np.median(ms) / 1e6, 2)}
    if ora_s:
        rec.update(oracle_s_median=round(float(np.median(ora_s)), 4), oracle_cores=cores,
                   max_rel_diff_vs_oracle=worst)
    print(json.dumps(rec), flush=True)
