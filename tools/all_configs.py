"""Device time per step of the hot path on every BASELINE config (library stage events).
usage: python tools/all_configs.py [--c5-batch 32]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--c5-batch", type=int, default=32)
p.add_argument("--iters", type=int, default=3)
a = p.parse_args()
for cfg in (1, 2, 3, 5, 4):
    lab, info = synth.make_config(cfg, batch=a.c5_batch) if cfg == 5 else synth.make_config(cfg)
    ndim = 2 if cfg in (1, 5) else 3
    t = torch.from_numpy(lab).cuda()
    ml = info["max_label"]
    F.sphericity_roundness(t, max_label=ml, ndim=ndim)
    torch.cuda.synchronize()
    F.profile(True)
    for _ in range(a.iters):
        F.sphericity_roundness(t, max_label=ml, ndim=ndim)
    ms, calls = F.profile_read()
    F.profile(False)
    tot = sum(ms.values()) / calls
    d = F.diagnostics(F.last_workspace())
    print(json.dumps({"config": f"C{cfg}", "elements": int(lab.size), "fill": round(info["fill"], 4),
                      "ms_per_call": round(tot, 3), "Gelem_per_s": round(lab.size / tot / 1e6, 2),
                      "stages_ms": {k: round(v / calls, 3) for k, v in ms.items() if v > 0},
                      "dmax": d["dmax"], "n_kept": d["n_kept"], "fallback_groups": d["n_fallback"]}), flush=True)
    del t
    torch.cuda.empty_cache()
