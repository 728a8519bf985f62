"""Per-stage device times (library CUDA events) of the hot path on one BASELINE config.
usage: python tools/stage_times.py [--config 4] [--iters 3] [--cache /tmp/c4.npy]
Development helper for A/B runs of kernel variants (reads the library's per-stage events)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=4)
p.add_argument("--iters", type=int, default=3)
p.add_argument("--cache", default=None)
a = p.parse_args()
if a.cache and os.path.exists(a.cache):
    lab = np.load(a.cache)
    ml = int(lab.max())
else:
    lab, info = synth.make_config(a.config)
    ml = info["max_label"]
    if a.cache:
        np.save(a.cache, lab)
ndim = 2 if a.config in (1, 5) else 3
t = torch.from_numpy(lab).cuda()
def call():
    try:
        F.sphericity_roundness(t, max_label=ml, ndim=ndim)
    except F.FastrsError as e:  # timing experiments may break invariants on purpose
        print("note:", e, file=sys.stderr)


call()
torch.cuda.synchronize()
F.profile(True)
for _ in range(a.iters):
    call()
ms, calls = F.profile_read()
F.profile(False)
d = F.diagnostics(F.last_workspace())
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("FASTRS_")},
                  "ms": {k: round(v / calls, 3) for k, v in ms.items()}, "total_ms": round(sum(ms.values()) / calls, 3),
                  "diag": d}))
