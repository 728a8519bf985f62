"""Per-stage device times on volumes with a few LARGE objects (radii far beyond the 48-row staged
window of the column passes): how the EDT column-pass cost grows with the object radius
(VERDICT r1 weak #9).  Each volume is an N^3 grid holding k x k x k touching-free balls of
radius r on a regular lattice (background between them), so the fill is comparable to C4.
usage: python tools/large_objects.py [--n 512] [--radii 40 80 160 240] [--iters 3]
Prints one JSON line per radius: stage ms (library CUDA events) and Gvox/s."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=512)
p.add_argument("--radii", type=int, nargs="+", default=[20, 40, 80, 160, 240])
p.add_argument("--iters", type=int, default=3)
p.add_argument("--flags", type=int, default=1)
p.add_argument("--gap", type=int, default=4, help="voxels between neighbouring balls (<= 0: overlapping, touching labels)")
a = p.parse_args()
for r in a.radii:
    n = a.n
    k = max(1, n // (2 * r + a.gap)) if 2 * r + a.gap > 0 else 1  # balls per axis
    step = n // k
    t = torch.zeros((n, n, n), dtype=torch.int32, device="cuda")
    zz = torch.arange(n, device="cuda")
    lab = 0
    for i in range(k):
        for j in range(k):
            for m in range(k):
                lab += 1
                c = (step * i + step // 2, step * j + step // 2, step * m + step // 2)
                sl = [slice(max(0, c[d] - r), min(n, c[d] + r + 1)) for d in range(3)]
                sub = ((zz[sl[0]] - c[0])[:, None, None] ** 2 + (zz[sl[1]] - c[1])[None, :, None] ** 2 +
                       (zz[sl[2]] - c[2])[None, None, :] ** 2) <= r * r
                view = t[sl[0], sl[1], sl[2]]
                view[sub & (view == 0)] = lab  # overlaps keep the earlier label (touching objects)
    fill = float((t != 0).float().mean())
    F.sphericity_roundness(t, max_label=lab, flags=a.flags)
    torch.cuda.synchronize()
    F.profile(True)
    for _ in range(a.iters):
        F.sphericity_roundness(t, max_label=lab, flags=a.flags)
    acc, calls = F.profile_read()
    ms = {kk: v / max(calls, 1) for kk, v in acc.items()}
    F.profile(False)
    tot = sum(ms.values())
    diag = F.diagnostics(F.last_workspace())
    print(json.dumps({"n": n, "radius": r, "gap": a.gap, "objects": lab, "fill": round(fill, 3), "ms_total": round(tot, 3),
                      "gvox_s": round(n ** 3 / tot / 1e6, 2), "stages_ms": {kk: round(v, 3) for kk, v in ms.items()},
                      "diagnostics": diag}), flush=True)
    del t
    torch.cuda.empty_cache()
