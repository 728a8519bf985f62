"""K4 pruning statistics on a BASELINE config (GPU, torch ops on the library's D): how many
foreground centres survive each offset class of the lattice containment test, in K4's order
(stage 1: the 26-neighbourhood; stage 2: |s|^2 = 4 .. 12).  Analysis only: the M(D, s) table is
rebuilt here from its definition (prefix maxima over the lattice points sorted by |u|^2).
usage: python tools/prune_stats.py [--config 4]"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
import synth  # noqa: E402

CLASSES = [(1, 0, 0), (1, 1, 0), (1, 1, 1), (2, 0, 0), (2, 1, 0), (2, 1, 1), (2, 2, 0), (2, 2, 1), (3, 0, 0),
           (3, 1, 0), (3, 1, 1), (2, 2, 2)]


def mtable(dmax: int, s) -> np.ndarray:
    r = int(np.ceil(np.sqrt(dmax))) + 1
    ax = np.arange(-r, r + 1)
    u = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    r2 = (u * u).sum(1)
    val = ((u - np.array(s)) ** 2).sum(1)
    o = np.argsort(r2, kind="stable")
    r2, val = r2[o], np.maximum.accumulate(val[o])
    D = np.arange(dmax + 1)
    idx = np.searchsorted(r2, D - 1, side="right") - 1  # last point with |u|^2 <= D-1
    m = np.where(idx >= 0, val[np.maximum(idx, 0)], 0)
    m[0] = 0
    return m


def offsets(cls):
    out = set()
    for p in itertools.permutations(cls):
        for sg in itertools.product((-1, 1), repeat=3):
            out.add(tuple(a * b for a, b in zip(p, sg)))
    return sorted(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    lab, info = synth.make_config(a.config)
    t = torch.from_numpy(lab).cuda()
    D = F.edt_sq(t).to(torch.int64)
    del t
    dmax = int(D.max())
    Dp = torch.nn.functional.pad(D, (3, 3, 3, 3, 3, 3))
    Z, Y, X = D.shape
    fg = D > 0
    alive = fg.clone()
    res = {"config": a.config, "n_fg": int(fg.sum()), "dmax": dmax, "classes": []}
    for ci, cls in enumerate(CLASSES):
        m = torch.from_numpy(mtable(dmax, cls)).cuda()
        thr = m[D]
        mx = torch.zeros_like(D)
        for dz, dy, dx in offsets(cls):
            mx = torch.maximum(mx, Dp[3 + dz:3 + dz + Z, 3 + dy:3 + dy + Y, 3 + dx:3 + dx + X])
        alone = fg & (mx > thr)  # dropped by this class alone
        alive &= ~(mx > thr)
        res["classes"].append({"class": cls, "n_offsets": len(offsets(cls)), "alive_after": int(alive.sum()),
                               "dropped_alone": int(alone.sum())})
        print(res["classes"][-1], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
