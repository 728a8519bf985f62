"""NEXT-2 sweep (Fig. 6a): S_LT (the hot path) against the S_MC baseline
(fastrs_mc_measure) per object on the synthetic configs, objects with V >= 1000 as in the
paper; plus the Eq. 3 width/length sphericity of the 2D configs.  Prints one JSON line per
config (Pearson r, mean |S_LT - S_MC|, counts, and the time of each GPU call)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
from paper_2504_05808_b200 import fastrs  # noqa: E402
import synth  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for cfg in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5]:
    lab, info = synth.make_config(cfg, batch=8) if cfg == 5 else synth.make_config(cfg)
    nd = 2 if cfg in (1, 5) else 3
    ml = info["max_label"]
    t = torch.from_numpy(lab).cuda()
    F.sphericity_roundness(t, max_label=ml, ndim=nd)  # warm
    fastrs.mc_measure(t, ml, ndim=nd)
    lt, ms_lt = timed(lambda: F.sphericity_roundness(t, max_label=ml, ndim=nd, stats=True))
    mc, ms_mc = timed(lambda: fastrs.mc_measure(t, ml, ndim=nd))
    s_lt, s_mc = lt["sphericity"].cpu().numpy(), mc["sphericity_mc"].cpu().numpy()
    vol = lt["volume"].cpu().numpy()
    keep = (vol >= 1000) & ~np.isnan(s_lt) & ~np.isnan(s_mc)
    line = {"config": f"C{cfg}", "objects": int(keep.sum()), "min_volume": 1000,
            "pearson_r": float(np.corrcoef(s_lt[keep], s_mc[keep])[0, 1]) if keep.sum() > 2 else None,
            "mean_abs_diff": float(np.mean(np.abs(s_lt[keep] - s_mc[keep]))) if keep.any() else None,
            "mean_S_LT": float(np.mean(s_lt[keep])) if keep.any() else None,
            "mean_S_MC": float(np.mean(s_mc[keep])) if keep.any() else None,
            "ms_sphericity_roundness": ms_lt, "ms_mc_measure": ms_mc}
    if nd == 2:
        wl, ms_wl = timed(lambda: fastrs.sphericity_wl(t, ml))
        swl = wl["swl"].cpu().numpy()
        k2 = keep & ~np.isnan(swl)
        line.update(mean_S_WL=float(np.mean(swl[k2])) if k2.any() else None, ms_sphericity_wl=ms_wl,
                    pearson_r_lt_wl=float(np.corrcoef(s_lt[k2], swl[k2])[0, 1]) if k2.sum() > 2 else None)
    print(json.dumps(line), flush=True)
