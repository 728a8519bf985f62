import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2504_05808_b200 import fastrs as F
lab, info = synth.make_config(4)
t = torch.from_numpy(lab).cuda()
F.edt_sq(t); print("C4 edt diag", {k: v for k, v in F.diagnostics(F.last_workspace()).items() if k in ("n_col_slow", "dmax")})


def t_edt(env):
    os.environ.update(env)
    try:
        for _ in range(2):
            F.edt_sq(t)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            F.edt_sq(t)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 5
    finally:
        for k in env:
            del os.environ[k]


print("edt_sq ms: list", t_edt({}), "inline", t_edt({"FASTRS_COL_INLINE": "1"}))
