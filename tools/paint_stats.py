"""K5b statistics on one config: candidates, balls painted after the screens, balls that covered
cells (fastrs_read_diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
import synth  # noqa: E402

for cfg in [int(a) for a in sys.argv[1:]] or [4]:
    lab, info = synth.make_config(cfg, batch=8) if cfg == 5 else synth.make_config(cfg)
    ndim = 2 if cfg in (1, 5) else 3
    t = torch.from_numpy(lab).cuda()
    F.sphericity_roundness(t, max_label=info["max_label"], ndim=ndim)
    torch.cuda.synchronize()
    d = F.diagnostics(F.last_workspace())
    print(f"C{cfg}", {k: d[k] for k in ("n_fg", "n_kept", "sum_group_list", "n_painted", "n_covering", "n_intervals")})
