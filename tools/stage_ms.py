"""Per-stage device time (library CUDA events, fastrs_profile) of the S&R call on one config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 1
lab, info = synth.make_config(cfg, batch=32) if cfg == 5 else synth.make_config(cfg)
nd = 2 if cfg in (1, 5) else 3
t = torch.from_numpy(lab).cuda()
ml = info["max_label"]
for _ in range(2):
    F.sphericity_roundness(t, max_label=ml, ndim=nd, flags=flags)
F.profile(True)
for _ in range(5):
    F.sphericity_roundness(t, max_label=ml, ndim=nd, flags=flags)
st, n = F.profile_read()
F.profile(False)
print(f"C{cfg} flags={flags}", {k: round(v / n, 3) for k, v in st.items()}, "total", round(sum(st.values()) / n, 3))
