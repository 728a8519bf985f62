"""Profiling driver: generate one BASELINE config and run the hot path a few times (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=3)
p.add_argument("--iters", type=int, default=2)
p.add_argument("--batch", type=int, default=8)
a = p.parse_args()
lab, info = synth.make_config(a.config, batch=a.batch) if a.config == 5 else synth.make_config(a.config)
ndim = 2 if a.config in (1, 5) else 3
t = torch.from_numpy(lab).cuda()
for _ in range(a.iters):
    r = F.sphericity_roundness(t, max_label=info["max_label"], ndim=ndim)
torch.cuda.synchronize()
F.profile(True)
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off captures exactly this call's kernels
F.sphericity_roundness(t, max_label=info["max_label"], ndim=ndim)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(F.profile_read(), F.diagnostics(F.last_workspace()))
