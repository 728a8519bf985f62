import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2504_05808_b200 as F
import synth
lab, info = synth.make_config(4)
t = torch.from_numpy(lab).cuda()
F.sphericity_roundness(t, max_label=info["max_label"])
torch.cuda.synchronize()
ws = F.last_workspace()
h = ws[:256].cpu().numpy().view(np.uint64)
print("examined, dcut, taken:", h[15], h[16], h[17], "n_regathers", F.diagnostics(ws).get("n_regathers"))
