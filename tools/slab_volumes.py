"""Exchange volumes of the z-slab path on C4 for P = 2, 4, 8 ranks, from the single-process emulation
(slab.simulate_slabs: the same phases and plans as the NCCL driver; results checked bit-identical to
the single call): bytes each rank receives for the z pass (N8 halo or N1 transpose) and for the
dilation (dense H-slice D halo or the kept-centre halo N4, from the actual packed sizes)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_05808_b200 as F  # noqa: E402
from paper_2504_05808_b200 import slab  # noqa: E402
import synth  # noqa: E402

lab, info = synth.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
t = torch.from_numpy(lab).cuda()
ml = info["max_label"]
want = F.sphericity_roundness(t, max_label=ml)
for P in (2, 4, 8):
    for transpose, lt_halo in ((False, "dense"), (False, "centres"), (True, "centres")):
        r = slab.simulate_slabs(t, P, ml, transpose=transpose, lt_halo=lt_halo)
        same = bool(torch.equal(r["sphericity"].nan_to_num(-1), want["sphericity"].nan_to_num(-1)))
        si = r["slab_info"]
        print(json.dumps({"P": P, "zpass": "N1 transpose" if transpose else "N8 halo", "lt_halo": lt_halo,
                          "h": si["h"], "H": si["H"], "bit_identical": same,
                          "max_recv_MiB_zpass": max(si["recv_bytes_zpass"]) / 2**20,
                          "max_recv_MiB_lt": max(si["recv_bytes_lt"]) / 2**20}), flush=True)
        torch.cuda.empty_cache()
