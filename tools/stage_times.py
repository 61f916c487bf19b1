"""Dev tool: one C1 search call per library variant, for an ncu launch list (per-kernel times)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402

ef = int(sys.argv[1]) if len(sys.argv) > 1 else 130
cfg = synth.get_config("C1")
w = synth.make_workload(cfg, device="cuda", gt=False)
dev = torch.device("cuda:0")
xt = torch.from_numpy(w["x"]).to(dev)
codes, lo, hi = vsag.encode_sq(xt, 8)
ix = vsag.Index(xt, codes, lo, hi, 8, torch.from_numpy(w["entry"]).to(dev), adj=torch.from_numpy(w["graph"]).to(dev))
q = torch.from_numpy(w["q"]).to(dev)
for _ in range(5):
    ix.search(q, 10, ef, ef)
torch.cuda.synchronize()
print("done")
