"""Dev tool: search-kernel launch time under different L2 conditions (C1, ef 136)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402

EF = int(sys.argv[1]) if len(sys.argv) > 1 else 136
cfg = synth.get_config("C1")
w = synth.make_workload(cfg, device="cuda", gt=False)
dev = torch.device("cuda:0")
xt = torch.from_numpy(w["x"]).to(dev)
codes, lo, hi = vsag.encode_sq(xt, 8)
ix = vsag.Index(xt, codes, lo, hi, 8, torch.from_numpy(w["entry"]).to(dev), adj=torch.from_numpy(w["graph"]).to(dev))
qs = [torch.from_numpy(w["q"]).to(dev)] + [torch.from_numpy(synth.generate_queries(cfg, cfg.nq, seed=100 + i)).to(dev)
                                          for i in range(1, 4)]
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)


def run(name, flush_each, rotate, n=20):
    ts = []
    for i in range(n):
        if flush_each:
            flush.zero_()
        _, _, tm = ix.search(qs[i % 4] if rotate else qs[0], 10, EF, EF, timing=True)
        ts.append(tm["ms_search"])
    print(f"{name:28s} median {np.median(ts):.4f} ms  min {min(ts):.4f}  max {max(ts):.4f}", flush=True)


for _ in range(5):
    ix.search(qs[0], 10, EF, EF)
for rep in range(2):
    run("flushed, set 0", True, False)
    run("unflushed, set 0 (warm)", False, False)
    run("unflushed, rotating sets", False, True)
    run("flushed, rotating sets", True, True)
