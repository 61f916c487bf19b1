"""Dev tool: search-kernel time vs the re-rank count R' at a fixed ef on C1 (the re-rank's share)."""
import os
import statistics
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
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for rr in (10, 32, 64, ef):
    for _ in range(3):
        ix.search(q, 10, ef, rr)
    ts = []
    for _ in range(15):
        flush.zero_()
        _, _, tm = ix.search(q, 10, ef, rr, timing=True)
        ts.append(tm["ms_search"])
    print(f"ef={ef} R'={rr}: search {statistics.median(ts):.4f} ms", flush=True)
