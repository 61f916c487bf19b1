"""Dev tool: search-kernel time vs query order (C1, ef 136): the batch as generated, sorted by
the generator's cluster label (upper bound of cache locality), and sorted by each query's best
entry seed (a key the library could compute from the seed pass)."""
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
q = w["q"]
labels = np.random.default_rng(1).integers(0, cfg.clusters, len(q))  # the generator's first draw
# best entry seed per query (exact code-space L2, fp64 on integer codes)
cq, _, _ = vsag.encode_sq(torch.from_numpy(q).to(dev), 8, lo, hi)
cs = codes[torch.from_numpy(w["entry"]).to(dev).long()].double()
cqd = cq.double()
tau = (cqd * cqd).sum(1, keepdim=True) + (cs * cs).sum(1)[None, :] - 2.0 * cqd @ cs.T
best = tau.argmin(1).cpu().numpy()
orders = {"generated": np.arange(len(q)), "by_cluster": np.argsort(labels, kind="stable"),
          "by_best_seed": np.argsort(best, kind="stable")}
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for rep in range(2):
    for name, perm in orders.items():
        qd = torch.from_numpy(np.ascontiguousarray(q[perm])).to(dev)
        for _ in range(3):
            ix.search(qd, 10, EF, EF)
        ts = []
        for _ in range(20):
            flush.zero_()
            _, _, tm = ix.search(qd, 10, EF, EF, timing=True)
            ts.append(tm["ms_search"])
        print(f"{name:14s} search {np.median(ts):.4f} ms", flush=True)
