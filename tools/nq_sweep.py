"""Dev tool: search-kernel time vs batch size on C1 (tail / wave effects of the persistent grid)."""
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
q = torch.from_numpy(w["q"]).to(dev)
qq = torch.cat([q, q, q], 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for nq in [592, 1184, 2664, 5328, 8000, 10000, 10656, 16000, 21312, 30000]:
    qb = qq[:nq].contiguous()
    for _ in range(2):
        ix.search(qb, 10, EF, EF)
    ts = []
    for _ in range(7):
        flush.zero_()
        _, _, tm = ix.search(qb, 10, EF, EF, timing=True)
        ts.append(tm["ms_search"])
    t = float(np.median(ts))
    print(f"nq={nq:6d} search_ms={t:7.3f} us/query={1e3 * t / nq:7.4f} qps={nq / t * 1e3 / 1e6:6.2f}M", flush=True)
