"""Hop statistics of search_kernel on C1 (build with -DVSAG_STATS: NVCC_EXTRA=-DVSAG_STATS)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "C1")
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 160
w = synth.make_workload(cfg, device="cuda", gt=False)
dev = torch.device("cuda:0")
xt = torch.from_numpy(w["x"]).to(dev)
codes, lo, hi = vsag.encode_sq(xt, cfg.bits)
ix = vsag.Index(xt, codes, lo, hi, cfg.bits, torch.from_numpy(w["entry"]).to(dev), adj=torch.from_numpy(w["graph"]).to(dev))
qd = torch.from_numpy(w["q"]).to(dev)
f = vsag.lib.vsag_debug_stats
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 64)()
ix.search(qd, cfg.k, ef, cfg.rerank_n(ef), cfg.metric)
torch.cuda.synchronize()
f(buf, 1)
ix.search(qd, cfg.k, ef, cfg.rerank_n(ef), cfg.metric)
torch.cuda.synchronize()
f(buf, 0)
s = np.array(list(buf), dtype=np.float64)
names = {0: "hops", 8: "sum_sel_pos", 2: "sum_m", 3: "hops_m>0", 4: "sum_ns(merged)", 5: "merges", 6: "merges_s>12",
         7: "merge_blocks", 9: "sum_pmin", 10: "sum_pmax", 11: "pending_expansions"}
for i, n in names.items():
    print(f"{n:16s} {s[i]:14.0f}  per hop {s[i] / s[0]:8.3f}")

