"""Dev tool: QLP early termination (NEXT-4b) on C1 -- recall@10 and cost (hops, re-ranked rows)
of a shrink stump whose threshold is set on a separate tuning query set (seed 101), evaluated
on the config's query set (seed 1), next to plain searches.

python tools/qlp_sweep.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config("C1")
w = synth.make_workload(cfg, device="cuda", gt=True)
dev = torch.device("cuda:0")
xt = torch.from_numpy(w["x"]).to(dev)
codes, lo, hi = vsag.encode_sq(xt, 8)
ix = vsag.Index(xt, codes, lo, hi, 8, torch.from_numpy(w["entry"]).to(dev), adj=torch.from_numpy(w["graph"]).to(dev))
qt = torch.from_numpy(synth.generate_queries(cfg, cfg.nq, seed=101)).to(dev)  # tuning set
qe = torch.from_numpy(w["q"]).to(dev)  # evaluation set (the config's queries)


def run(qd, ef, qlp=None):
    ids, _, tr = ix.search(qd, 10, ef, ef, trace=True, visited_slots=16384, qlp=qlp)
    return ids.cpu().numpy(), {k: v.cpu().numpy() for k, v in tr.items()}


def cost(tr):
    return float(tr["hops"].mean()), float(tr["n_hp"].mean())


for ef in (128, 136, 160, 192, 256):
    ids, tr = run(qe, ef)
    h, r = cost(tr)
    print(f"plain ef={ef:3d}: recall {synth.recall_at_k(ids, w['gt'], 10):.4f} hops {h:6.1f} reranked {r:6.1f}",
          flush=True)
for ef_hi, hop, ef_lo, feat in [(192, 30, 96, 2), (256, 30, 96, 2), (256, 40, 128, 2), (256, 40, 128, 1),
                                (192, 20, 64, 2)]:
    for frac in (0.5, 0.8):
        # threshold: the smallest value at which `frac` of the tuning queries shrink
        lo_t, hi_t = 0, 1 << 26
        while lo_t < hi_t:
            mid = (lo_t + hi_t) // 2
            _, trt = run(qt, ef_hi, (hop, ef_lo, feat, mid))
            if (trt["n_hp"] == ef_lo).mean() >= frac:
                hi_t = mid
            else:
                lo_t = mid + 1
        ids, tr = run(qe, ef_hi, (hop, ef_lo, feat, lo_t))
        h, r = cost(tr)
        shr = float((tr["n_hp"] == ef_lo).mean())
        print(f"qlp ef {ef_hi}->{ef_lo} at hop {hop}, feature {feat}, tuned shrink {frac:.1f} (thr {lo_t}): "
              f"recall {synth.recall_at_k(ids, w['gt'], 10):.4f} hops {h:6.1f} reranked {r:6.1f} shrunk {shr:.2f}",
              flush=True)
