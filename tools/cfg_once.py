"""Dev tool: one config (C2/C3/C4) at one ef, a few search calls (for ncu instruction counts / A/B):
python tools/cfg_once.py C3 256 [visited_kind] [visited_slots]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402

name, ef = sys.argv[1], int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "auto"
slots = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = synth.get_config(name)
if name == "C4":
    cfg = cfg.scaled(n=int(os.environ.get("C4N", "2000000")))
w = synth.make_workload(cfg, device="cuda", gt=False)
dev = torch.device("cuda:0")
xt = torch.from_numpy(w["x"]).to(dev)
codes, lo, hi = vsag.encode_sq(xt, cfg.bits)
ix = vsag.Index(xt, codes, lo, hi, cfg.bits, torch.from_numpy(w["entry"]).to(dev), adj=torch.from_numpy(w["graph"]).to(dev))
q = torch.from_numpy(w["q"]).to(dev)
ts = []
for _ in range(4):
    _, _, tm = ix.search(q, cfg.k, ef, cfg.rerank_n(ef), cfg.metric, timing=True, visited_kind=kind, visited_slots=slots)
    ts.append(tm["ms_search"])
_, _, tr = ix.search(q, cfg.k, ef, cfg.rerank_n(ef), cfg.metric, trace=True, visited_kind=kind, visited_slots=slots)
torch.cuda.synchronize()
print(f"{name} ef={ef} kind={kind} slots={tm['visited_slots']} search_ms={min(ts):.3f} step_ms={tm['ms_total']:.3f} "
      f"blocks={tm['blocks']} n_lp={float(tr['n_lp'].float().mean()):.1f} n_miss={float(tr['n_miss'].float().mean()):.1f}")
