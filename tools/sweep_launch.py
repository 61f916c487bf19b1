"""Dev tool: time search_kernel launch configurations on one workload (prints a table).

python tools/sweep_launch.py --config C1 --ef 160 [--reps 20]
"""
import argparse
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--ef", type=int, default=160)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--grid", default="lanes=4,8;slots=2048;wpb=4")
    args = ap.parse_args()
    cfg = synth.get_config(args.config)
    w = synth.make_workload(cfg, device="cuda", gt=True)
    dev = torch.device("cuda:0")
    xt = torch.from_numpy(w["x"]).to(dev)
    codes, lo, hi = vsag.encode_sq(xt, cfg.bits)
    ix = vsag.Index(xt, codes, lo, hi, cfg.bits, torch.from_numpy(w["entry"]).to(dev),
                    adj=torch.from_numpy(w["graph"]).to(dev))
    qd = torch.from_numpy(w["q"]).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    grid = dict(kv.split("=") for kv in args.grid.split(";"))
    axes = {k: [int(v) for v in vals.split(",")] for k, vals in grid.items()}
    rr = cfg.rerank_n(args.ef)
    print(f"{'lanes':>5} {'slots':>5} {'wpb':>3} | {'search ms':>9} {'total ms':>8} "
          f"{'recall':>6} {'n_lp':>7} {'blocks':>6}")
    for combo in itertools.product(*axes.values()):
        kw = dict(zip(axes.keys(), combo))
        try:
            opts = dict(code_lanes=kw["lanes"], visited_slots=kw["slots"], warps_per_block=kw["wpb"])
            for _ in range(3):
                ix.search(qd, cfg.k, args.ef, rr, cfg.metric, **opts)
            ts, tt = [], []
            for _ in range(args.reps):
                flush.zero_()
                ids, _, tm = ix.search(qd, cfg.k, args.ef, rr, cfg.metric, timing=True, **opts)
                ts.append(tm["ms_search"])
                tt.append(tm["ms_total"])
            _, _, tr = ix.search(qd, cfg.k, args.ef, rr, cfg.metric, trace=True, **opts)
            rec = synth.recall_at_k(ids.cpu().numpy(), w["gt"], cfg.k)
            print(f"{kw['lanes']:>5} {kw['slots']:>5} {kw['wpb']:>3} | "
                  f"{np.median(ts):9.3f} {np.median(tt):8.3f} {rec:6.4f} {tr['n_lp'].float().mean().item():7.1f} "
                  f"{tm['blocks']:6d}", flush=True)
        except vsag.VsagError as e:
            print(kw, "error", e)


if __name__ == "__main__":
    main()
