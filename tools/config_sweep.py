"""Measurement beyond the bench line: ef sweeps of BASELINE.json configs C2 and C3 at full size
(and C4 at a reduced N), recall@k against exact ground truth, search-step time, QPS.

python tools/config_sweep.py C2 C3 [--c4n 2000000] > profiles/r01_config_sweep.json
Every config is built by synth (seeded, synthetic stand-ins).  C2 is run with
the literal SQ4 code-space L2 and with NEXT-1 (99% truncated range + weighted L2).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def sweep(cfg, w, variants, reps=5):
    dev = torch.device("cuda:0")
    xt = torch.from_numpy(w["x"]).to(dev)
    qd = torch.from_numpy(w["q"]).to(dev)
    out = {}
    for name, (metric, quantile) in variants.items():
        lo, hi = vsag.train_sq(xt, quantile)
        codes, _, _ = vsag.encode_sq(xt, cfg.bits, lo, hi)
        ix = vsag.Index(xt, codes, lo, hi, cfg.bits, torch.from_numpy(w["entry"]).to(dev),
                        adj=torch.from_numpy(w["graph"]).to(dev))
        res = {}
        for ef in cfg.efs:
            rr = cfg.rerank_n(ef)
            ix.search(qd, cfg.k, ef, rr, metric)
            ts = []
            for _ in range(reps):
                ids, _, tm = ix.search(qd, cfg.k, ef, rr, metric, timing=True)
                ts.append(tm["ms_total"])
            _, _, tr = ix.search(qd, cfg.k, ef, rr, metric, trace=True)
            rec = synth.recall_at_k(ids.cpu().numpy(), w["gt"], cfg.k)
            ms = float(np.median(ts))
            res[ef] = dict(recall=round(rec, 4), ms=round(ms, 4), qps=round(len(w["q"]) / ms * 1e3),
                           hops=round(float(tr["hops"].float().mean()), 1),
                           n_lp=round(float(tr["n_lp"].float().mean()), 1))
            log(f"  {cfg.name} {name} ef={ef} {res[ef]}")
        out[name] = res
        ix.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--c4n", type=int, default=2_000_000)
    args = ap.parse_args()
    report = {"gpu": torch.cuda.get_device_name(0)}
    for name in args.configs:
        cfg = synth.get_config(name)
        if name == "C4":
            cfg = cfg.scaled(n=args.c4n)
        t = time.time()
        w = synth.make_workload(cfg, device="cuda", gt=True, log=log)
        log(f"[{cfg.name}] workload {time.time() - t:.0f} s")
        if name == "C2":
            variants = {"sq4_l2": ("l2", 1.0), "sq4_l2w_q99": ("l2w", 0.99)}
        else:
            variants = {f"sq{cfg.bits}_{cfg.metric}": (cfg.metric, 1.0)}
        report[cfg.name] = dict(n=cfg.n, d=cfg.d, nq=cfg.nq, k=cfg.k, degree=cfg.degree, bits=cfg.bits,
                                seeds=cfg.n_seeds, results=sweep(cfg, w, variants))
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
