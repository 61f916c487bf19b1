"""One-call construction of a config's inputs (base, queries, graph, entry set, ground truth).

Input preparation only (no method arithmetic).  `device="cuda"` builds the graph and
ground truth with torch on the GPU (full-size configs); `device="cpu"` uses numpy.
"""
from __future__ import annotations

import time

import numpy as np

from .configs import Config
from .generators import entry_set, generate_base, generate_queries
from .graph import build_graph
from .groundtruth import ground_truth


def make_workload(cfg: Config, device: str = "cpu", gt: bool = True, csr: bool = False, log=None) -> dict:
    t0 = time.time()
    x = generate_base(cfg)
    q = generate_queries(cfg)
    t1 = time.time()
    g = build_graph(x, cfg.degree, device=device)
    t2 = time.time()
    w = dict(cfg=cfg, x=x, q=q, graph=g, entry=entry_set(cfg.n, cfg.n_seeds))
    if gt:
        w["gt"] = ground_truth(x, q, cfg.k, metric=cfg.metric, device=device)
    t3 = time.time()
    if csr:
        rows = [r[r >= 0] for r in g]
        w["row_ptr"] = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
        w["col"] = np.concatenate(rows).astype(np.int32)
    if log:
        log(f"[workload {cfg.name}] gen {t1 - t0:.1f}s graph {t2 - t1:.1f}s gt {t3 - t2:.1f}s")
    return w
