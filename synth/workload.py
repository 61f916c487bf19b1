"""One-call construction of a config's inputs (base, queries, graph, entry set, ground truth).

Input preparation only (no method arithmetic).  `device="cuda"` builds the graph and
ground truth with torch on the GPU (full-size configs); `device="cpu"` uses numpy.
"""
from __future__ import annotations

import os
import time

import numpy as np

from .configs import Config
from .generators import entry_set, generate_base, generate_queries
from .graph import build_graph
from .groundtruth import ground_truth


GEN_VERSION = "v1"


def _cache_path(cfg: Config):
    d = os.environ.get("VSAG_CACHE_DIR")
    if not d:
        return None
    key = f"{cfg.name}-{cfg.kind}-{cfg.n}-{cfg.d}-{cfg.nq}-{cfg.degree}-{cfg.n_seeds}-{cfg.clusters}-{GEN_VERSION}"
    return os.path.join(d, key)


def make_workload(cfg: Config, device: str = "cpu", gt: bool = True, csr: bool = False, log=None) -> dict:
    """Inputs of one config.  If $VSAG_CACHE_DIR is set, the (deterministic) arrays are cached
    there as .npy files so repeated processes in one session skip the generation."""
    cp = _cache_path(cfg)
    if cp and os.path.exists(os.path.join(cp, "done")) and (not gt or os.path.exists(os.path.join(cp, "gt.npy"))):
        w = dict(cfg=cfg, **{k: np.load(os.path.join(cp, k + ".npy")) for k in ("x", "q", "graph", "entry")})
        if gt:
            w["gt"] = np.load(os.path.join(cp, "gt.npy"))
        _add_csr(w, csr)
        if log:
            log(f"[workload {cfg.name}] loaded from cache {cp}")
        return w
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
    if cp:
        os.makedirs(cp, exist_ok=True)
        for k in ("x", "q", "graph", "entry", "gt"):
            if k in w:
                np.save(os.path.join(cp, k + ".npy"), w[k])
        open(os.path.join(cp, "done"), "w").close()
    _add_csr(w, csr)
    if log:
        log(f"[workload {cfg.name}] gen {t1 - t0:.1f}s graph {t2 - t1:.1f}s gt {t3 - t2:.1f}s")
    return w


def _add_csr(w: dict, csr: bool):
    if csr:
        rows = [r[r >= 0] for r in w["graph"]]
        w["row_ptr"] = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
        w["col"] = np.concatenate(rows).astype(np.int32)
