"""Seeded base/query/entry generators. No method arithmetic here."""
from __future__ import annotations

import numpy as np

from .configs import Config

CHUNK = 1_000_000


def _params(cfg: Config):
    """Cluster parameters, always drawn from seed 0 first (so queries share them)."""
    rng = np.random.default_rng(0)
    if cfg.kind == "gauss10":
        means = rng.uniform(-1.0, 1.0, (cfg.clusters, cfg.d))
        return rng, {"means": means}
    if cfg.kind == "gamma_int":
        mu = rng.gamma(0.35, 30.0, (cfg.clusters, cfg.d))
        return rng, {"mu": mu}
    if cfg.kind == "scaled_mix":
        s = rng.uniform(0.05, 1.0, cfg.d)
        mu = rng.standard_normal((cfg.clusters, cfg.d))
        return rng, {"s": s, "mu": mu}
    if cfg.kind == "sphere":
        m = rng.standard_normal((cfg.clusters, cfg.d))
        m /= np.linalg.norm(m, axis=1, keepdims=True)
        return rng, {"m": m}
    raise ValueError(cfg.kind)


def _rows(cfg: Config, p: dict, rng: np.random.Generator, count: int) -> np.ndarray:
    a = rng.integers(0, cfg.clusters, count)
    if cfg.kind == "gauss10":
        x = p["means"][a] + cfg.sigma * rng.standard_normal((count, cfg.d))
    elif cfg.kind == "gamma_int":
        # Gamma(0.35,30) + Gamma(0.15,30): unclipped marginal is Gamma(0.5,30) per dimension.
        x = np.clip(np.rint(p["mu"][a] + rng.gamma(0.15, 30.0, (count, cfg.d))), 0.0, 255.0)
    elif cfg.kind == "scaled_mix":
        x = (p["mu"][a] + cfg.sigma * rng.standard_normal((count, cfg.d))) * p["s"]
    elif cfg.kind == "sphere":
        x = p["m"][a] + cfg.sigma * rng.standard_normal((count, cfg.d))
        x /= np.linalg.norm(x, axis=1, keepdims=True)
    else:
        raise ValueError(cfg.kind)
    return x.astype(np.float32)


def generate_base(cfg: Config) -> np.ndarray:
    """Base set X[n, d] float32, seed 0, drawn in 1M-row chunks in row order."""
    rng, p = _params(cfg)
    out = np.empty((cfg.n, cfg.d), dtype=np.float32)
    for lo in range(0, cfg.n, CHUNK):
        hi = min(cfg.n, lo + CHUNK)
        out[lo:hi] = _rows(cfg, p, rng, hi - lo)
    return out


def generate_queries(cfg: Config, nq: int | None = None, seed: int = 1) -> np.ndarray:
    """Queries Q[nq, d] float32 from the same mixture, seed 1."""
    _, p = _params(cfg)
    rng = np.random.default_rng(seed)
    return _rows(cfg, p, rng, nq if nq is not None else cfg.nq)


def entry_set(n: int, s: int, seed: int = 2) -> np.ndarray:
    """Entry set I (AMB-11): s distinct seeded-random base ids, sorted, int32."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(s, n), replace=False)).astype(np.int32)
