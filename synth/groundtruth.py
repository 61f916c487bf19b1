"""Exact brute-force ground truth and recall (Recall@k = |ANN_k ∩ NN_k| / k).

NN_k is the exact top-k by tau_h with ties by id (SURVEY AMB-22):
squared L2, or negated inner product for "ip".  Distances are evaluated in float64.
This is evaluation, not the method: it never runs SQ codes or the graph.
"""
from __future__ import annotations

import numpy as np


def _gt_numpy(x: np.ndarray, q: np.ndarray, k: int, metric: str, block: int = 256) -> np.ndarray:
    x64 = x.astype(np.float64)
    q64 = q.astype(np.float64)
    n = x.shape[0]
    out = np.empty((q.shape[0], k), dtype=np.int32)
    ids = np.arange(n)
    for lo in range(0, q.shape[0], block):
        hi = min(q.shape[0], lo + block)
        if metric == "l2":
            d = ((x64 ** 2).sum(1)[None, :] + (q64[lo:hi] ** 2).sum(1)[:, None]
                 - 2.0 * (q64[lo:hi] @ x64.T))
        else:
            d = -(q64[lo:hi] @ x64.T)
        m = min(n, k + 32)
        part = np.argpartition(d, m - 1, axis=1)[:, :m] if m < n else np.tile(ids, (hi - lo, 1))
        for r in range(hi - lo):
            c = part[r]
            if metric == "l2":
                dd = ((x64[c] - q64[lo + r]) ** 2).sum(1)
            else:
                dd = -(x64[c] @ q64[lo + r])
            out[lo + r] = c[np.lexsort((c, dd))][:k]
    return out


def _gt_torch(x, q, k: int, metric: str, block: int = 1024):
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        n = x.shape[0]
        n2 = (x * x).sum(1)
        out = torch.empty((q.shape[0], k), dtype=torch.int64, device=x.device)
        m = min(n, k + 32)
        for lo in range(0, q.shape[0], block):
            hi = min(q.shape[0], lo + block)
            if metric == "l2":
                d = n2[None, :] - 2.0 * (q[lo:hi] @ x.T)
            else:
                d = -(q[lo:hi] @ x.T)
            _, c = torch.topk(d, m, dim=1, largest=False, sorted=False)
            xq = q[lo:hi].double()
            xc = x[c].double()
            if metric == "l2":
                dd = ((xc - xq[:, None, :]) ** 2).sum(-1)
            else:
                dd = -(xc * xq[:, None, :]).sum(-1)
            c_sorted, perm = torch.sort(c, dim=1, stable=True)
            dd = torch.gather(dd, 1, perm)
            _, perm2 = torch.sort(dd, dim=1, stable=True)
            out[lo:hi] = torch.gather(c_sorted, 1, perm2)[:, :k]
        return out
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def ground_truth(x, q, k: int, metric: str = "l2", device: str = "cpu") -> np.ndarray:
    if device == "cpu":
        return _gt_numpy(np.asarray(x), np.asarray(q), k, metric)
    import torch
    xt = torch.as_tensor(np.asarray(x), device=device)
    qt = torch.as_tensor(np.asarray(q), device=device)
    return _gt_torch(xt, qt, k, metric).int().cpu().numpy()


def recall_at_k(found: np.ndarray, gt: np.ndarray, k: int) -> float:
    """Mean over queries of |found[:k] ∩ gt[:k]| / k."""
    found = np.asarray(found)[:, :k]
    gt = np.asarray(gt)[:, :k]
    hits = 0
    for f, g in zip(found, gt):
        hits += len(set(int(v) for v in f if v >= 0) & set(int(v) for v in g))
    return hits / (k * gt.shape[0])
