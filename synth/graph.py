"""Input preparation: the fixed-degree proximity graph (construction is OUT of scope;
BASELINE.json: "built once by the oracle's deterministic builder (exact 64-NN then
greedy RNG pruning to 32, ties by id)").

Recipe: exact K = 2R nearest candidates per node (self excluded,
ties by id), then the paper's pruning test at alpha = 1 (PAPER.md:544,
"alpha * tau(x_j, x_k) <= T_ij"): candidate j is pruned iff some already-kept k has
d(j, k) <= d(i, j); stop at R kept; then fill to exactly R with the nearest pruned
candidates in (dist, id) order.  Rows are emitted in candidate (dist, id) order.
Squared L2 is used for every config (on the unit-normalised C3/C4 data this is the
same order as inner product).

Two backends with identical rules: numpy float64 (CPU, small n, used by the CPU
tests) and torch on CUDA (fp32 GEMM candidates + fp64 re-sort; full-size configs).
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------------------- numpy
def _knn_numpy(x: np.ndarray, kk: int, block: int = 1024) -> np.ndarray:
    n = x.shape[0]
    x64 = x.astype(np.float64)
    n2 = np.einsum("ij,ij->i", x64, x64)
    out = np.empty((n, kk), dtype=np.int64)
    ids = np.arange(n)
    for lo in range(0, n, block):
        hi = min(n, lo + block)
        d = n2[lo:hi, None] + n2[None, :] - 2.0 * (x64[lo:hi] @ x64.T)
        d[np.arange(hi - lo), np.arange(lo, hi)] = np.inf
        m = min(n - 1, kk + 16)
        part = np.argpartition(d, m - 1, axis=1)[:, :m] if m < n else np.tile(ids, (hi - lo, 1))
        for r in range(hi - lo):
            c = part[r]
            c = c[c != lo + r]
            # exact fp64 distance by direct differences, ties by id
            dd = ((x64[c] - x64[lo + r]) ** 2).sum(1)
            order = np.lexsort((c, dd))
            out[lo + r] = c[order][:kk]
    return out


def _prune_numpy(x: np.ndarray, cand: np.ndarray, r: int, block: int = 512) -> np.ndarray:
    n, kk = cand.shape
    x64 = x.astype(np.float64)
    out = np.empty((n, r), dtype=np.int32)
    for lo in range(0, n, block):
        hi = min(n, lo + block)
        b = hi - lo
        c = cand[lo:hi]
        xc = x64[c]                                            # [B, K, d]
        dic = ((xc - x64[lo:hi, None, :]) ** 2).sum(-1)        # [B, K]
        n2 = (xc * xc).sum(-1)
        dcc = n2[:, :, None] + n2[:, None, :] - 2.0 * np.matmul(xc, xc.transpose(0, 2, 1))  # [B, K, K]
        keep = np.zeros((b, kk), dtype=bool)
        cnt = np.zeros(b, dtype=np.int64)
        for t in range(kk):
            pruned = (keep[:, :t] & (dcc[:, t, :t] <= dic[:, t:t + 1])).any(1) if t else np.zeros(b, bool)
            k_t = (~pruned) & (cnt < r)
            keep[:, t] = k_t
            cnt += k_t
        notk = ~keep
        fill_rank = np.cumsum(notk, 1)
        sel = keep | (notk & (fill_rank <= (r - cnt)[:, None]))
        for i in range(b):
            out[lo + i] = c[i][np.nonzero(sel[i])[0][:r]]
    return out


# ----------------------------------------------------------------------------- torch
def _knn_torch(x, kk: int, block: int = 2048, tf32: bool = False):
    import torch
    n = x.shape[0]
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = tf32
    try:
        n2 = (x * x).sum(1)
        out = torch.empty((n, kk), dtype=torch.int64, device=x.device)
        margin = 16 if not tf32 else 48
        m = min(n - 1, kk + margin)
        # a distance tile of at most ~16 GB (the expression below holds ~3 of them at once)
        block = int(max(64, min(block, 16e9 // (4 * n))))
        for lo in range(0, n, block):
            hi = min(n, lo + block)
            d = n2[lo:hi, None] + n2[None, :] - 2.0 * (x[lo:hi] @ x.T)
            d[torch.arange(hi - lo, device=x.device), torch.arange(lo, hi, device=x.device)] = float("inf")
            _, c = torch.topk(d, m + 1 if m + 1 <= n else n, dim=1, largest=False, sorted=False)
            del d
            rows = torch.arange(lo, hi, device=x.device)[:, None]
            # exact fp64 re-sort of the candidates, ties by id; self removed
            diff = x[c].double() - x[lo:hi, None, :].double()
            dd = (diff * diff).sum(-1)
            dd = torch.where(c == rows, torch.full_like(dd, float("inf")), dd)
            # lexicographic (dist, id): sort by id first, then stable sort by dist
            c_sorted, perm = torch.sort(c, dim=1, stable=True)
            dd = torch.gather(dd, 1, perm)
            _, perm2 = torch.sort(dd, dim=1, stable=True)
            out[lo:hi] = torch.gather(c_sorted, 1, perm2)[:, :kk]
        return out
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _prune_torch(x, cand, r: int, block: int = 8192):
    import torch
    n, kk = cand.shape
    out = torch.empty((n, r), dtype=torch.int32, device=x.device)
    for lo in range(0, n, block):
        hi = min(n, lo + block)
        c = cand[lo:hi]
        xc = x[c].double()                                   # [B, K, d]
        xi = x[lo:hi].double()
        dic = ((xc - xi[:, None, :]) ** 2).sum(-1)           # [B, K]
        n2 = (xc * xc).sum(-1)
        dcc = n2[:, :, None] + n2[:, None, :] - 2.0 * torch.bmm(xc, xc.transpose(1, 2))
        b = hi - lo
        keep = torch.zeros((b, kk), dtype=torch.bool, device=x.device)
        cnt = torch.zeros(b, dtype=torch.int64, device=x.device)
        for t in range(kk):
            if t == 0:
                pruned = torch.zeros(b, dtype=torch.bool, device=x.device)
            else:
                pruned = (keep[:, :t] & (dcc[:, t, :t] <= dic[:, t:t + 1])).any(1)
            k_t = (~pruned) & (cnt < r)
            keep[:, t] = k_t
            cnt += k_t.long()
        # fill to r with the nearest pruned candidates (candidate order)
        notk = ~keep
        fill_rank = torch.cumsum(notk.long(), 1)             # 1-based rank among non-kept
        need = (r - cnt)[:, None]
        sel = keep | (notk & (fill_rank <= need))
        pos = torch.arange(kk, device=x.device).expand(b, kk)
        key = torch.where(sel, pos, pos + kk)
        order = torch.sort(key, dim=1).indices[:, :r]
        out[lo:hi] = torch.gather(c, 1, order).int()
    return out


# ----------------------------------------------------------------------------- API
def knn_candidates(x, kk: int, device: str = "cpu", tf32: bool = False):
    if device == "cpu":
        return _knn_numpy(np.asarray(x), kk)
    import torch
    xt = torch.as_tensor(np.asarray(x), device=device)
    return _knn_torch(xt, kk, tf32=tf32).cpu().numpy()


def rng_prune_fill(x, cand, r: int, device: str = "cpu"):
    if device == "cpu":
        return _prune_numpy(np.asarray(x), np.asarray(cand), r)
    import torch
    xt = torch.as_tensor(np.asarray(x), device=device)
    ct = torch.as_tensor(np.asarray(cand), device=device)
    return _prune_torch(xt, ct, r).cpu().numpy()


def build_graph(x: np.ndarray, r: int, device: str = "cpu", kk: int | None = None,
                tf32: bool | None = None) -> np.ndarray:
    """Fixed-degree [n, r] int32 adjacency (no -1 when n > r; -1 padded otherwise)."""
    n = x.shape[0]
    kk = kk or 2 * r
    kk = min(kk, n - 1)
    if n - 1 < r:
        # degenerate tiny graph: complete graph, padded
        out = np.full((n, r), -1, dtype=np.int32)
        for i in range(n):
            nb = [j for j in range(n) if j != i]
            out[i, : len(nb)] = nb
        return out
    if device == "cpu":
        cand = _knn_numpy(x, kk)
        return _prune_numpy(x, cand, r)
    import torch
    xt = torch.as_tensor(x, device=device)
    if tf32 is None:
        tf32 = n > 2_000_000
    cand = _knn_torch(xt, kk, tf32=tf32)
    g = _prune_torch(xt, cand, r)
    return g.cpu().numpy()


# ----------------------------------------------------------------------------- labelled graph
ALPHAS = (1.0, 1.2, 1.4, 1.6, 1.8, 2.0)


def build_labelled_graph(x: np.ndarray, m_c: int, alphas=ALPHAS, kk: int | None = None):
    """Input preparation for NEXT-2: a graph whose edges carry the paper's labels.

    Prune-based labeling (Alg. 2, with r = 0): the exact kk-NN of each
    node (fp64, ties by id) in ascending distance T_ij (Euclidean); for each pruning rate
    alpha in ascending order, every still unlabelled candidate j is pruned iff some closer
    candidate k with 0 < L_ik <= alpha has alpha * tau(x_j, x_k) <= T_ij; otherwise it gets
    L_ij = alpha; at most m_c labels are given; unlabelled candidates are dropped.  Rows keep
    ascending distance order, padded with -1 (label +inf).  Returns (adj [n, m_c] int32,
    labels [n, m_c] float32).  Construction is out of scope; this only makes test inputs.
    """
    kk = kk or 2 * m_c
    n = x.shape[0]
    x64 = x.astype(np.float64)
    cand = _knn_numpy(x, min(kk, n - 1))
    adj = np.full((n, m_c), -1, np.int32)
    lab = np.full((n, m_c), np.inf, np.float32)
    for i in range(n):
        c = cand[i]
        xc = x64[c]
        t = np.sqrt(((xc - x64[i]) ** 2).sum(1))
        dcc = np.sqrt(((xc[:, None, :] - xc[None, :, :]) ** 2).sum(-1))
        L = np.zeros(len(c))
        count = 0
        for a in alphas:
            if count >= m_c:
                break
            for j in range(len(c)):
                if count >= m_c:
                    break
                if L[j] != 0:
                    continue
                pruned = any(0 < L[k] <= a and a * dcc[j, k] <= t[j] for k in range(j))
                if not pruned:
                    L[j] = a
                    count += 1
        keep = np.nonzero(L > 0)[0][:m_c]
        adj[i, :len(keep)] = c[keep]
        lab[i, :len(keep)] = L[keep]
    return adj, lab
