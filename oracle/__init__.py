"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper over liboracle.so (oracle.cpp: a plain single-threaded CPU
transcription of the VSAG hot path, arXiv 2503.17911 Alg. 1 / §5 / App. G).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg and
`--impl reference` arm may import this package.  The product path
(paper_2503_17911_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.cpp")

METRIC = {"l2": 0, "ip": 1, "l2w": 2}
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain g++, -O2, no FMA contraction, no fast-math)."""
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        return LIB_PATH
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-pthread", "-o", LIB_PATH + ".tmp", SRC]
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        L.oracle_code_bytes.restype = i64
        L.oracle_code_bytes.argtypes = [i32, i32]
        L.oracle_train_sq.restype = i32
        L.oracle_train_sq.argtypes = [P, i64, i32, P, P]
        L.oracle_train_sq_quantile.restype = i32
        L.oracle_train_sq_quantile.argtypes = [P, i64, i32, ctypes.c_double, P, P]
        L.oracle_l2w_weights.restype = i32
        L.oracle_l2w_weights.argtypes = [P, P, i32, i32, P]
        L.oracle_encode_sq.restype = i32
        L.oracle_encode_sq.argtypes = [P, i64, i32, i32, P, P, P]
        L.oracle_ip_weights.restype = i32
        L.oracle_ip_weights.argtypes = [P, i32, P, P, P]
        L.oracle_tau_l.restype = i32
        L.oracle_tau_l.argtypes = [P, P, i32, i32, P, P, i32, P]
        L.oracle_tau_h.restype = ctypes.c_float
        L.oracle_tau_h.argtypes = [P, P, i32, i32]
        L.oracle_search_batch_labels.restype = i32
        L.oracle_search_batch_labels.argtypes = [P, P, P, P, i64, i32, i32, P, P, i32, P, i32, P, i64, i32, i32,
                                                 i32, i32, P, i32, ctypes.c_float, i32, P, P, P, P, P, P, i32, P, P,
                                                 i32]
        L.oracle_search_batch_qlp.restype = i32
        L.oracle_search_batch_qlp.argtypes = [P, P, P, P, i64, i32, i32, P, P, i32, P, i32, P, i64, i32, i32,
                                              i32, i32, P, i32, ctypes.c_float, i32, i32, i32, i32, i64,
                                              P, P, P, P, P, P, i32, P, P, i32]
        L.oracle_rerank_lower_bound.restype = ctypes.c_double
        L.oracle_rerank_lower_bound.argtypes = [i64, i32, P, P, i32]
        L.oracle_search_batch.restype = i32
        L.oracle_search_batch.argtypes = [P, P, P, P, i64, i32, i32, P, P, i32, P, i32, P, i64, i32, i32, i32,
                                          i32, P, P, P, P, P, P, i32, P, P, i32]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what} failed with status {code}")
        self.code = code


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def code_bytes(d: int, bits: int) -> int:
    return int(lib().oracle_code_bytes(d, bits))


def train_sq(x):
    x = _f32(x)
    n, d = x.shape
    lo = np.empty(d, np.float32)
    hi = np.empty(d, np.float32)
    st = lib().oracle_train_sq(_p(x), n, d, _p(lo), _p(hi))
    if st:
        raise OracleError(st, "oracle_train_sq")
    return lo, hi


def train_sq_quantile(x, q: float):
    """Truncated SQ range (App. G; NEXT-1a): per-dimension order statistics at floor((1-q)(n-1)), floor(q(n-1))."""
    x = _f32(x)
    n, d = x.shape
    lo = np.empty(d, np.float32)
    hi = np.empty(d, np.float32)
    st = lib().oracle_train_sq_quantile(_p(x), n, d, float(q), _p(lo), _p(hi))
    if st:
        raise OracleError(st, "oracle_train_sq_quantile")
    return lo, hi


def l2w_weights(lower, upper, bits: int):
    """(W, w[d]) of the weighted code-space L2 (NEXT-1b)."""
    lower, upper = _f32(lower), _f32(upper)
    w = np.empty(lower.shape[0], np.int32)
    W = lib().oracle_l2w_weights(_p(lower), _p(upper), lower.shape[0], bits, _p(w))
    return int(W), w


def encode_sq(x, bits: int, lower, upper):
    x = _f32(x)
    n, d = x.shape
    out = np.empty((n, code_bytes(d, bits)), np.uint8)
    st = lib().oracle_encode_sq(_p(x), n, d, bits, _p(_f32(lower)), _p(_f32(upper)), _p(out))
    if st:
        raise OracleError(st, "oracle_encode_sq")
    return out


def ip_weights(q, lower, upper):
    q = _f32(q)
    w = np.empty(q.shape[0], np.int32)
    st = lib().oracle_ip_weights(_p(q), q.shape[0], _p(_f32(lower)), _p(_f32(upper)), _p(w))
    if st:
        raise OracleError(st, "oracle_ip_weights")
    return w


def tau_l(q, code, bits: int, lower, upper, metric: str = "l2") -> int:
    q = _f32(q)
    code = np.ascontiguousarray(code, np.uint8)
    out = np.zeros(1, np.int64)
    st = lib().oracle_tau_l(_p(q), _p(code), q.shape[0], bits, _p(_f32(lower)), _p(_f32(upper)),
                            METRIC[metric], _p(out))
    if st:
        raise OracleError(st, "oracle_tau_l")
    return int(out[0])


def rerank_lower_bound(tau_l: int, d: int, lower, upper, bits: int) -> float:
    """NEXT-3 (R-27): lower bound on tau_h from tau_l (L2, base inside the trained range)."""
    return float(lib().oracle_rerank_lower_bound(int(tau_l), d, _p(_f32(lower)), _p(_f32(upper)), bits))


def tau_h(q, x, metric: str = "l2") -> np.float32:
    q = _f32(q)
    x = _f32(x)
    return np.float32(lib().oracle_tau_h(_p(q), _p(x), q.shape[0], METRIC[metric]))


def search_batch(base, codes, lower, upper, bits: int, adj, entry, queries, k: int, ef: int,
                 rerank_n: int = 0, metric: str = "l2", row_ptr=None, degree: int | None = None,
                 trace: bool = False, max_hops: int = 0, nthreads: int = 1, labels=None, m_s: int = 0,
                 alpha_s: float = 0.0, adaptive: bool = False, qlp=None):
    """Run the oracle over a batch.  Returns dict(ids, dists[, hops, n_lp, n_hp, expanded, pool_ids, pool_tau]).
    qlp: optional (hop, ef_low, feature, threshold) -- QLP early termination (NEXT-4b)."""
    base = _f32(base)
    n, d = base.shape
    codes = np.ascontiguousarray(codes, np.uint8)
    queries = _f32(queries).reshape(-1, d)
    nq = queries.shape[0]
    adj = np.ascontiguousarray(adj, np.int32)
    if row_ptr is not None:
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        degree = int(degree or 0)
    else:
        degree = int(adj.shape[1]) if degree is None else degree
    entry = np.ascontiguousarray(entry, np.int32)
    rr = rerank_n or ef
    cap = max(ef, rr)
    ids = np.empty((nq, k), np.int32)
    dists = np.empty((nq, k), np.float32)
    tr = {}
    if trace:
        tr = dict(hops=np.empty(nq, np.int32), n_lp=np.empty(nq, np.int32), n_hp=np.empty(nq, np.int32),
                  pool_ids=np.empty((nq, cap), np.int32), pool_tau=np.empty((nq, cap), np.int32))
        if max_hops > 0:
            tr["expanded"] = np.empty((nq, max_hops), np.int32)
    labels = None if labels is None else _f32(labels)
    qh, qe, qf, qt = qlp if qlp is not None else (0, 0, 0, 0)
    st = lib().oracle_search_batch_qlp(
        _p(base), _p(codes), _p(_f32(lower)), _p(_f32(upper)), n, d, bits, _p(row_ptr), _p(adj), degree,
        _p(entry), entry.shape[0], _p(queries), nq, k, ef, rerank_n, METRIC[metric], _p(labels), int(m_s),
        float(alpha_s), int(adaptive), int(qh), int(qe), int(qf), int(qt), _p(ids), _p(dists),
        _p(tr.get("hops")), _p(tr.get("n_lp")), _p(tr.get("n_hp")), _p(tr.get("expanded")), max_hops,
        _p(tr.get("pool_ids")), _p(tr.get("pool_tau")), nthreads)
    if st:
        raise OracleError(st, "oracle_search_batch")
    out = dict(ids=ids, dists=dists)
    out.update(tr)
    return out
