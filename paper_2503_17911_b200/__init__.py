"""paper_2503_17911_b200 -- thin Python binding over libvsag.so (include/vsag.h).

B200-native batched search hot path of VSAG (arXiv 2503.17911): SQ8/SQ4 encode,
deterministic-access greedy search with exact int32 tau_l, fp32 selective re-rank.
This module only marshals arguments (tensor data pointers, the current CUDA
stream) into the C ABI; every step of the path runs in the CUDA kernels of
libvsag.so.  There is no CPU fallback: if the library is missing or cannot be
loaded, importing this package raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# VSAG_LIB_VARIANT=name loads libvsag_<name>.so from this directory (A/B timing of kernel variants)
LIB_PATH = os.path.join(HERE, "libvsag.so" if not os.environ.get("VSAG_LIB_VARIANT") else
                        f"libvsag_{os.environ['VSAG_LIB_VARIANT']}.so")

VSAG_OK, VSAG_ERR_INVALID_ARG, VSAG_ERR_UNSUPPORTED, VSAG_ERR_OVERFLOW, VSAG_ERR_OOM, VSAG_ERR_CUDA = range(6)
METRIC = {"l2": 0, "ip": 1, "l2w": 2}
LAYOUT = {"table": 0, "colocated": 1, 0: 0, 1: 1}
VISITED_KIND = {"auto": 0, "u16": 2, "u32": 3, "bitset": 4, 0: 0, 2: 2, 3: 3, 4: 4}
EXPORTS = ("vsag_code_bytes", "vsag_encode_sq", "vsag_train_sq", "vsag_index_load", "vsag_search_batch",
           "vsag_search_batch_ex",
           "vsag_search_batch_host", "vsag_index_get_info", "vsag_index_set_labels", "vsag_index_set_prs",
           "vsag_index_free", "vsag_last_error")


class VsagError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[vsag status {code}] {msg}")
        self.code = code


class Trace(ctypes.Structure):
    _fields_ = [("max_hops", ctypes.c_int32), ("hops", ctypes.c_void_p), ("expanded", ctypes.c_void_p),
                ("n_lp", ctypes.c_void_p), ("n_hp", ctypes.c_void_p), ("n_miss", ctypes.c_void_p),
                ("pool_ids", ctypes.c_void_p), ("pool_tau", ctypes.c_void_p)]


class SearchParams(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("ef", ctypes.c_int32), ("rerank_n", ctypes.c_int32),
                ("metric", ctypes.c_int32), ("visited_slots", ctypes.c_int32),
                ("warps_per_block", ctypes.c_int32), ("code_lanes", ctypes.c_int32),
                ("max_degree", ctypes.c_int32), ("alpha_s", ctypes.c_float), ("rerank_adaptive", ctypes.c_int32),
                ("qlp_ef_low", ctypes.c_int32), ("qlp_hop", ctypes.c_int32), ("qlp_feature", ctypes.c_int32),
                ("visited_kind", ctypes.c_int32), ("qlp_threshold", ctypes.c_int64),
                ("ev_search_start", ctypes.c_void_p), ("ev_search_stop", ctypes.c_void_p)]


class Timing(ctypes.Structure):
    _fields_ = [("ms_query_prep", ctypes.c_float), ("ms_seed", ctypes.c_float), ("ms_search", ctypes.c_float),
                ("ms_total", ctypes.c_float), ("launches", ctypes.c_int32), ("visited_slots", ctypes.c_int32),
                ("warps_per_block", ctypes.c_int32), ("blocks", ctypes.c_int32),
                ("visited_kind", ctypes.c_int32)]


class IndexInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("code_bytes", ctypes.c_int32), ("code_stride", ctypes.c_int32), ("degree", ctypes.c_int32),
                ("layout", ctypes.c_int32), ("n_entry", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
                ("prs_nodes", ctypes.c_int64), ("prs_bytes", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libvsag.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.vsag_code_bytes.restype = i64
    L.vsag_code_bytes.argtypes = [i32, i32]
    L.vsag_encode_sq.restype = i32
    L.vsag_encode_sq.argtypes = [P, i64, i32, i32, i32, P, P, P, P]
    L.vsag_train_sq.restype = i32
    L.vsag_train_sq.argtypes = [P, i64, i32, ctypes.c_double, P, P, P]
    L.vsag_index_load.restype = i32
    L.vsag_index_load.argtypes = [P, P, P, P, i64, i32, i32, P, P, i32, P, i32, i32, P, ctypes.POINTER(P)]
    L.vsag_search_batch.restype = i32
    L.vsag_search_batch.argtypes = [P, P, i64, i32, i32, i32, i32, P, P, P, P]
    L.vsag_search_batch_ex.restype = i32
    L.vsag_search_batch_ex.argtypes = [P, P, i64, ctypes.POINTER(SearchParams), P, P, P, P, P]
    L.vsag_search_batch_host.restype = i32
    L.vsag_search_batch_host.argtypes = [P, P, i64, ctypes.POINTER(SearchParams), P, P, P]
    L.vsag_index_set_labels.restype = i32
    L.vsag_index_set_labels.argtypes = [P, P, P, P]
    L.vsag_index_set_prs.restype = i32
    L.vsag_index_set_prs.argtypes = [P, ctypes.c_double, P]
    L.vsag_index_get_info.restype = i32
    L.vsag_index_get_info.argtypes = [P, ctypes.POINTER(IndexInfo)]
    L.vsag_index_free.restype = i32
    L.vsag_index_free.argtypes = [P]
    L.vsag_last_error.restype = ctypes.c_char_p
    L.vsag_last_error.argtypes = []
    return L


lib = _load()


def _check(st: int):
    if st != VSAG_OK:
        raise VsagError(st, lib.vsag_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def _out(out, nq: int, k: int, device, host: bool):
    """Caller-given (ids, dists): int32 / float32, shape (nq, k), contiguous, on the index's
    device (or on the host for search_host) -- the kernels write nq * k values through them."""
    if not (isinstance(out, (tuple, list)) and len(out) == 2):
        raise TypeError("out must be a pair (ids, dists)")
    ids, dists = out
    for t, dt, name in ((ids, torch.int32, "out ids"), (dists, torch.float32, "out dists")):
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a tensor")
        if t.dtype != dt:
            raise TypeError(f"{name} must be {dt}, got {t.dtype}")
        if tuple(t.shape) != (nq, k):
            raise ValueError(f"{name} must have shape {(nq, k)}, got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if host and t.is_cuda:
            raise TypeError(f"{name} must be a host tensor")
        if not host and (not t.is_cuda or t.device != device):
            raise TypeError(f"{name} must be a CUDA tensor on {device}")
    return ids, dists


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def code_bytes(d: int, bits: int) -> int:
    return int(lib.vsag_code_bytes(d, bits))


def encode_sq(x: torch.Tensor, bits: int, lower: torch.Tensor | None = None, upper: torch.Tensor | None = None):
    """Rows a1+a2.  Trains per-dimension min/max when lower/upper are None.  Returns (codes, lower, upper)."""
    x = _dev(x, torch.float32, "x")
    n, d = x.shape
    train = lower is None
    if train:
        lower = torch.empty(d, dtype=torch.float32, device=x.device)
        upper = torch.empty(d, dtype=torch.float32, device=x.device)
    else:
        lower, upper = _dev(lower, torch.float32, "lower"), _dev(upper, torch.float32, "upper")
    codes = torch.empty((n, code_bytes(d, bits)), dtype=torch.uint8, device=x.device)
    with torch.cuda.device(x.device):
        _check(lib.vsag_encode_sq(_ptr(x), n, d, bits, int(train), _ptr(lower), _ptr(upper), _ptr(codes),
                                  _stream(x.device)))
    return codes, lower, upper


def train_sq(x: torch.Tensor, quantile: float = 1.0):
    """Row a1 with truncation (App. G; NEXT-1a): per-dimension order statistics at
    floor((1-q)(n-1)) and floor(q(n-1)).  Returns (lower, upper); encode with encode_sq(x, bits, lower, upper)."""
    x = _dev(x, torch.float32, "x")
    n, d = x.shape
    lower = torch.empty(d, dtype=torch.float32, device=x.device)
    upper = torch.empty(d, dtype=torch.float32, device=x.device)
    with torch.cuda.device(x.device):
        _check(lib.vsag_train_sq(_ptr(x), n, d, float(quantile), _ptr(lower), _ptr(upper), _stream(x.device)))
    return lower, upper


class Index:
    """Row a3: an immutable device index.  Borrows base/codes/lower/upper (kept referenced here)."""

    def __init__(self, base, codes, lower, upper, bits: int, entry, adj=None, degree: int | None = None,
                 row_ptr=None, layout="table"):
        self._h = None
        self.base = _dev(base, torch.float32, "base")
        self.codes = _dev(codes, torch.uint8, "codes")
        self.lower = _dev(lower, torch.float32, "lower")
        self.upper = _dev(upper, torch.float32, "upper")
        self.device = self.base.device
        n, d = self.base.shape
        adj = _dev(adj, torch.int32, "adj")
        if row_ptr is not None:
            row_ptr = _dev(row_ptr, torch.int64, "row_ptr")
            if degree is None:
                degree = int((row_ptr[1:] - row_ptr[:-1]).max().item())
        else:
            degree = int(adj.shape[1]) if degree is None else degree
        entry = _dev(entry, torch.int32, "entry")
        self.bits, self.d, self.n, self.degree = bits, d, n, degree
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib.vsag_index_load(_ptr(self.base), _ptr(self.codes), _ptr(self.lower), _ptr(self.upper), n, d,
                                       bits, _ptr(row_ptr), _ptr(adj), degree, _ptr(entry), entry.numel(),
                                       LAYOUT[layout], _stream(self.device), ctypes.byref(h)))
        self._h = h

    def info(self) -> dict:
        inf = IndexInfo()
        _check(lib.vsag_index_get_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in IndexInfo._fields_}

    def set_prs(self, delta: float):
        """NEXT-4: co-locate the neighbour codes of the round(delta * n) highest in-degree nodes."""
        with torch.cuda.device(self.device):
            _check(lib.vsag_index_set_prs(self._h, float(delta), _stream(self.device)))

    def set_labels(self, labels, row_ptr=None):
        """NEXT-2: per-edge labels (Alg. 2) in the adjacency's layout ([n, degree], or CSR columns)."""
        labels = _dev(labels, torch.float32, "labels")
        if row_ptr is not None:
            row_ptr = _dev(row_ptr, torch.int64, "row_ptr")
        with torch.cuda.device(self.device):
            _check(lib.vsag_index_set_labels(self._h, _ptr(row_ptr), _ptr(labels), _stream(self.device)))

    @staticmethod
    def _params(k, ef, rerank_n, metric, visited_slots, warps_per_block, code_lanes=0, max_degree=0, alpha_s=0.0,
                rerank_adaptive=False, qlp=None, visited_kind=0, events=None):
        sp = SearchParams()
        if events is not None:  # (start, stop) torch.cuda.Event, recorded around the search kernel
            for ev in events:
                if ev.cuda_event == 0:  # torch creates the event lazily on its first record
                    ev.record()
            sp.ev_search_start, sp.ev_search_stop = events[0].cuda_event, events[1].cuda_event
        sp.visited_kind = VISITED_KIND[visited_kind]
        sp.rerank_adaptive = int(rerank_adaptive)
        if qlp is not None:  # NEXT-4b: (checkpoint hop, ef_low, feature, threshold)
            sp.qlp_hop, sp.qlp_ef_low, sp.qlp_feature, sp.qlp_threshold = (int(v) for v in qlp)
        sp.k, sp.ef, sp.rerank_n, sp.metric = k, ef, rerank_n, METRIC[metric]
        sp.visited_slots, sp.warps_per_block, sp.code_lanes = visited_slots, warps_per_block, code_lanes
        sp.max_degree, sp.alpha_s = max_degree, alpha_s
        return sp

    def search(self, queries, k: int, ef: int, rerank_n: int = 0, metric: str = "l2", trace: bool = False,
               max_hops: int = 0, visited_slots: int = 0, warps_per_block: int = 0, timing: bool = False,
               out=None, code_lanes: int = 0, max_degree: int = 0, alpha_s: float = 0.0,
               rerank_adaptive: bool = False, qlp=None, visited_kind="auto", events=None):
        """Rows a4-a8 on device tensors.  Returns (ids, dists[, trace dict][, timing dict]).
        qlp: optional (hop, ef_low, feature, threshold), QLP early termination (NEXT-4b).
        visited_kind: "auto", "u16", "u32" (shared-memory caches) or "bitset" (exact, device memory).
        events: optional (start, stop) torch.cuda.Event recorded around the search kernel (no sync)."""
        q = _dev(queries, torch.float32, "queries")
        if q.device != self.device or q.dim() != 2 or q.shape[1] != self.d:
            raise ValueError(f"queries must be [nq, {self.d}] on {self.device}")
        nq = q.shape[0]
        dev = self.device
        if out is None:
            ids = torch.empty((nq, max(k, 0)), dtype=torch.int32, device=dev)  # k < 1: the ABI rejects it
            dists = torch.empty((nq, max(k, 0)), dtype=torch.float32, device=dev)
        else:
            ids, dists = _out(out, nq, k, dev, host=False)
        sp = self._params(k, ef, rerank_n, metric, visited_slots, warps_per_block, code_lanes, max_degree, alpha_s,
                          rerank_adaptive, qlp, visited_kind, events)
        tr = None
        tdict = {}
        if trace:
            L = max(ef, rerank_n or ef)
            z = lambda *s: torch.empty(s, dtype=torch.int32, device=dev)  # noqa: E731
            tdict = dict(hops=z(nq), n_lp=z(nq), n_hp=z(nq), n_miss=z(nq), pool_ids=z(nq, L), pool_tau=z(nq, L))
            if max_hops > 0:
                tdict["expanded"] = z(nq, max_hops)
            tr = Trace(max_hops, *[_ptr(tdict.get(f)) for f in ("hops", "expanded", "n_lp", "n_hp", "n_miss",
                                                                  "pool_ids", "pool_tau")])
        tm = Timing() if timing else None
        with torch.cuda.device(dev):
            _check(lib.vsag_search_batch_ex(self._h, _ptr(q), nq, ctypes.byref(sp), _ptr(ids), _ptr(dists),
                                            ctypes.byref(tr) if tr is not None else None,
                                            ctypes.byref(tm) if tm is not None else None, _stream(dev)))
        res = [ids, dists]
        if trace:
            res.append(tdict)
        if timing:
            res.append({f: getattr(tm, f) for f, _ in Timing._fields_})
        return tuple(res)

    def search_host(self, queries, k: int, ef: int, rerank_n: int = 0, metric: str = "l2",
                    visited_slots: int = 0, warps_per_block: int = 0, out=None, code_lanes: int = 0,
                    max_degree: int = 0, alpha_s: float = 0.0, rerank_adaptive: bool = False, qlp=None,
                    visited_kind="auto"):
        """End-to-end form: host (ideally pinned) float32 queries in, host ids/dists out."""
        q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(queries)
        if q.is_cuda or q.dtype != torch.float32:
            raise TypeError("queries must be a host float32 tensor/array")
        q = q.contiguous()
        if q.dim() != 2 or q.shape[1] != self.d:
            raise ValueError(f"queries must be [nq, {self.d}]")
        nq = q.shape[0]
        if out is None:
            ids = torch.empty((nq, max(k, 0)), dtype=torch.int32, pin_memory=True)
            dists = torch.empty((nq, max(k, 0)), dtype=torch.float32, pin_memory=True)
        else:
            ids, dists = _out(out, nq, k, None, host=True)
        sp = self._params(k, ef, rerank_n, metric, visited_slots, warps_per_block, code_lanes, max_degree, alpha_s,
                          rerank_adaptive, qlp, visited_kind)
        with torch.cuda.device(self.device):
            _check(lib.vsag_search_batch_host(self._h, _ptr(q), nq, ctypes.byref(sp), _ptr(ids), _ptr(dists),
                                              _stream(self.device)))
        return ids, dists

    def close(self):
        if self._h is not None:
            _check(lib.vsag_index_free(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
