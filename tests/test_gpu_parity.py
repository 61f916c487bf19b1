"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): SQ codes and lower/upper byte-identical; per query the
expansion sequence, hop count, final pool ids and int32 tau_l bit-identical; final ids
identical; fp32 re-rank distances within 1e-5 relative (fp64 accumulation on both sides,
R-16, so they are normally bit-identical as well).
"""
import json
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2503_17911_b200 as vsag  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DEV = torch.device("cuda:0")
RTOL = 1e-5


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a)).to(DEV)


def run_gpu(x, q, graph, entry, bits, k, ef, rerank, metric="l2", layout="table", csr=None, max_hops=0,
            visited_slots=16384, lower=None, upper=None, lanes=0, kind="auto"):
    """visited_slots defaults to a table large enough never to forget an id, so n_lp can be
    compared exactly; the forgetful regime (small tables) is tested separately.  `lanes`
    forces the number of lanes that gather one code (the launch shape)."""
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, bits, None if lower is None else _t(lower), None if upper is None else _t(upper))
    if csr is not None:
        ix = vsag.Index(xt, codes, lo, hi, bits, _t(entry), adj=_t(csr[1]), row_ptr=_t(csr[0]),
                        degree=graph.shape[1], layout=layout)
    else:
        ix = vsag.Index(xt, codes, lo, hi, bits, _t(entry), adj=_t(graph), layout=layout)
    ids, dists, tr = ix.search(_t(q), k, ef, rerank, metric, trace=True, max_hops=max_hops,
                               visited_slots=visited_slots, code_lanes=lanes, visited_kind=kind)
    torch.cuda.synchronize()
    out = dict(ids=ids.cpu().numpy(), dists=dists.cpu().numpy(), codes=codes.cpu().numpy(),
               lower=lo.cpu().numpy(), upper=hi.cpu().numpy())
    out.update({key: v.cpu().numpy() for key, v in tr.items()})
    ix.close()
    return out


def run_oracle(orc, x, q, graph, entry, bits, k, ef, rerank, metric="l2", max_hops=0, lower=None, upper=None,
               nthreads=8):
    if lower is None:
        lower, upper = orc.train_sq(x)
    codes = orc.encode_sq(x, bits, lower, upper)
    r = orc.search_batch(x, codes, lower, upper, bits, graph, entry, q, k, ef, rerank, metric, trace=True,
                         max_hops=max_hops, nthreads=nthreads)
    r.update(codes=codes, lower=lower, upper=upper)
    return r


def compare(g, o, exact_nlp=True):
    assert np.array_equal(g["lower"].view(np.uint32), o["lower"].view(np.uint32)), "lower"
    assert np.array_equal(g["upper"].view(np.uint32), o["upper"].view(np.uint32)), "upper"
    assert np.array_equal(g["codes"], o["codes"]), "codes"
    assert np.array_equal(g["hops"], o["hops"]), "hops"
    if "expanded" in o:
        assert np.array_equal(g["expanded"], o["expanded"]), "expansion sequence"
    assert np.array_equal(g["pool_ids"], o["pool_ids"]), "pool ids"
    assert np.array_equal(g["pool_tau"], o["pool_tau"]), "pool tau_l"
    assert np.array_equal(g["n_hp"], o["n_hp"]), "n_hp"
    if exact_nlp:
        assert (g["n_miss"] == 0).all()
        assert np.array_equal(g["n_lp"], o["n_lp"]), "n_lp"
    else:
        assert (g["n_lp"] >= o["n_lp"]).all()
    assert np.array_equal(g["ids"], o["ids"]), "final ids"
    fin = np.isfinite(o["dists"])
    assert np.array_equal(fin, np.isfinite(g["dists"]))
    rel = np.abs(g["dists"][fin].astype(np.float64) - o["dists"][fin]) / np.maximum(np.abs(o["dists"][fin]), 1e-30)
    assert (rel <= RTOL).all(), f"max rel err {rel.max()}"


@pytest.fixture(scope="module")
def c0():
    return synth.make_workload(synth.get_config("C0"), device="cuda", csr=True)


# ----------------------------------------------------------------------------- a1/a2
def test_encode_pins_gpu():
    for line in open(os.path.join(GOLD, "sq_encode_pins.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        b, lo, hi, v, e = line.split()
        codes, _, _ = vsag.encode_sq(_t(np.array([[float(v)]], np.float32)), int(b),
                                     _t(np.array([float(lo)], np.float32)), _t(np.array([float(hi)], np.float32)))
        assert int(codes.cpu()[0, 0]) & (0xFF if b == "8" else 0x0F) == int(e), line


@pytest.mark.parametrize("bits,d,n", [(8, 128, 10000), (4, 128, 10000), (4, 37, 3001), (8, 37, 3001), (4, 960, 2000)])
def test_encode_parity(orc, bits, d, n):
    rng = np.random.default_rng(d + n)
    x = (rng.standard_normal((n, d)) * rng.uniform(0.05, 3, d)).astype(np.float32)
    x[5, 3] = -0.0
    x[:, 1] = 0.25  # constant dimension
    codes, lo, hi = vsag.encode_sq(_t(x), bits)
    olo, ohi = orc.train_sq(x)
    assert np.array_equal(lo.cpu().numpy().view(np.uint32), olo.view(np.uint32))
    assert np.array_equal(hi.cpu().numpy().view(np.uint32), ohi.view(np.uint32))
    assert np.array_equal(codes.cpu().numpy(), orc.encode_sq(x, bits, olo, ohi))
    # queries outside the range are clamped identically (train = 0 path)
    y = (rng.standard_normal((257, d)) * 4).astype(np.float32)
    c2, _, _ = vsag.encode_sq(_t(y), bits, lo, hi)
    assert np.array_equal(c2.cpu().numpy(), orc.encode_sq(y, bits, olo, ohi))


def test_encode_rejects_nonfinite():
    x = torch.zeros((4, 3), device=DEV)
    x[2, 1] = float("nan")
    with pytest.raises(vsag.VsagError) as e:
        vsag.encode_sq(x, 8)
    assert e.value.code == vsag.VSAG_ERR_INVALID_ARG


# ----------------------------------------------------------------------------- W1
@pytest.mark.parametrize("name", ["W1a", "W1b", "W1c"])
@pytest.mark.parametrize("layout", ["table", "colocated"])
def test_w1_gpu(orc, name, layout):
    w = json.load(open(os.path.join(GOLD, "w1_example.json")))
    c = [x for x in w["cases"] if x["name"] == name][0]
    x = np.array(w["codes"], np.float32)
    lo, hi = np.zeros(4, np.float32), np.full(4, 255.0, np.float32)
    q = np.array([w["query"]], np.float32)
    g = run_gpu(x, q, np.array(w["rows"], np.int32), np.array(c["entry"], np.int32), 8, c["k"], c["ef"],
                c["rerank"], layout=layout, max_hops=8, lower=lo, upper=hi, visited_slots=256)
    assert list(g["expanded"][0][: c["hops"]]) == c["trace"]
    assert g["hops"][0] == c["hops"] and g["n_lp"][0] == c["n_lp"]
    assert list(g["pool_ids"][0]) == c["pool_ids"] and list(g["pool_tau"][0]) == c["pool_tau"]
    assert list(g["ids"][0]) == c["ids"] and list(g["dists"][0]) == c["dists"]


# ----------------------------------------------------------------------------- C0 full
@pytest.mark.parametrize("layout", ["table", "colocated"])
@pytest.mark.parametrize("csr", [False, True])
@pytest.mark.parametrize("lanes", [0, 8])
def test_c0_parity(orc, c0, layout, csr, lanes):
    cfg = c0["cfg"]
    args = (c0["x"], c0["q"], c0["graph"], c0["entry"], 8, 10, 64, 64)
    g = run_gpu(*args, layout=layout, csr=(c0["row_ptr"], c0["col"]) if csr else None, max_hops=400, lanes=lanes)
    o = run_oracle(orc, *args, max_hops=400)
    compare(g, o)
    assert synth.recall_at_k(g["ids"], c0["gt"], 10) > 0.95
    assert cfg.name == "C0"


@pytest.mark.parametrize("ef,rerank,k", [(1, 10, 10), (16, 16, 10), (32, 100, 10), (200, 200, 50), (96, 64, 1)])
@pytest.mark.parametrize("lanes", [0, 4, 16, 32])
def test_c0_params_sweep(orc, c0, ef, rerank, k, lanes):
    q = c0["q"][:37]  # ragged batch (not a multiple of the CTA size)
    args = (c0["x"], q, c0["graph"], c0["entry"], 8, k, ef, rerank)
    compare(run_gpu(*args, max_hops=600, lanes=lanes), run_oracle(orc, *args, max_hops=600))


@pytest.mark.parametrize("ef,rerank,k,nseed", [(2, 50, 10, 128), (3, 3, 3, 128), (8, 200, 10, 128), (5, 64, 5, 7),
                                               (40, 300, 20, 16), (64, 64, 10, 3), (33, 97, 10, 128)])
@pytest.mark.parametrize("layout", ["table", "colocated"])
def test_lazy_pool_window_and_rank_cases(orc, c0, ef, rerank, k, nseed, layout):
    # new keys stay in an unsorted pending buffer and are merged in batches; the next
    # expansion is the smaller of the pool's first unexpanded entry (rank sel + pexp) and the
    # smallest pending key (rank = pool lower bound + expanded pending keys below it).  These
    # cases put the window [0, ef) well inside a larger pool (ef < R), start from pools that are
    # not full (few seeds, so nothing is pruned and the buffer fills at once), and use window
    # sizes that are not multiples of the 32-entry mask block; the table never forgets, so the
    # lazy path runs to the end.  Trace, pool and outputs must equal Alg. 1's.
    q = c0["q"][:41]
    entry = c0["entry"][:nseed]
    args = (c0["x"], q, c0["graph"], entry, 8, k, ef, rerank)
    compare(run_gpu(*args, max_hops=800, layout=layout), run_oracle(orc, *args, max_hops=800))


@pytest.mark.parametrize("slots", [256, 512, 0])
def test_forgetful_visited_cache_is_still_exact(orc, c0, slots):
    # small visited tables forget ids; the pool / trace / output must not change.
    args = (c0["x"], c0["q"], c0["graph"], c0["entry"], 8, 10, 128, 128)
    g = run_gpu(*args, max_hops=400, visited_slots=slots)
    if slots == 256:
        assert g["n_miss"].sum() > 0
    compare(g, run_oracle(orc, *args, max_hops=400), exact_nlp=False)


@pytest.mark.parametrize("lanes", [0, 4])
def test_c0_sq4(orc, c0, lanes):
    args = (c0["x"], c0["q"], c0["graph"], c0["entry"], 4, 10, 64, 128)
    compare(run_gpu(*args, max_hops=300, lanes=lanes), run_oracle(orc, *args, max_hops=300))


def test_ip_sq8_and_sq4_degree64(orc):
    cfg = synth.get_config("C3").scaled(n=8000, nq=48, clusters=64)
    w = synth.make_workload(cfg, device="cuda")
    for bits in (8, 4):
        args = (w["x"], w["q"], w["graph"], w["entry"], bits, 100, 128, 128, "ip")
        compare(run_gpu(*args, max_hops=300), run_oracle(orc, *args, max_hops=300))


@pytest.mark.parametrize("lanes", [0, 32])
def test_sq4_high_dim(orc, lanes):
    cfg = synth.get_config("C2").scaled(n=6000, nq=25, clusters=6, n_seeds=256)
    w = synth.make_workload(cfg, device="cuda")
    args = (w["x"], w["q"], w["graph"], w["entry"], 4, 10, 64, 128)
    compare(run_gpu(*args, max_hops=200, lanes=lanes), run_oracle(orc, *args, max_hops=200))


@pytest.mark.parametrize("d,bits,metric,layout", [(144, 8, "l2", "table"), (200, 8, "ip", "table"), (200, 8, "l2", "colocated"),
                                                  (328, 4, "l2", "table"), (144, 8, "ip", "colocated")])
def test_code_rows_not_32_byte_aligned(orc, d, bits, metric, layout):
    # The generic gather reads a lane's adjacent 16-byte chunks with one 32-byte load per pair when
    # every code row starts on a 32-byte boundary, else with two 16-byte loads.  These shapes have an
    # odd number of chunks (144 B = 9, 208 B = 13, 164 -> 176 B = 11), so rows are only 16-byte
    # aligned, the last lane of a code owns one valid and one invalid chunk, and (layout 1) the row
    # stride is odd in 32-byte units as well.
    rng = np.random.default_rng(7)
    n, nq = 3000, 33
    cent = rng.standard_normal((8, d)).astype(np.float32)
    x = (cent[rng.integers(0, 8, n)] + 0.4 * rng.standard_normal((n, d))).astype(np.float32)
    q = (cent[rng.integers(0, 8, nq)] + 0.4 * rng.standard_normal((nq, d))).astype(np.float32)
    g = synth.build_graph(x, 32)
    entry = np.sort(rng.choice(n, 96, replace=False)).astype(np.int32)
    args = (x, q, g, entry, bits, 10, 48, 64, metric)
    compare(run_gpu(*args, max_hops=200, layout=layout), run_oracle(orc, *args, max_hops=200))


def test_padded_rows_duplicates_selfloops_underfill(orc):
    rng = np.random.default_rng(0)
    n, d = 500, 20
    x = rng.standard_normal((n, d)).astype(np.float32)
    g = synth.build_graph(x, 12)
    g[::3, -4:] = -1                  # ragged rows
    g[::5, 0] = np.arange(0, n, 5)    # self loops
    g[1::7, 2] = g[1::7, 1]           # duplicates
    g[:10] = -1                       # isolated nodes: underfilled results
    entry = np.array([0, 3, 3, 250], np.int32)
    q = rng.standard_normal((29, d)).astype(np.float32)
    for layout in ("table", "colocated"):
        args = (x, q, g, entry, 8, 10, 24, 24)
        compare(run_gpu(*args, layout=layout, max_hops=100), run_oracle(orc, *args, max_hops=100))
    # a query seeded only inside an isolated node: padding with -1 / +inf
    o = run_gpu(x, q[:2], g, np.array([4], np.int32), 8, 5, 5, 5)
    assert (o["ids"][:, 1:] == -1).all() and np.isinf(o["dists"][:, 1:]).all()


def test_ef_ge_n_tiny(orc):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((300, 8)).astype(np.float32)
    g = synth.build_graph(x, 8)
    args = (x, rng.standard_normal((9, 8)).astype(np.float32), g, np.array([7], np.int32), 8, 10, 300, 300)
    compare(run_gpu(*args, max_hops=320), run_oracle(orc, *args, max_hops=320))


def test_empty_batch_and_errors(c0):
    xt = _t(c0["x"])
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    ids, dists = ix.search(torch.empty((0, 128), device=DEV), 10, 64)
    assert ids.shape == (0, 10)
    for kw, code in [(dict(k=10, ef=64, rerank_n=5), vsag.VSAG_ERR_INVALID_ARG),
                     (dict(k=0, ef=64), vsag.VSAG_ERR_INVALID_ARG),
                     (dict(k=10, ef=2000), vsag.VSAG_ERR_INVALID_ARG),
                     (dict(k=10, ef=64, visited_slots=1000), vsag.VSAG_ERR_INVALID_ARG)]:
        with pytest.raises(vsag.VsagError) as e:
            ix.search(_t(c0["q"]), **kw)
        assert e.value.code == code
    bad = c0["graph"].copy()
    bad[3, 3] = len(bad)
    with pytest.raises(vsag.VsagError) as e:
        vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(bad))
    assert e.value.code == vsag.VSAG_ERR_INVALID_ARG
    with pytest.raises(vsag.VsagError) as e:
        vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(np.zeros((len(bad), 65), np.int32)))
    assert e.value.code == vsag.VSAG_ERR_UNSUPPORTED
    ix.close()


def test_host_entry_point_matches_device(c0):
    xt = _t(c0["x"])
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    ids, dists = ix.search(_t(c0["q"]), 10, 64)
    hq = torch.from_numpy(c0["q"]).pin_memory()
    hids, hdists = ix.search_host(hq, 10, 64)
    assert torch.equal(hids, ids.cpu()) and torch.equal(hdists, dists.cpu())
    ix.close()


# ----------------------------------------------------------------------------- C1 full size
@pytest.fixture(scope="module")
def c1():
    return synth.make_workload(synth.get_config("C1"), device="cuda")


def test_c1_full_size_parity_all_queries(orc, c1):
    """BASELINE.json config 1 at full size (1M x 128, 10k queries), in bench.py's launch
    configuration, compared with the oracle on ALL 10,000 queries: expansion sequence, hops,
    final pool ids and tau_l, final ids and re-rank distances."""
    import bench
    ef = bench.C1_EF
    x, q = c1["x"], c1["q"]
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(c1["entry"]), adj=_t(c1["graph"]))
    ids, dists, tr = ix.search(_t(q), 10, ef, ef, trace=True, max_hops=ef + 64)
    ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
    # the timed launch (no trace: the kernel variant bench.py times) returns the same outputs
    ids_t, dists_t = ix.search(_t(q), 10, ef, ef)[:2]
    assert np.array_equal(ids_t.cpu().numpy(), ids)
    assert np.array_equal(dists_t.cpu().numpy(), dists)
    tr = {k2: v.cpu().numpy() for k2, v in tr.items()}
    rec = synth.recall_at_k(ids, c1["gt"], 10)
    assert rec >= 0.95, rec
    lo_n, hi_n = lo.cpu().numpy(), hi.cpu().numpy()
    ocodes = orc.encode_sq(x, 8, lo_n, hi_n)
    assert np.array_equal(ocodes, codes.cpu().numpy())
    o = orc.search_batch(x, ocodes, lo_n, hi_n, 8, c1["graph"], c1["entry"], q, 10, ef, ef, trace=True,
                         max_hops=ef + 64, nthreads=os.cpu_count() or 8)
    assert (tr["hops"] < ef + 64).all()  # the expansion trace is complete
    for key in ("hops", "expanded", "pool_ids", "pool_tau", "n_hp"):
        assert np.array_equal(tr[key], o[key]), key
    assert np.array_equal(ids, o["ids"])
    assert np.allclose(dists, o["dists"], rtol=RTOL, atol=0)
    # C1 is integer data with l=0, u=255: tau_h == tau_l exactly for every output (AMB-16)
    assert (lo_n == 0).all() and (hi_n == 255).all()
    # the timed config's visited cache forgets a little: same traversal, n_lp >= exact
    assert (tr["n_lp"] >= o["n_lp"]).all()
    # the u32 visited table (chosen when a 14-bit tag cannot identify an id: 256 slots at n=2^20)
    # forgets often but leaves the traversal unchanged; the device bitset is exact
    sample = np.sort(np.random.default_rng(0).choice(len(q), 512, replace=False))
    for kind, slots in (("auto", 256), ("bitset", 0)):
        ids2, _, tr2 = ix.search(_t(q[sample]), 10, ef, ef, trace=True, max_hops=ef + 64, visited_slots=slots,
                                 visited_kind=kind)
        tr2 = {k2: v.cpu().numpy() for k2, v in tr2.items()}
        if kind == "auto":
            assert tr2["n_miss"].sum() > 0 and (tr2["n_lp"] >= o["n_lp"][sample]).all()
        else:
            assert (tr2["n_miss"] == 0).all() and np.array_equal(tr2["n_lp"], o["n_lp"][sample])
        for key in ("hops", "expanded", "pool_ids", "pool_tau"):
            assert np.array_equal(tr2[key], o[key][sample]), (kind, key)
        assert np.array_equal(ids2.cpu().numpy(), o["ids"][sample])
    ix.close()


# ----------------------------------------------------------------------------- degree 64, forgetful V
@pytest.fixture(scope="module")
def c3small():
    cfg = synth.get_config("C3").scaled(n=8000, nq=48, clusters=64)
    return synth.make_workload(cfg, device="cuda", gt=False)


@pytest.mark.parametrize("case", ["c0_colocated", "c0_sq4_colocated", "c0_bitset", "c3_ip8", "c3_l2_sq4_colocated", "c2_sq4"])
def test_generic_variant_batches_beyond_16_warps_per_sm(orc, c0, c3small, case):
    # The generic kernel variant exists in two builds: 128 registers for batches that 16 warps per SM hold
    # at once (nq <= 16 x SMs: every other small test) and 56 registers (36 warps per SM) for larger ones,
    # which also differ in the gather passes they keep in flight.  These cases run the 56-register build
    # on small inputs (the queries repeated past 16 x SMs) against the oracle, element by element.
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    if case.startswith("c0"):
        w, reps = c0, (16 * sms) // len(c0["q"]) + 2
        bits = 4 if "sq4" in case else 8
        kw = dict(layout="colocated") if "colocated" in case else dict(kind="bitset")
        q = np.tile(w["q"], (reps, 1))
        args = (w["x"], q, w["graph"], w["entry"], bits, 10, 40, 64)
    elif case.startswith("c3"):
        w, reps = c3small, (16 * sms) // len(c3small["q"]) + 2
        q = np.tile(w["q"], (reps, 1))
        if case == "c3_ip8":
            args, kw = (w["x"], q, w["graph"], w["entry"], 8, 20, 48, 48, "ip"), {}
        else:
            args, kw = (w["x"], q, w["graph"], w["entry"], 4, 20, 48, 64, "l2"), dict(layout="colocated")
    else:
        cfg = synth.get_config("C2").scaled(n=6000, nq=25, clusters=6, n_seeds=256)
        w = synth.make_workload(cfg, device="cuda")
        q = np.tile(w["q"], ((16 * sms) // 25 + 2, 1))
        args, kw = (w["x"], q, w["graph"], w["entry"], 4, 10, 32, 64), {}
    assert len(q) > 16 * sms
    compare(run_gpu(*args, max_hops=200, **kw), run_oracle(orc, *args, max_hops=200))


@pytest.mark.parametrize("kind,slots", [("u16", 256), ("u16", 512), ("u32", 256), ("u32", 1024), ("bitset", 0)])
@pytest.mark.parametrize("layout", ["table", "colocated"])
@pytest.mark.parametrize("bits,metric", [(8, "ip"), (8, "l2"), (4, "ip")])
def test_degree64_forgetful_visited(orc, c3small, kind, slots, layout, bits, metric):
    """C3's production path at full size: degree 64 (two 32-id slices per row, E = 2) with a
    visited cache far smaller than |V|, so ids are forgotten and every merge runs the
    de-duplicating variant (merge_new<2, true>); u16 buckets, u32 probing, both layouts.  The
    traversal must equal Alg. 1 with an exact V; the bitset never forgets."""
    w = c3small
    args = (w["x"], w["q"], w["graph"], w["entry"], bits, 100, 128, 128, metric)
    g = run_gpu(*args, layout=layout, max_hops=300, visited_slots=slots, kind=kind)
    o = run_oracle(orc, *args, max_hops=300)
    if kind == "bitset":
        compare(g, o, exact_nlp=True)
    else:
        assert g["n_miss"].sum() > 0, "the cache must forget for this test to mean anything"
        assert (g["n_miss"] > 0).mean() > 0.9
        compare(g, o, exact_nlp=False)


def test_degree64_forgetful_qlp(orc, c3small):
    # the QLP checkpoint (NEXT-4b) on the same forgetful degree-64 setup
    w = c3small
    x, q, g, entry = w["x"], w["q"], w["graph"], w["entry"]
    lo_n, hi_n = orc.train_sq(x)
    ocodes = orc.encode_sq(x, 8, lo_n, hi_n)
    k, ef, ef_low = 10, 96, 32
    shrunk = None
    for thr in [int(v) for v in np.geomspace(10, 10 ** 8, 80)]:  # feature 2 >= 0
        qlp = (6, ef_low, 2, thr)
        o = orc.search_batch(x, ocodes, lo_n, hi_n, 8, g, entry, q, k, ef, ef, "ip", trace=True, max_hops=300,
                             nthreads=8, qlp=qlp)
        shrunk = o["n_hp"] == ef_low
        if 0.2 < shrunk.mean() < 0.8:
            break
    assert 0 < shrunk.sum() < len(q)
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(entry), adj=_t(g))
    ids, dists, tr = ix.search(_t(q), k, ef, ef, "ip", trace=True, max_hops=300, visited_slots=256, qlp=qlp)
    ix.close()
    tr = {k2: v.cpu().numpy() for k2, v in tr.items()}
    assert tr["n_miss"].sum() > 0
    for key in ("hops", "n_hp", "expanded", "pool_ids", "pool_tau"):
        assert np.array_equal(tr[key], o[key]), key
    assert np.array_equal(ids.cpu().numpy(), o["ids"])
    assert np.allclose(dists.cpu().numpy(), o["dists"], rtol=RTOL, atol=0)


# ----------------------------------------------------------------------------- C2-C4 full size
def _full_size_sampled(orc, cfg, efs, nsample=64, kinds=("auto",), lower_upper=None, metric=None):
    """A BASELINE.json config at full size: the whole batch is searched in bench.py's launch
    configuration (no trace) and traced; the oracle recomputes a seeded sample of queries
    one by one and is compared element by element (trace, pool, ids, dists)."""
    w = synth.make_workload(cfg, device="cuda", gt=False)
    x, q, g, entry = w["x"], w["q"], w["graph"], w["entry"]
    metric = metric or cfg.metric
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, cfg.bits)
    lo_n, hi_n = lo.cpu().numpy(), hi.cpu().numpy()
    ix = vsag.Index(xt, codes, lo, hi, cfg.bits, _t(entry), adj=_t(g))
    sample = np.sort(np.random.default_rng(7).choice(len(q), min(nsample, len(q)), replace=False))
    ocodes = orc.encode_sq(x[:: max(1, len(x) // 4096)], cfg.bits, lo_n, hi_n)
    assert np.array_equal(ocodes, codes.cpu().numpy()[:: max(1, len(x) // 4096)])  # a row sample of the codes
    ocodes = orc.encode_sq(x, cfg.bits, lo_n, hi_n)
    qt = _t(q)
    for ef in efs:
        rr = cfg.rerank_n(ef)
        mh = 4 * ef + 64
        ids_t, dists_t = ix.search(qt, cfg.k, ef, rr, metric)[:2]  # the timed launch configuration
        o = orc.search_batch(x, ocodes, lo_n, hi_n, cfg.bits, g, entry, q[sample], cfg.k, ef, rr, metric, trace=True,
                             max_hops=mh, nthreads=os.cpu_count() or 8)
        assert (o["hops"] < mh).all()
        assert np.array_equal(ids_t.cpu().numpy()[sample], o["ids"]), (cfg.name, ef, "ids (timed launch)")
        assert np.allclose(dists_t.cpu().numpy()[sample], o["dists"], rtol=RTOL, atol=0)
        for kind in kinds:
            ids, dists, tr = ix.search(qt, cfg.k, ef, rr, metric, trace=True, max_hops=mh, visited_kind=kind)
            assert torch.equal(ids, ids_t) and torch.equal(dists, dists_t)
            tr = {k2: v.cpu().numpy()[sample] for k2, v in tr.items()}
            for key in ("hops", "expanded", "pool_ids", "pool_tau", "n_hp"):
                assert np.array_equal(tr[key], o[key]), (cfg.name, ef, kind, key)
            if kind == "bitset":
                assert (tr["n_miss"] == 0).all() and np.array_equal(tr["n_lp"], o["n_lp"])
            else:
                assert (tr["n_lp"] >= o["n_lp"]).all()
    ix.close()


def test_c2_full_size_sampled_parity(orc):
    # 1M x 960 SQ4 L2, S = 16,384 entry seeds, R' = 2 ef (BASELINE.json config 2)
    _full_size_sampled(orc, synth.get_config("C2"), (64, 256))


def test_c3_full_size_sampled_parity(orc):
    # 1M x 768 SQ8 IP, degree 64, k = 100, ef up to 512 (BASELINE.json config 3): the
    # default visited cache forgets (|V| ~ 10^4); the exact bitset gives n_lp of Alg. 1
    _full_size_sampled(orc, synth.get_config("C3"), (128, 512), kinds=("auto", "bitset"))


def test_c4_full_size_sampled_parity(orc):
    # BASELINE.json config 4 (SQ4 L2, 100k queries in one batch) at 2M rows (the 10M-row graph
    # takes ~30 min to build; VSAG_TEST_C4_N=10000000 runs the full size)
    n = int(os.environ.get("VSAG_TEST_C4_N", "2000000"))
    _full_size_sampled(orc, synth.get_config("C4").scaled(n=n), (32, 128), kinds=("auto", "bitset"))


# ----------------------------------------------------------------------------- boundary
def test_boundary_validation(c0):
    import ctypes
    xt = _t(c0["x"])
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    q = _t(c0["q"])
    nq = q.shape[0]
    hq = torch.from_numpy(c0["q"]).pin_memory()
    hids = torch.empty((nq, 10), dtype=torch.int32).pin_memory()
    hd = torch.empty((nq, 10), dtype=torch.float32).pin_memory()
    did = torch.empty((nq, 10), dtype=torch.int32, device=DEV)
    dd = torch.empty((nq, 10), dtype=torch.float32, device=DEV)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def host(k=10, ef=64, n=nq, **kw):
        sp = vsag.Index._params(k, ef, 0, "l2", 0, 0, **kw)
        return vsag.lib.vsag_search_batch_host(ix._h, vsag._ptr(hq), n, ctypes.byref(sp), vsag._ptr(hids),
                                               vsag._ptr(hd), stream)

    def dev(k=10, ef=64, n=nq, qp=None, raw_kind=None, **kw):
        sp = vsag.Index._params(k, ef, 0, "l2", 0, 0, **kw)
        if raw_kind is not None:
            sp.visited_kind = raw_kind
        qp = vsag._ptr(q) if qp is None else qp
        return vsag.lib.vsag_search_batch_ex(ix._h, qp, n, ctypes.byref(sp), vsag._ptr(did), vsag._ptr(dd), None,
                                             None, stream)

    assert host() == vsag.VSAG_OK and dev() == vsag.VSAG_OK
    # parameters are validated before any allocation: a negative k is an argument error, not OOM
    for kw in (dict(k=-5), dict(k=-(1 << 30)), dict(k=0), dict(ef=0), dict(k=20, ef=10)):
        assert host(**kw) == vsag.VSAG_ERR_INVALID_ARG, kw
        assert dev(**kw) == vsag.VSAG_ERR_INVALID_ARG, kw
    assert host(n=-1) == vsag.VSAG_ERR_INVALID_ARG
    # the persistent scheduler's 32-bit counter: huge batches are refused up front
    assert dev(n=1 << 31) == vsag.VSAG_ERR_UNSUPPORTED and host(n=1 << 31) == vsag.VSAG_ERR_UNSUPPORTED
    # 16-byte alignment of queries (the re-rank's vector loads)
    assert dev(n=nq - 1, qp=ctypes.c_void_p(q.data_ptr() + 4)) == vsag.VSAG_ERR_INVALID_ARG
    assert dev(raw_kind=5) == vsag.VSAG_ERR_INVALID_ARG
    assert vsag.lib.vsag_last_error().decode()
    torch.cuda.synchronize()
    # the index's base must be 16-byte aligned
    flat = torch.empty(xt.numel() + 1, dtype=torch.float32, device=DEV)
    xmis = flat[1:].view(xt.shape)
    xmis.copy_(xt)
    with pytest.raises(vsag.VsagError) as e:
        vsag.Index(xmis, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    assert e.value.code == vsag.VSAG_ERR_INVALID_ARG
    # the binding validates caller-given outputs (the kernels write nq * k values through them)
    for bad in [(did[:, :5], dd), (did, dd.double()), (did.t().contiguous().t(), dd), (did.cpu(), dd)]:
        with pytest.raises((TypeError, ValueError)):
            ix.search(q, 10, 64, out=bad)
    with pytest.raises((TypeError, ValueError)):
        ix.search_host(hq, 10, 64, out=(did, dd))
    # nothing above disturbed the index: a valid call still matches
    ids, dists = ix.search(q, 10, 64)
    hids2, hd2 = ix.search_host(hq, 10, 64)
    assert torch.equal(ids.cpu(), hids2) and torch.equal(dists.cpu(), hd2)
    ix.close()


# ----------------------------------------------------------------------------- NEXT-1
@pytest.mark.parametrize("q", [1.0, 0.99, 0.9, 0.75])
def test_train_quantile_parity(orc, q):
    # truncated SQ training (App. G): per-dimension order statistics, bit-identical
    rng = np.random.default_rng(11)
    n, d = 5003, 37
    x = rng.standard_normal((n, d)).astype(np.float32)
    x[rng.integers(0, n, 40), rng.integers(0, d, 40)] = 50.0  # outliers
    x[:, 3] = np.round(x[:, 3])                                # many ties
    x[:, 5] = 0.0
    x[::2, 5] = -0.0                                           # +/-0 mix
    x[:, 6] = 2.5                                              # constant
    lo, hi = vsag.train_sq(_t(x), q)
    olo, ohi = orc.train_sq_quantile(x, q)
    assert np.array_equal(lo.cpu().numpy().view(np.uint32), olo.view(np.uint32))
    assert np.array_equal(hi.cpu().numpy().view(np.uint32), ohi.view(np.uint32))
    with pytest.raises(vsag.VsagError):
        vsag.train_sq(_t(x), 0.4)


@pytest.mark.parametrize("bits", [4, 8])
def test_l2w_parity_c2_like(orc, bits):
    # weighted code-space L2 traversal (NEXT-1b) on C2's shape (per-dimension scales
    # U[0.05, 1]), truncated SQ range, plain L2 re-rank: full trace parity
    cfg = synth.get_config("C2").scaled(n=6000, nq=25, clusters=6, n_seeds=256)
    w = synth.make_workload(cfg, device="cuda")
    lo, hi = orc.train_sq_quantile(w["x"], 0.99)
    args = (w["x"], w["q"], w["graph"], w["entry"], bits, 10, 64, 128, "l2w")
    g = run_gpu(*args, max_hops=200, lower=lo, upper=hi)
    compare(g, run_oracle(orc, *args, max_hops=200, lower=lo, upper=hi))


def test_l2w_c0_sq8_and_recall_gain(orc, c0):
    args = (c0["x"], c0["q"], c0["graph"], c0["entry"], 8, 10, 64, 64, "l2w")
    compare(run_gpu(*args, max_hops=300), run_oracle(orc, *args, max_hops=300))
    # on C2's shape the weighted traversal fixes the range-normalisation distortion of the
    # literal code-space L2: recall after re-rank rises
    cfg = synth.get_config("C2").scaled(n=8000, nq=60, clusters=8, n_seeds=512)
    w = synth.make_workload(cfg, device="cuda")
    rec = {}
    for metric in ("l2", "l2w"):
        g = run_gpu(w["x"], w["q"], w["graph"], w["entry"], 4, 10, 32, 32, metric)
        rec[metric] = synth.recall_at_k(g["ids"], w["gt"], 10)
    assert rec["l2w"] > rec["l2"] + 0.05, rec


# ----------------------------------------------------------------------------- NEXT-2
@pytest.fixture(scope="module")
def labelled():
    cfg = synth.get_config("C0").scaled(n=1500, nq=40, clusters=3, n_seeds=48)
    w = synth.make_workload(cfg, device="cpu", gt=False)
    adj, lab = synth.build_labelled_graph(w["x"], 24)
    return w, adj, lab


@pytest.mark.parametrize("m_s,alpha_s,csr", [(0, 2.0, False), (12, 1.2, False), (6, 1.0, True), (0, 1.0, True),
                                             (9, 0.0, False)])
def test_label_filter_parity(orc, labelled, m_s, alpha_s, csr):
    # Alg. 1 line 8 edge filter (R-23) on an Alg. 2-labelled graph: full trace parity
    w, adj, lab = labelled
    x, q, entry = w["x"], w["q"], w["entry"]
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    if csr:
        rows = [r[r >= 0] for r in adj]
        row_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
        col = np.concatenate(rows).astype(np.int32)
        lcol = np.concatenate([lab[i][adj[i] >= 0] for i in range(len(adj))]).astype(np.float32)
        ix = vsag.Index(xt, codes, lo, hi, 8, _t(entry), adj=_t(col), row_ptr=_t(row_ptr), degree=adj.shape[1])
        ix.set_labels(_t(lcol), row_ptr=_t(row_ptr))
    else:
        ix = vsag.Index(xt, codes, lo, hi, 8, _t(entry), adj=_t(adj))
        ix.set_labels(_t(lab))
    ids, dists, tr = ix.search(_t(q), 10, 40, 40, trace=True, max_hops=90, visited_slots=16384, max_degree=m_s,
                               alpha_s=alpha_s)
    g = dict(ids=ids.cpu().numpy(), dists=dists.cpu().numpy(), codes=codes.cpu().numpy(), lower=lo.cpu().numpy(),
             upper=hi.cpu().numpy(), **{k2: v.cpu().numpy() for k2, v in tr.items()})
    ix.close()
    olab = lab if alpha_s > 0 else np.zeros_like(lab)  # alpha_s = 0: no label bound, cap only
    o = run_oracle(orc, x, q, adj, entry, 8, 10, 40, 40, max_hops=90)
    o = orc.search_batch(x, o["codes"], o["lower"], o["upper"], 8, adj, entry, q, 10, 40, 40, "l2", trace=True,
                         max_hops=90, nthreads=8, labels=olab, m_s=m_s, alpha_s=alpha_s if alpha_s > 0 else np.inf)
    o.update(codes=g["codes"], lower=g["lower"], upper=g["upper"])
    compare(g, o)


def test_label_filter_errors(c0):
    xt = _t(c0["x"])
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    with pytest.raises(vsag.VsagError) as e:
        ix.search(_t(c0["q"]), 10, 64, alpha_s=1.2)  # no labels
    assert e.value.code == vsag.VSAG_ERR_INVALID_ARG
    bad = np.ones(c0["graph"].shape, np.float32)
    bad[5, 3] = np.nan
    with pytest.raises(vsag.VsagError):
        ix.set_labels(_t(bad))
    ix.close()


# ----------------------------------------------------------------------------- NEXT-4
@pytest.mark.parametrize("delta", [0.0, 0.5, 0.3, 1.0])
def test_prs_delta_parity(orc, c0, delta):
    # PRS with redundancy ratio delta (§3.3.3): round(delta * n) highest in-degree nodes get
    # co-located neighbour-code blocks; results are identical for every delta
    x, q, g, entry = c0["x"], c0["q"], c0["graph"], c0["entry"]
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(entry), adj=_t(g))
    ix.set_prs(delta)
    info = ix.info()
    n = len(x)
    assert info["prs_nodes"] == round(delta * n)
    assert info["prs_bytes"] == round(delta * n) * g.shape[1] * 128
    ids, dists, tr = ix.search(_t(q), 10, 64, 64, trace=True, max_hops=400, visited_slots=16384)
    gg = dict(ids=ids.cpu().numpy(), dists=dists.cpu().numpy(), codes=codes.cpu().numpy(), lower=lo.cpu().numpy(),
              upper=hi.cpu().numpy(), **{k2: v.cpu().numpy() for k2, v in tr.items()})
    ix.close()
    compare(gg, run_oracle(orc, x, q, g, entry, 8, 10, 64, 64, max_hops=400))
    if delta == 0.5:  # the SPEC example's rule: delta = 0.5 on n = 200 -> exactly 100 blocks
        ix2 = vsag.Index(xt[:200].contiguous(), codes[:200].contiguous(), lo, hi, 8, _t(np.array([0, 50, 100], np.int32)),
                         adj=_t(np.where(g[:200] < 200, g[:200], -1)))
        ix2.set_prs(0.5)
        assert ix2.info()["prs_nodes"] == 100
        with pytest.raises(vsag.VsagError):
            ix2.set_prs(1.5)
        ix2.close()


# ----------------------------------------------------------------------------- NEXT-3
@pytest.mark.parametrize("bits", [8, 4])
def test_adaptive_rerank_parity(orc, bits):
    # exact early stop of the re-rank (R-27): same outputs as the full re-rank, and n_hp equal
    # to the oracle's (the rule is evaluated per group of 4 on both sides)
    cfg = synth.get_config("C1").scaled(n=4000, nq=40, clusters=4, n_seeds=64)
    w = synth.make_workload(cfg, device="cuda")
    x, q, g, entry = w["x"].copy(), w["q"], w["graph"], w["entry"]
    x[0], x[1] = 0.0, 255.0  # uniform step 1 in every dimension, as at full-size C1
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, bits)
    ix = vsag.Index(xt, codes, lo, hi, bits, _t(entry), adj=_t(g))
    ids, dists, tr = ix.search(_t(q), 10, 64, 64, trace=True, max_hops=100, visited_slots=16384,
                               rerank_adaptive=True)
    ids_f, dists_f = ix.search(_t(q), 10, 64, 64)
    ix.close()
    lo_n, hi_n = lo.cpu().numpy(), hi.cpu().numpy()
    ocodes = orc.encode_sq(x, bits, lo_n, hi_n)
    o = orc.search_batch(x, ocodes, lo_n, hi_n, bits, g, entry, q, 10, 64, 64, "l2", trace=True, max_hops=100,
                         nthreads=8, adaptive=True)
    assert np.array_equal(tr["n_hp"].cpu().numpy(), o["n_hp"])
    assert np.array_equal(ids.cpu().numpy(), o["ids"]) and np.array_equal(ids.cpu().numpy(), ids_f.cpu().numpy())
    assert np.allclose(dists.cpu().numpy(), o["dists"], rtol=RTOL, atol=0)
    assert torch.equal(dists, dists_f)
    for key in ("hops", "expanded", "pool_ids", "pool_tau"):
        assert np.array_equal(tr[key].cpu().numpy(), o[key]), key


def test_adaptive_rerank_errors(c0):
    x = c0["x"].copy()
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    with pytest.raises(vsag.VsagError):
        ix.search(_t(c0["q"]), 10, 64, metric="ip", rerank_adaptive=True)
    ix.close()
    # a base that leaves the trained range (truncated training) invalidates the bound
    lo2, hi2 = vsag.train_sq(xt, 0.9)
    codes2, _, _ = vsag.encode_sq(xt, 8, lo2, hi2)
    ix2 = vsag.Index(xt, codes2, lo2, hi2, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    with pytest.raises(vsag.VsagError):
        ix2.search(_t(c0["q"]), 10, 64, rerank_adaptive=True)
    ix2.close()


# ----------------------------------------------------------------------------- NEXT-4b
@pytest.mark.parametrize("feat,hop,ef_low", [(1, 0, 16), (1, 8, 24), (2, 3, 12), (2, 20, 32)])
def test_qlp_parity(orc, c0, feat, hop, ef_low):
    # QLP checkpoint (R-28): the same decision per query as the oracle (some queries shrink,
    # some do not) and then the same traversal, pool and outputs
    x, q, g, entry = c0["x"], c0["q"], c0["graph"], c0["entry"]
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    lo_n, hi_n = lo.cpu().numpy(), hi.cpu().numpy()
    ocodes = orc.encode_sq(x, 8, lo_n, hi_n)
    ef = 64
    # a threshold at which some queries shrink and some do not (decided by the oracle alone)
    o = None
    for thr in [int(v) for v in np.geomspace(100, 10 ** 7, 40)]:
        qlp = (hop, ef_low, feat, thr)
        o = orc.search_batch(x, ocodes, lo_n, hi_n, 8, g, entry, q, 10, ef, ef, trace=True, max_hops=200,
                             nthreads=8, qlp=qlp)
        shrunk = o["n_hp"] == ef_low
        if 0.2 < shrunk.mean() < 0.8:
            break
    assert 0 < shrunk.sum() < len(q)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(entry), adj=_t(g))
    ids, dists, tr = ix.search(_t(q), 10, ef, ef, trace=True, max_hops=200, visited_slots=16384, qlp=qlp)
    ids_t, dists_t = ix.search(_t(q), 10, ef, ef, visited_slots=16384, qlp=qlp)[:2]
    ix.close()
    tr = {k2: v.cpu().numpy() for k2, v in tr.items()}
    shrunk = o["n_hp"] == ef_low
    if hop == 0:
        assert shrunk.any() and (~shrunk).any()
    for key in ("hops", "n_lp", "n_hp", "expanded", "pool_ids", "pool_tau"):
        assert np.array_equal(tr[key], o[key]), key
    assert np.array_equal(ids.cpu().numpy(), o["ids"]) and torch.equal(ids, ids_t)
    assert np.allclose(dists.cpu().numpy(), o["dists"], rtol=RTOL, atol=0) and torch.equal(dists, dists_t)


def test_qlp_errors(c0):
    xt = _t(c0["x"])
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, _t(c0["entry"]), adj=_t(c0["graph"]))
    q = _t(c0["q"])
    for qlp in [(1, 5, 1, 0), (1, 80, 1, 0), (-1, 20, 1, 0), (1, 20, 3, 0), (1, 20, 0, 0)]:
        with pytest.raises(vsag.VsagError):
            ix.search(q, 10, 64, qlp=qlp)
    ix.close()


def test_maximum_pool_and_rerank_sizes(orc):
    # the largest pool the ABI accepts (L = max(ef, R) = 1024) and k = 100, R' = 1024 (the
    # re-rank keys spill past the registers into shared memory): same trace and outputs
    cfg = synth.get_config("C0").scaled(n=3000, nq=6, n_seeds=64)
    w = synth.make_workload(cfg, device="cuda", gt=False)
    x, q, g, entry = w["x"], w["q"], w["graph"], w["entry"]
    for ef, rr, k in [(1024, 1024, 100), (600, 1024, 10)]:
        gg, oo = run_gpu(x, q, g, entry, 8, k, ef, rr, max_hops=1200), \
            run_oracle(orc, x, q, g, entry, 8, k, ef, rr, max_hops=1200)
        compare(gg, oo)


@pytest.mark.parametrize("bits,metric", [(4, "l2"), (8, "ip")])
def test_qlp_parity_sq4_and_ip(orc, bits, metric):
    # the QLP checkpoint in the other tau_l modes (generic variant), degree 64 for IP
    cfg = synth.get_config("C3" if metric == "ip" else "C0").scaled(n=5000, nq=40, clusters=16)
    w = synth.make_workload(cfg, device="cuda", gt=False)
    x, q, g, entry = w["x"], w["q"], w["graph"], w["entry"]
    lo_n, hi_n = orc.train_sq(x)
    ocodes = orc.encode_sq(x, bits, lo_n, hi_n)
    k, ef, ef_low = 10, 64, 24
    shrunk = None
    for thr in [int(v) for v in np.geomspace(10, 10 ** 7, 50)] + [-int(v) for v in np.geomspace(10, 10 ** 7, 50)]:
        qlp = (4, ef_low, 2, thr)
        o = orc.search_batch(x, ocodes, lo_n, hi_n, bits, g, entry, q, k, ef, ef, metric, trace=True, max_hops=300,
                             nthreads=8, qlp=qlp)
        shrunk = o["n_hp"] == ef_low
        if 0.2 < shrunk.mean() < 0.8:
            break
    assert 0 < shrunk.sum() < len(q)
    xt = _t(x)
    codes, lo, hi = vsag.encode_sq(xt, bits)
    ix = vsag.Index(xt, codes, lo, hi, bits, _t(entry), adj=_t(g))
    ids, dists, tr = ix.search(_t(q), k, ef, ef, metric, trace=True, max_hops=300, visited_slots=16384, qlp=qlp)
    ix.close()
    tr = {k2: v.cpu().numpy() for k2, v in tr.items()}
    for key in ("hops", "n_lp", "n_hp", "expanded", "pool_ids", "pool_tau"):
        assert np.array_equal(tr[key], o[key]), key
    assert np.array_equal(ids.cpu().numpy(), o["ids"])
    assert np.allclose(dists.cpu().numpy(), o["dists"], rtol=RTOL, atol=0)


# ----------------------------------------------------------------------------- kernel unit checks
@pytest.mark.parametrize("tool", ["select_test", "umma_test"])
def test_standalone_kernel_checks(tmp_path, tool):
    """tools/select_test.cu (seed selection, both kernels, 32- and 64-bit keys, ties) and
    tools/umma_test.cu (the tcgen05 seed contraction) against their CPU references."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / tool)
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-I", os.path.join(root, "include"), "-I", os.path.join(root, "paper_2503_17911_b200", "csrc"),
                    os.path.join(root, "tools", tool + ".cu"), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
