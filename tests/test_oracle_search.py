"""Pins for the oracle's greedy search + rerank (rows a5-a8 of SURVEY.md §8).

Pinned against: the hand-traced worked example W1 (tests/golden/w1_example.json),
brute force on tiny inputs (ef >= N on a connected graph; lossless codes + full
rerank == exact kNN), the set-semantics invariants that follow from Alg. 1
 under readings R-8..R-14, and the C0 fingerprint computed
independently during the survey (tests/golden/c0_fingerprint.json).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _w1():
    return json.load(open(os.path.join(GOLD, "w1_example.json")))


@pytest.mark.parametrize("case", [c["name"] for c in _w1()["cases"]])
def test_w1_worked_example(orc, case):
    w = _w1()
    c = [x for x in w["cases"] if x["name"] == case][0]
    codes_f = np.array(w["codes"], np.float32)
    lo, hi = np.zeros(4, np.float32), np.full(4, 255.0, np.float32)
    codes = orc.encode_sq(codes_f, 8, lo, hi)
    assert (codes == codes_f.astype(np.uint8)).all()
    q = np.array([w["query"]], np.float32)
    taus = [orc.tau_l(q[0], codes[i], 8, lo, hi) for i in range(8)]
    assert taus == w["tau_l"]
    r = orc.search_batch(codes_f, codes, lo, hi, 8, np.array(w["rows"], np.int32), np.array(c["entry"]),
                         q, c["k"], c["ef"], c["rerank"], trace=True, max_hops=8)
    assert list(r["expanded"][0][: c["hops"]]) == c["trace"]
    assert r["hops"][0] == c["hops"] and r["n_lp"][0] == c["n_lp"]
    assert list(r["pool_ids"][0]) == c["pool_ids"] and list(r["pool_tau"][0]) == c["pool_tau"]
    assert list(r["ids"][0]) == c["ids"] and list(r["dists"][0]) == c["dists"]
    assert r["n_hp"][0] == min(c["rerank"], len(c["pool_ids"]))


def _tiny(n=300, d=12, r=8, seed=0, integer=False):
    rng = np.random.default_rng(seed)
    if integer:
        x = rng.integers(0, 256, (n, d)).astype(np.float32)
        x[0] = 0
        x[1] = 255
    else:
        x = rng.standard_normal((n, d)).astype(np.float32)
    g = synth.build_graph(x, r)
    return x, g


def _reachable(g, entry):
    seen = set(int(e) for e in entry)
    stack = list(seen)
    while stack:
        i = stack.pop()
        for j in g[i]:
            if j >= 0 and int(j) not in seen:
                seen.add(int(j))
                stack.append(int(j))
    return seen


def _brute_tau_l2(orc, q, codes_u8_unpacked, lo, hi, bits):
    cq = orc.encode_sq(q[None], bits, lo, hi)[0]
    if bits == 4:
        full = np.empty(len(q), np.int64)
        full[0::2] = cq & 0x0F
        full[1::2] = cq[: (len(q) + 1) // 2][: len(full[1::2])] >> 4
        cq = full
    diff = codes_u8_unpacked.astype(np.int64) - cq.astype(np.int64)[None]
    return (diff * diff).sum(1)


def _unpack(codes, d, bits):
    if bits == 8:
        return codes.astype(np.int64)
    full = np.empty((codes.shape[0], d), np.int64)
    full[:, 0::2] = codes[:, : (d + 1) // 2] & 0x0F
    full[:, 1::2] = (codes[:, : d // 2] >> 4)
    return full


@pytest.mark.parametrize("bits", [8, 4])
def test_ef_ge_n_pool_is_bruteforce_topL(orc, bits):
    # BASELINE.json north_star invariant: ef >= N on a connected graph -> quantized search
    # returns the exact tau_l top-L (ties by id) over all N.
    # (General form: the pool equals the brute-force order of the set reachable from I.)
    x, g = _tiny(n=250, d=10, r=8, seed=1)
    entry = np.array([3], np.int32)
    reach = np.array(sorted(_reachable(g, entry)))
    assert len(reach) > 200
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, bits, lo, hi)
    q = np.random.default_rng(2).standard_normal((5, 10)).astype(np.float32)
    n = len(x)
    r = orc.search_batch(x, codes, lo, hi, bits, g, entry, q, 10, n, n, trace=True)
    full = _unpack(codes, 10, bits)
    m = len(reach)
    for qi in range(len(q)):
        tau = _brute_tau_l2(orc, q[qi], full[reach], lo, hi, bits)
        order = np.lexsort((reach, tau))
        assert list(r["pool_ids"][qi][:m]) == list(reach[order])
        assert list(r["pool_tau"][qi][:m]) == list(tau[order])
        assert (r["pool_ids"][qi][m:] == -1).all()
        assert r["hops"][qi] == m  # every reachable node expanded exactly once
        assert r["n_lp"][qi] == m  # each node evaluated once (entry counted once)


def test_complete_graph_one_expansion_visits_all(orc):
    n, d = 40, 6
    x = np.random.default_rng(4).standard_normal((n, d)).astype(np.float32)
    g = np.array([[j for j in range(n) if j != i] for i in range(n)], np.int32)
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, 8, lo, hi)
    q = x[:3] + 0.01
    r = orc.search_batch(x, codes, lo, hi, 8, g, np.array([0]), q, 5, 1, n, trace=True, max_hops=4)
    assert (r["n_lp"] == n).all()
    # ef = 1: the first expansion (the entry) already put every node into the pool
    assert (r["pool_ids"] >= 0).all()


def test_lossless_full_rerank_equals_exact_knn(orc):
    # Integer data in [0,255] with l=0, u=255: SQ8 codes are lossless, tau_l == tau_h; with
    # ef = R = N the output is the exact kNN (ties by id) -- brute-force pin of the whole path.
    x, g = _tiny(n=300, d=16, r=8, seed=5, integer=True)
    lo, hi = orc.train_sq(x)
    assert (lo == 0).all() and (hi == 255).all()
    codes = orc.encode_sq(x, 8, lo, hi)
    q = np.random.default_rng(6).integers(0, 256, (20, 16)).astype(np.float32)
    entry = synth.entry_set(len(x), 8)
    reach = np.array(sorted(_reachable(g, entry)))
    assert len(reach) > 250
    r = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, len(x), len(x))
    gt = reach[synth.ground_truth(x[reach], q, 10)]  # exact kNN over the reachable set
    assert (r["ids"] == gt).all()
    ex = ((q[:, None, :].astype(np.float64) - x[gt].astype(np.float64)) ** 2).sum(-1)
    assert (r["dists"] == ex.astype(np.float32)).all()


@pytest.fixture(scope="module")
def c0small(orc):
    cfg = synth.get_config("C0").scaled(n=3000, nq=40)
    x = synth.generate_base(cfg)
    q = synth.generate_queries(cfg)
    g = synth.build_graph(x, 16)
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, 8, lo, hi)
    entry = synth.entry_set(cfg.n, 64)
    return x, q, g, lo, hi, codes, entry


def _check_pool_invariants(r, cap):
    for ids, tau in zip(r["pool_ids"], r["pool_tau"]):
        m = ids >= 0
        assert m.sum() <= cap
        assert (~m[np.argmax(~m):]).all() if (~m).any() else True  # padding only at the tail
        v_ids, v_tau = ids[m], tau[m].astype(np.int64)
        assert len(set(v_ids.tolist())) == len(v_ids)  # duplicate-free
        keys = v_tau * (1 << 32) + v_ids
        assert (np.diff(keys) > 0).all()  # strictly ascending (tau, id)


def test_invariants_sorted_dupfree_bounded(orc, c0small):
    x, q, g, lo, hi, codes, entry = c0small
    for ef, rr in ((16, 16), (32, 64), (64, 64)):
        r = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, ef, rr, trace=True, max_hops=400)
        _check_pool_invariants(r, max(ef, rr))
        assert (r["hops"] <= r["n_lp"]).all()
        assert (r["n_lp"] <= len(x) + len(entry)).all()
        for ids, dists in zip(r["ids"], r["dists"]):
            assert len(set(ids.tolist())) == len(ids)
            assert (np.diff(dists) >= 0).all()
        # output distances are the exact tau_h of the output ids
        for qi in range(3):
            for t in range(10):
                assert r["dists"][qi, t] == orc.tau_h(q[qi], x[r["ids"][qi, t]])


def test_permutation_invariance(orc, c0small):
    # Set semantics: row order, seed order and seed duplicates do not matter.
    x, q, g, lo, hi, codes, entry = c0small
    base = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 32, 32, trace=True, max_hops=200)
    rng = np.random.default_rng(9)
    gp = np.array([rng.permutation(row) for row in g], np.int32)
    ep = np.concatenate([entry[::-1], entry[:5]])
    r = orc.search_batch(x, codes, lo, hi, 8, gp, ep, q, 10, 32, 32, trace=True, max_hops=200)
    for key in ("ids", "dists", "expanded", "pool_ids", "pool_tau", "hops", "n_lp"):
        assert (r[key] == base[key]).all(), key


def test_rerank_count_independence(orc, c0small):
    # Window equivalence: the expansion trace and the first ef pool entries
    # do not depend on R >= ef.
    x, q, g, lo, hi, codes, entry = c0small
    a = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 32, 32, trace=True, max_hops=200)
    b = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 32, 96, trace=True, max_hops=200)
    assert (a["expanded"] == b["expanded"]).all() and (a["hops"] == b["hops"]).all()
    assert (a["pool_ids"] == b["pool_ids"][:, :32]).all()
    assert (a["pool_tau"] == b["pool_tau"][:, :32]).all()


def test_rerank_whole_pool_is_exact_topk_of_pool(orc, c0small):
    # re-ranking the whole pool returns the exact tau_h top-k of the pool.
    x, q, g, lo, hi, codes, entry = c0small
    r = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 48, 48, trace=True)
    for qi in range(len(q)):
        pool = r["pool_ids"][qi]
        th = ((x[pool].astype(np.float64) - q[qi].astype(np.float64)) ** 2).sum(1).astype(np.float32)
        order = np.lexsort((pool, th))[:10]
        assert list(pool[order]) == list(r["ids"][qi])


def test_csr_equals_fixed_degree_and_determinism(orc, c0small):
    x, q, g, lo, hi, codes, entry = c0small
    a = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 32, 32, trace=True, max_hops=200)
    # CSR with ragged rows: drop the last slot of every odd row on both sides
    g2 = g.copy()
    g2[1::2, -1] = -1
    rows = [r[r >= 0] for r in g2]
    row_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    col = np.concatenate(rows).astype(np.int32)
    b = orc.search_batch(x, codes, lo, hi, 8, g2, entry, q, 10, 32, 32, trace=True, max_hops=200)
    c = orc.search_batch(x, codes, lo, hi, 8, col, entry, q, 10, 32, 32, row_ptr=row_ptr, trace=True,
                         max_hops=200)
    for key in ("ids", "dists", "expanded", "pool_ids", "pool_tau", "n_lp"):
        assert (b[key] == c[key]).all(), key
    a2 = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 32, 32, trace=True, max_hops=200, nthreads=4)
    for key in ("ids", "dists", "expanded", "pool_ids", "pool_tau", "n_lp"):
        assert (a[key] == a2[key]).all(), key


def test_recall_rises_with_ef(orc, c0small):
    x, q, g, lo, hi, codes, entry = c0small
    gt = synth.ground_truth(x, q, 10)
    rec = [synth.recall_at_k(orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, ef, ef)["ids"], gt, 10)
           for ef in (10, 32, 128)]
    assert rec[0] <= rec[1] + 0.01 and rec[1] <= rec[2] + 0.01 and rec[2] > 0.9


def test_underfill_pads(orc):
    # A component with fewer than k reachable nodes: ids -1, dists +inf.
    x = np.random.default_rng(1).standard_normal((6, 4)).astype(np.float32)
    g = np.array([[1, -1], [0, -1], [3, -1], [2, -1], [5, -1], [4, -1]], np.int32)
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, 8, lo, hi)
    r = orc.search_batch(x, codes, lo, hi, 8, g, np.array([0]), x[:1], 4, 4, 4, trace=True)
    assert sorted(r["ids"][0][:2].tolist()) == [0, 1]
    assert list(r["ids"][0][2:]) == [-1, -1] and np.isinf(r["dists"][0][2:]).all()
    assert r["n_hp"][0] == 2


def test_invalid_args(orc, c0small):
    x, q, g, lo, hi, codes, entry = c0small
    with pytest.raises(orc.OracleError):
        orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 5, 5)  # ef < k
    with pytest.raises(orc.OracleError):
        orc.search_batch(x, codes, lo, hi, 8, g, np.array([len(x)]), q, 10, 16, 16)  # entry out of range
    bad = g.copy()
    bad[0, 0] = len(x)
    with pytest.raises(orc.OracleError):
        orc.search_batch(x, codes, lo, hi, 8, bad, entry, q, 10, 16, 16)


def test_c0_fingerprint(orc):
    # Independent cross-check against the survey's own transcription (golden/c0_fingerprint.json).
    f = json.load(open(os.path.join(GOLD, "c0_fingerprint.json")))
    cfg = synth.get_config("C0")
    x = synth.generate_base(cfg)
    q = synth.generate_queries(cfg)
    lo, hi = orc.train_sq(x)
    assert np.allclose(lo[:3], f["lower3"], rtol=0, atol=1e-7) and np.allclose(hi[:3], f["upper3"], rtol=0, atol=1e-7)
    codes = orc.encode_sq(x, 8, lo, hi)
    assert hashlib.sha256(codes.tobytes()).hexdigest()[:16] == f["codes_sha256_16"]
    g = synth.build_graph(x, 32)
    entry = synth.entry_set(cfg.n, cfg.n_seeds)
    r = orc.search_batch(x, codes, lo, hi, 8, g, entry, q, 10, 64, 64, trace=True)
    gt = synth.ground_truth(x, q, 10)
    assert synth.recall_at_k(r["ids"], gt, 10) == pytest.approx(f["recall10"], abs=1e-9)
    assert r["hops"].mean() == pytest.approx(f["mean_hops"], abs=1e-9)
    assert r["n_lp"].mean() == pytest.approx(f["mean_n_lp"], abs=1e-9)
    assert list(r["ids"][0]) == f["query0_top10"]
    assert hashlib.sha256(np.ascontiguousarray(r["ids"], dtype=np.int32).tobytes()).hexdigest()[:16] == \
        f["all_ids_sha256_16"]
    # |V| = the seeds that entered the pool (min(L, |I|), R-10) + every newly visited neighbour
    # (n_lp counts |I| + those)
    v_size = r["n_lp"] - len(entry) + min(64, len(entry))
    assert int(v_size.max()) == f["max_V"]
