"""Pins for NEXT-3: an exact early stop of the selective re-rank
(Alg. 1 line 18; §5.3 P:683-685 "adapt re-ranking scope"; SPEC's error-bound rule S:360).

The bound (R-27): for L2 with every base value inside the trained range,
tau_h >= D_min^2 * max(0, tau_l - 2 sqrt(d tau_l)) (with fp margins).  Checked against exact
tau_h on random and adversarial pairs (values on the edges of their quantisation cells);
the adaptive re-rank returns exactly the full re-rank's ids and distances with fewer tau_h.
"""
import numpy as np
import pytest

import synth


def test_bound_hand_value(orc):
    lo, hi = np.zeros(4, np.float32), np.full(4, 255.0, np.float32)  # SQ8 step 1
    lb = orc.rerank_lower_bound(100, 4, lo, hi, 8)
    assert abs(lb - (100 - 2.0002 * 20) * (1 - 1e-5)) < 1e-9
    assert orc.rerank_lower_bound(10, 4, lo, hi, 8) == 0.0  # below 4 d: no information
    # the smallest non-constant step is used (a constant dimension is ignored)
    lo2, hi2 = np.zeros(3, np.float32), np.array([15.0, 30.0, 0.0], np.float32)
    assert abs(orc.rerank_lower_bound(1000, 3, lo2, hi2, 4) - (1000 - 2.0002 * np.sqrt(3000)) * (1 - 1e-5)) < 1e-6


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("d", [8, 64, 128])
def test_bound_holds_on_random_and_edge_pairs(orc, bits, d):
    rng = np.random.default_rng(d + bits)
    n = 300
    x = rng.uniform(-2, 3, (n, d)).astype(np.float32) * rng.uniform(0.1, 2, d).astype(np.float32)
    lo, hi = orc.train_sq(x)
    levels = 2 ** bits - 1
    step = (hi.astype(np.float64) - lo) / levels
    # push half of the values to the edge of their quantisation cell (worst case for the bound)
    c = np.rint((x - lo) / step)
    edge = lo + (c + rng.choice([-0.4999, 0.4999], x.shape)) * step
    x = np.where(rng.random(x.shape) < 0.5, np.clip(edge, lo, hi), x).astype(np.float32)
    codes = orc.encode_sq(x, bits, lo, hi)
    qs = np.concatenate([rng.uniform(-3, 4, (20, d)), x[:20] + 0.01], 0).astype(np.float32)  # incl. out of range
    worst = np.inf
    for q in qs:
        for i in range(0, n, 3):
            tl = orc.tau_l(q, codes[i], bits, lo, hi, "l2")
            th = float(orc.tau_h(q, x[i], "l2"))
            lb = orc.rerank_lower_bound(tl, d, lo, hi, bits)
            assert th >= lb, (tl, th, lb)
            if lb > 0:
                worst = min(worst, th / lb)
    assert worst >= 1.0


@pytest.mark.parametrize("bits", [8, 4])
def test_adaptive_rerank_is_exact(orc, bits):
    cfg = synth.get_config("C1").scaled(n=4000, nq=40, clusters=4, n_seeds=64)
    w = synth.make_workload(cfg, device="cpu")
    x, q, g, entry = w["x"].copy(), w["q"], w["graph"], w["entry"]
    x[0], x[1] = 0.0, 255.0  # every dimension spans [0, 255], as at full-size C1 (uniform step)
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, bits, lo, hi)
    a = orc.search_batch(x, codes, lo, hi, bits, g, entry, q, 10, 64, 64, "l2", trace=True)
    b = orc.search_batch(x, codes, lo, hi, bits, g, entry, q, 10, 64, 64, "l2", trace=True, adaptive=True)
    assert np.array_equal(a["ids"], b["ids"]) and np.array_equal(a["dists"], b["dists"])
    assert np.array_equal(a["pool_ids"], b["pool_ids"])
    assert (b["n_hp"] <= a["n_hp"]).all() and ((b["n_hp"] % 4 == 0) | (b["n_hp"] == a["n_hp"])).all()
    if bits == 8:  # the bound does cut the re-rank on C1-shaped data (uniform step 1)
        assert b["n_hp"].mean() < a["n_hp"].mean(), (b["n_hp"].mean(), a["n_hp"].mean())
        assert (b["n_hp"] < a["n_hp"]).any()


def test_adaptive_rejects_ip(orc):
    cfg = synth.get_config("C0").scaled(n=500, nq=3, clusters=2, n_seeds=8)
    w = synth.make_workload(cfg, device="cpu", gt=False)
    lo, hi = orc.train_sq(w["x"])
    codes = orc.encode_sq(w["x"], 8, lo, hi)
    with pytest.raises(orc.OracleError):
        orc.search_batch(w["x"], codes, lo, hi, 8, w["graph"], w["entry"], w["q"], 5, 16, 16, "ip", adaptive=True)
