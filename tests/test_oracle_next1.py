"""Pins for NEXT-1: truncated SQ training (App. G)
and the integer-weighted code-space L2 tau_l.

Truncation: hand-sorted order statistics, SPEC.md's worked example, the q = 1
special case (= plain min/max training), and the operational claim of App. G (a planted
outlier no longer spoils the resolution of the other values).  Weights: hand values, the
half-away rounding boundary, the int32 cap, and the special case of equal ranges where
the weighted distance is W times the plain one (so the whole search trace is unchanged).
"""
import numpy as np
import pytest


# ----------------------------------------------------------------------------- truncated SQ
def test_quantile_hand_order_statistics(orc):
    # n = 5, q = 0.75: indices floor(0.25 * 4) = 1 and floor(0.75 * 4) = 3 of the sorted column
    x = np.array([[5, -2], [1, 7], [4, 0], [2, 3], [3, 3]], np.float32)
    lo, hi = orc.train_sq_quantile(x, 0.75)
    assert list(lo) == [2.0, 0.0] and list(hi) == [4.0, 3.0]


def test_quantile_spec_outlier_example(orc):
    # 99 values in [0, 0.29] plus an outlier 1.0, q = 0.99 -> upper is element
    # floor(0.99 * 99) = 98 of the sorted sequence, i.e. the largest regular value
    vals = np.linspace(0.0, 0.29, 99, dtype=np.float32)
    col = np.concatenate([vals, [np.float32(1.0)]])
    rng = np.random.default_rng(0)
    col = col[rng.permutation(100)]
    lo, hi = orc.train_sq_quantile(col[:, None], 0.99)
    assert hi[0] == vals.max() and lo[0] == vals.min()


def test_quantile_one_is_min_max_and_constant_dimension(orc):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((257, 9)).astype(np.float32)
    x[:, 4] = 0.5  # constant dimension
    lq, hq = orc.train_sq_quantile(x, 1.0)
    lm, hm = orc.train_sq(x)
    assert np.array_equal(lq, lm) and np.array_equal(hq, hm)
    lo, hi = orc.train_sq_quantile(x, 0.9)
    assert lo[4] == hi[4] == np.float32(0.5)
    assert (lo <= hi).all()


def test_quantile_rejects_bad_q(orc):
    x = np.zeros((4, 2), np.float32)
    for q in (0.5, 1.5, 0.0):
        with pytest.raises(orc.OracleError):
            orc.train_sq_quantile(x, q)


def test_truncation_improves_resolution_with_outliers(orc):
    # App. G: "using the absolute maximum ... would leave 70% of the quantization intervals
    # underutilized".  One planted outlier per dimension: the mean round-trip error of the
    # regular values is strictly smaller with q = 0.99 than with q = 1.
    rng = np.random.default_rng(2)
    n, d = 1000, 8
    x = rng.uniform(0.0, 0.3, (n, d)).astype(np.float32)
    out_rows = rng.choice(n, d, replace=False)
    x[out_rows, np.arange(d)] = 1.0
    regular = np.ones((n, d), bool)
    regular[out_rows, np.arange(d)] = False

    def err(lo, hi, bits):
        c = orc.encode_sq(x, bits, lo, hi).astype(np.float64)
        if bits == 4:  # unpack low nibble first
            c = np.stack([c.astype(np.int64) & 15, c.astype(np.int64) >> 4], -1).reshape(n, -1)[:, :d]
        dec = lo + c * ((hi - lo) / (2 ** bits - 1)).astype(np.float64)
        return np.abs(dec - np.clip(x, lo, hi))[regular].mean()

    for bits in (4, 8):
        lq, hq = orc.train_sq_quantile(x, 0.99)
        lm, hm = orc.train_sq(x)
        assert (hq < 0.31).all() and (hm == 1.0).all()
        assert err(lq, hq, bits) < 0.5 * err(lm, hm, bits)


# ----------------------------------------------------------------------------- weighted L2
def test_l2w_weights_hand_values(orc):
    W, w = orc.l2w_weights(np.zeros(3, np.float32), np.array([1, 2, 0], np.float32), 4)
    # r^2 = [1, 4, 0], max 4: round(8192 * [1/4, 1, 0])
    assert W == 8192 and list(w) == [2048, 8192, 0]
    # half-away rounding at an exact .5: r = 2^-7 against r = 1 gives 8192 * 2^-14 = 0.5 -> 1
    W, w = orc.l2w_weights(np.zeros(2, np.float32), np.array([2.0 ** -7, 1.0], np.float32), 4)
    assert list(w) == [1, 8192]


def test_l2w_weight_cap_keeps_int32(orc):
    # W = min(8192, floor((2^31 - 1) / (d (2^b - 1)^2)))
    W, _ = orc.l2w_weights(np.zeros(960, np.float32), np.ones(960, np.float32), 4)
    assert W == 8192
    W, _ = orc.l2w_weights(np.zeros(128, np.float32), np.ones(128, np.float32), 8)
    assert W == (2 ** 31 - 1) // (128 * 255 * 255) == 258
    assert W * 128 * 255 * 255 < 2 ** 31


def test_l2w_tau_hand_value(orc):
    # lower 0, upper [1, 2, 0] (SQ4): query [1.0, 0.0, x] -> codes [15, 0, 0];
    # base [0.0, 2.0, x] -> codes [0, 15, 0]; tau = 2048 * 15^2 + 8192 * 15^2 + 0
    lo, hi = np.zeros(3, np.float32), np.array([1, 2, 0], np.float32)
    code = orc.encode_sq(np.array([[0.0, 2.0, 0.7]], np.float32), 4, lo, hi)[0]
    t = orc.tau_l(np.array([1.0, 0.0, -3.0], np.float32), code, 4, lo, hi, "l2w")
    assert t == 2048 * 225 + 8192 * 225 == 2304000


@pytest.mark.parametrize("bits", [4, 8])
def test_l2w_equal_ranges_is_scaled_l2(orc, bits):
    # equal ranges: every w_j = W, so tau_l^w = W * tau_l and the traversal is unchanged
    import synth
    rng = np.random.default_rng(3)
    n, d = 600, 24
    x = rng.uniform(0, 1, (n, d)).astype(np.float32)
    x[0], x[1] = 0.0, 1.0  # every dimension spans exactly [0, 1]
    lo, hi = orc.train_sq(x)
    assert (lo == 0).all() and (hi == 1).all()
    W, w = orc.l2w_weights(lo, hi, bits)
    assert (w == W).all()
    codes = orc.encode_sq(x, bits, lo, hi)
    q = rng.uniform(0, 1, (7, d)).astype(np.float32)
    for i in range(3):
        assert orc.tau_l(q[i], codes[i], bits, lo, hi, "l2w") == W * orc.tau_l(q[i], codes[i], bits, lo, hi, "l2")
    g = synth.build_graph(x, 10)
    entry = np.array([5, 77, 300], np.int32)
    a = orc.search_batch(x, codes, lo, hi, bits, g, entry, q, 5, 20, 20, "l2", trace=True, max_hops=60)
    b = orc.search_batch(x, codes, lo, hi, bits, g, entry, q, 5, 20, 20, "l2w", trace=True, max_hops=60)
    for key in ("hops", "expanded", "pool_ids", "n_lp", "ids", "dists"):
        assert np.array_equal(a[key], b[key]), key
    has = a["pool_ids"] >= 0
    assert np.array_equal(b["pool_tau"][has].astype(np.int64), W * a["pool_tau"][has].astype(np.int64))
