"""Pins for the oracle's SQ training / encoding (rows a1, a2 of SURVEY.md §8) and tau_l / tau_h.

Each check is tied to something other than the oracle itself: hand values (tests/golden,
with citations), the textbook decomposition identity of PAPER.md:649, exact rational
arithmetic, and closed-form properties of a uniform (2^b - 1)-step quantiser (App. G,
PAPER.md:1238).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _encode_pins():
    rows = []
    for line in open(os.path.join(GOLD, "sq_encode_pins.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        b, lo, hi, v, e = line.split()
        rows.append((int(b), float(lo), float(hi), float(v), int(e)))
    return rows


@pytest.mark.parametrize("bits,lo,hi,v,expected", _encode_pins())
def test_encode_hand_pins(orc, bits, lo, hi, v, expected):
    code = orc.encode_sq(np.array([[v]], np.float32), bits, [lo], [hi])
    assert int(code[0, 0]) & (0xFF if bits == 8 else 0x0F) == expected


def test_sq4_packing_low_nibble_first(orc):
    # SPEC.md:110 / :172: two codes per byte, low nibble first.  [1,2,15,0,7,8] -> 0x21 0x0F 0x87
    x = np.array([[1, 2, 15, 0, 7, 8]], np.float32)
    c = orc.encode_sq(x, 4, np.zeros(6), np.full(6, 15.0))
    assert list(c[0]) == [0x21, 0x0F, 0x87]
    # odd d: last high nibble is 0
    c = orc.encode_sq(np.array([[1, 2, 3]], np.float32), 4, np.zeros(3), np.full(3, 15.0))
    assert list(c[0]) == [0x21, 0x03]
    assert orc.code_bytes(3, 4) == 2 and orc.code_bytes(960, 4) == 480 and orc.code_bytes(128, 8) == 128


def test_train_min_max(orc):
    # per-dimension min/max over the base (BASELINE.json config 0)
    x = np.array([[0, 5, 0.5], [1, -2, 0.5], [2, 7, 0.5], [3, 1, 0.5]], np.float32)
    lo, hi = orc.train_sq(x)
    assert list(lo) == [0, -2, 0.5] and list(hi) == [3, 7, 0.5]
    # constant column encodes to 0 everywhere
    c = orc.encode_sq(x, 8, lo, hi)
    assert (c[:, 2] == 0).all()
    # {0,1,2,3} -> [0, 3], codes 0, 85, 170, 255 (exact thirds of 255)
    assert list(c[:, 0]) == [0, 85, 170, 255]
    with pytest.raises(orc.OracleError):
        orc.train_sq(np.array([[np.nan]], np.float32))


def test_train_negative_zero_canonical(orc):
    lo, hi = orc.train_sq(np.array([[-0.0], [0.0]], np.float32))
    assert np.signbit(lo[0]) == False and lo[0] == 0.0 and hi[0] == 0.0  # noqa: E712


@pytest.mark.parametrize("bits", [4, 8])
def test_encode_round_trip_bound_and_monotone(orc, bits):
    # Closed form of a uniform quantiser with 2^b - 1 steps over [l, u] (App. G):
    # |decode(encode(v)) - clamp(v)| <= step / 2 (+ fp32 slack), encode non-decreasing in v.
    rng = np.random.default_rng(5)
    d = 16
    lo = rng.uniform(-2, 0, d).astype(np.float32)
    hi = (lo + rng.uniform(0.1, 3, d)).astype(np.float32)
    x = rng.uniform(lo - 0.5, hi + 0.5, (500, d)).astype(np.float32)
    x.sort(axis=0)
    c = orc.encode_sq(x, bits, lo, hi)
    if bits == 4:
        full = np.empty((500, d), np.int64)
        full[:, 0::2] = c & 0x0F
        full[:, 1::2] = c >> 4
    else:
        full = c.astype(np.int64)
    levels = (1 << bits) - 1
    step = (hi.astype(np.float64) - lo) / levels
    dec = lo + full * step
    clamped = np.clip(x.astype(np.float64), lo, hi)
    assert (np.abs(dec - clamped) <= step / 2 * (1 + 1e-5) + 1e-6).all()
    assert (np.diff(full, axis=0) >= 0).all()
    assert full.min() == 0 and full.max() == levels


def test_integer_closed_form_c1(orc):
    # with l = 0 and u = 255 in every dimension (C1's integer data),
    # SQ8 is lossless: code == value for every element.
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, (300, 128)).astype(np.float32)
    x[0] = 0
    x[1] = 255
    lo, hi = orc.train_sq(x)
    assert (lo == 0).all() and (hi == 255).all()
    assert (orc.encode_sq(x, 8, lo, hi) == x.astype(np.uint8)).all()


def _tau_pins():
    out = []
    for line in open(os.path.join(GOLD, "tau_l_pins.txt")):
        if line.startswith("#") or not line.strip():
            continue
        head, q, lo, hi, code, exp = [s.strip() for s in line.split("|")]
        metric, bits = head.split()
        f = lambda s: [float(t) for t in s.split()]  # noqa: E731
        out.append((metric, int(bits), f(q), f(lo), f(hi), [int(t) for t in code.split()], int(exp)))
    return out


@pytest.mark.parametrize("metric,bits,q,lo,hi,code,expected", _tau_pins())
def test_tau_l_hand_pins(orc, metric, bits, q, lo, hi, code, expected):
    assert orc.tau_l(q, np.array(code, np.uint8), bits, lo, hi, metric) == expected


def test_tau_l_l2_decomposition_identity(orc):
    # ||b - q||^2 = ||b||^2 + ||q||^2 - 2 b.q, exact on integers.
    rng = np.random.default_rng(11)
    for bits in (8, 4):
        d = 37
        lo, hi = np.zeros(d, np.float32), np.full(d, float((1 << bits) - 1), np.float32)
        for _ in range(20):
            qv = rng.integers(0, 1 << bits, d)
            bv = rng.integers(0, 1 << bits, d)
            code = orc.encode_sq(bv[None].astype(np.float32), bits, lo, hi)[0]
            expect = int((bv * bv).sum() + (qv * qv).sum() - 2 * (bv * qv).sum())
            assert orc.tau_l(qv.astype(np.float32), code, bits, lo, hi, "l2") == expect


def test_ip_weights_rank_like_decoded_ip(orc):
    # R-7: w_d is 127 * a_d / s rounded; -sum w c orders codes like -q.x_hat (decoded IP)
    # up to the rounding of w.  Pin: exact proportionality when a_d/s*127 are integers.
    lo = np.zeros(4, np.float32)
    hi = np.ones(4, np.float32)
    q = np.array([127, -127, 0, 63.5 * 2], np.float32)  # a = q, s = 127 -> w = 127, -127, 0, 127
    assert list(orc.ip_weights(q, lo, hi)) == [127, -127, 0, 127]
    assert list(orc.ip_weights(np.zeros(4, np.float32), lo, hi)) == [0, 0, 0, 0]


def _exact_l2(q, x):
    return sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(q, x))


def _exact_ip(q, x):
    return -sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(q, x))


def test_tau_h_correctly_rounded(orc):
    # R-16: fp64 accumulation rounded once to fp32 equals the correctly rounded fp32 of
    # the exact real value (checked with rational arithmetic) on random inputs.
    rng = np.random.default_rng(7)
    for d in (1, 3, 128, 200):
        for _ in range(10):
            q = rng.standard_normal(d).astype(np.float32)
            x = rng.standard_normal(d).astype(np.float32)
            assert orc.tau_h(q, x, "l2") == np.float32(float(_exact_l2(q, x)))
            assert orc.tau_h(q, x, "ip") == np.float32(float(_exact_ip(q, x)))
    # (1,2,3) vs (4,6,8) -> 50
    assert orc.tau_h(np.array([1, 2, 3], np.float32), np.array([4, 6, 8], np.float32)) == 50.0
