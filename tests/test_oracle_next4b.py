"""Pins for NEXT-4b (second half): QLP early termination at a checkpoint
(§4.3: "after traversing certain hops in the graph, we employ the decision tree
along with the current features to determine whether the candidate size should be reduced").
The GBDT is replaced by a fixed decision stump on one integer feature (R-28):
0 = points scanned (n_lp), 1 = sum of the 5 best tau_l, 2 = tau_l(k-th) - tau_l(best).

Pinned by: QLP off == plain search; a shrink to ef_low = ef when L = ef changes nothing; the
first h expansions are those of the plain search; and at the checkpoint before the first
expansion the decision flips exactly at the feature value computed by brute force over the
entry set (numpy integer arithmetic on the pinned SQ8 codes).
"""
import numpy as np
import pytest

import synth


@pytest.fixture(scope="module")
def small():
    cfg = synth.get_config("C0").scaled(n=3000, nq=24, n_seeds=48)
    return synth.make_workload(cfg, device="cpu", gt=False)


def _run(orc, w, ef, k=10, rr=0, qlp=None, trace=True):
    x, q = w["x"], w["q"]
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, 8, lo, hi)
    return orc.search_batch(x, codes, lo, hi, 8, w["graph"], w["entry"], q, k, ef, rr, trace=trace,
                            max_hops=256, qlp=qlp)


def _same(a, b, keys=("ids", "dists", "hops", "n_lp", "n_hp", "expanded", "pool_ids", "pool_tau")):
    for key in keys:
        assert np.array_equal(a[key], b[key]), key


def test_qlp_off_is_plain_search(orc, small):
    _same(_run(orc, small, 40), _run(orc, small, 40, qlp=(0, 0, 0, 0)))
    # a stump that never fires is the plain search too
    _same(_run(orc, small, 40), _run(orc, small, 40, qlp=(5, 20, 0, -1)))


def test_shrink_to_the_same_size_changes_nothing(orc, small):
    for feat in (0, 1, 2):
        _same(_run(orc, small, 32), _run(orc, small, 32, qlp=(7, 32, feat, 1 << 40)))


@pytest.mark.parametrize("h", [1, 6, 20])
def test_expansions_before_the_checkpoint_are_the_plain_search(orc, small, h):
    base = _run(orc, small, 48)
    o = _run(orc, small, 48, qlp=(h, 12, 0, 1 << 40))
    for i in range(len(small["q"])):
        n = min(h, base["hops"][i])
        assert np.array_equal(o["expanded"][i, :n], base["expanded"][i, :n])
    # the shrink evicts: R' drops to ef_low for every query that reached the checkpoint
    reached = base["hops"] >= h
    assert (o["n_hp"][reached] == 12).all()


@pytest.mark.parametrize("feat", [1, 2])
def test_decision_flips_at_the_brute_force_feature_value(orc, small, feat):
    """Checkpoint before the first expansion: the pool is the top-L of the entry set by
    (tau_l, id), so the feature follows from brute force over the seeds."""
    x, q, entry = small["x"], small["q"], np.unique(small["entry"])
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, 8, lo, hi).astype(np.int64)
    qc = orc.encode_sq(q, 8, lo, hi).astype(np.int64)
    k, ef = 10, 40
    base = _run(orc, small, ef, k=k)
    for i in range(len(q)):
        tau = ((codes[entry] - qc[i]) ** 2).sum(1)
        order = np.lexsort((entry, tau))[:ef]
        t = tau[order]
        f = int(t[:5].sum()) if feat == 1 else int(t[k - 1] - t[0])
        qi = q[i:i + 1]
        one = dict(x=x, q=qi, graph=small["graph"], entry=small["entry"])
        fires = _run(orc, one, ef, k=k, qlp=(0, 16, feat, f))
        holds = _run(orc, one, ef, k=k, qlp=(0, 16, feat, f - 1))
        assert fires["n_hp"][0] == 16 and fires["pool_ids"][0, 16:].max() == -1  # shrunk
        for key in ("ids", "hops", "expanded", "pool_ids", "n_hp"):
            assert np.array_equal(holds[key][0], base[key][i]), key


def test_invalid_qlp_is_rejected(orc, small):
    for qlp in [(1, 5, 0, 0), (1, 50, 0, 0), (-1, 20, 0, 0), (1, 20, 3, 0)]:  # ef_low < k, > ef, hop < 0, feature
        with pytest.raises(orc.OracleError):
            _run(orc, small, 40, qlp=qlp)
