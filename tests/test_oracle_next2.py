"""Pins for NEXT-2: the edge filter of Alg. 1 line 8
with per-edge labels L (Alg. 2 prune-based labeling) and the search-time
parameters m_s (degree cap) and alpha_s (label bound).

The paper's worked example (Fig. 6: visit x1, x3, x4) is checked as a hand trace;
its equivalence claim (the filtered search "is equivalent to searching in a graph
constructed with m_c = 3 and alpha_c = 1.2") is checked against a search on the explicitly
materialised subgraph; alpha_s = inf without a cap is the unfiltered search.
"""
import numpy as np
import pytest

import synth


def _subgraph(adj, lab, m_s, alpha_s):
    out = np.full_like(adj, -1)
    for i in range(adj.shape[0]):
        keep = [j for j, l in zip(adj[i], lab[i]) if j >= 0 and l <= alpha_s]
        if m_s > 0:
            keep = keep[:m_s]
        out[i, :len(keep)] = keep
    return out


def test_fig6_worked_example(orc):
    # node 0's neighbours x1..x5 in ascending distance, labels (1.0, 1.4, 1.0, 1.2, 1.0);
    # m_s = 3, alpha_s = 1.2: x2 fails the label, x5 the degree cap -> evaluate x1, x3, x4
    d = 2
    x = np.array([[0, 0], [1, 0], [2, 0], [3, 0], [4, 0], [5, 0]], np.float32)
    adj = np.full((6, 5), -1, np.int32)
    lab = np.full((6, 5), np.inf, np.float32)
    adj[0] = [1, 2, 3, 4, 5]
    lab[0] = [1.0, 1.4, 1.0, 1.2, 1.0]
    lo, hi = np.zeros(d, np.float32), np.full(d, 5.0, np.float32)
    codes = orc.encode_sq(x, 8, lo, hi)
    q = np.array([[0.0, 0.0]], np.float32)
    r = orc.search_batch(x, codes, lo, hi, 8, adj, np.array([0], np.int32), q, 4, 8, 8, "l2", trace=True,
                         max_hops=8, labels=lab, m_s=3, alpha_s=1.2)
    assert r["n_lp"][0] == 1 + 3
    assert sorted(r["pool_ids"][0][:4]) == [0, 1, 3, 4] and (r["pool_ids"][0][4:] == -1).all()
    assert list(r["expanded"][0][:4]) == [0, 1, 3, 4]


@pytest.fixture(scope="module")
def labelled():
    cfg = synth.get_config("C0").scaled(n=1500, nq=20, clusters=3, n_seeds=48)
    w = synth.make_workload(cfg, device="cpu", gt=False)
    adj, lab = synth.build_labelled_graph(w["x"], 24)
    return w, adj, lab


def test_labels_follow_alg2(labelled):
    w, adj, lab = labelled
    valid = adj >= 0
    assert set(np.unique(lab[valid]).tolist()) <= set(np.float32(synth.graph.ALPHAS).tolist())
    assert np.isinf(lab[~valid]).all()
    # the smallest pruning rate keeps the nearest neighbour of every node
    assert (lab[:, 0] == 1.0).all()


@pytest.mark.parametrize("m_s,alpha_s", [(0, np.inf), (24, 2.0), (12, 1.2), (6, 1.0), (0, 1.4), (5, 3.0)])
def test_filtered_search_equals_search_on_subgraph(orc, labelled, m_s, alpha_s):
    w, adj, lab = labelled
    x, q = w["x"], w["q"]
    lo, hi = orc.train_sq(x)
    codes = orc.encode_sq(x, 8, lo, hi)
    a = orc.search_batch(x, codes, lo, hi, 8, adj, w["entry"], q, 10, 40, 40, "l2", trace=True, max_hops=80,
                         labels=lab, m_s=m_s, alpha_s=alpha_s)
    b = orc.search_batch(x, codes, lo, hi, 8, _subgraph(adj, lab, m_s, alpha_s), w["entry"], q, 10, 40, 40, "l2",
                         trace=True, max_hops=80)
    for key in ("hops", "expanded", "n_lp", "pool_ids", "pool_tau", "ids", "dists"):
        assert np.array_equal(a[key], b[key]), key
    if m_s == 0 and np.isinf(alpha_s):  # no filter at all
        c = orc.search_batch(x, codes, lo, hi, 8, adj, w["entry"], q, 10, 40, 40, "l2", trace=True, max_hops=80)
        for key in ("expanded", "pool_ids", "ids"):
            assert np.array_equal(a[key], c[key]), key
