"""Input-preparation checks (synth/): seeded determinism, shapes, the RNG prune + fill rule
(SURVEY AMB-21, PAPER.md:544 at alpha = 1) on a hand example, and numpy/torch builder agreement."""
import numpy as np
import pytest

import synth


def test_generators_deterministic_and_shaped():
    for name in ("C0", "C1", "C2", "C3", "C4"):
        cfg = synth.get_config(name).scaled(n=2000, nq=16)
        a = synth.generate_base(cfg)
        b = synth.generate_base(cfg)
        assert a.shape == (2000, cfg.d) and a.dtype == np.float32 and (a == b).all()
        q = synth.generate_queries(cfg)
        assert q.shape == (16, cfg.d) and np.isfinite(q).all()
        if cfg.kind == "sphere":
            assert np.allclose(np.linalg.norm(a, axis=1), 1, atol=1e-5)
        if cfg.kind == "gamma_int":
            assert (a == np.rint(a)).all() and a.min() >= 0 and a.max() <= 255


def test_entry_set():
    e = synth.entry_set(1000, 64)
    assert len(np.unique(e)) == 64 and (np.diff(e) > 0).all() and e.min() >= 0 and e.max() < 1000


def test_rng_prune_fill_hand_example():
    # points on a line 0,1,2,3,10: node 0's candidates by distance are 1,2,3,4; 1 is kept, 2,3,4 are
    # pruned by 1 (d(j,1) <= d(0,j)); fill to R=2 with the nearest pruned -> [1, 2].
    x = np.array([[0.0], [1.0], [2.0], [3.0], [10.0]], np.float32)
    g = synth.build_graph(x, 2, kk=4)
    assert list(g[0]) == [1, 2]
    # node 4: candidates 3 (49), 2 (64), 1 (81), 0 (100): keep 3; 2 pruned (d(2,3)=1 <= 64); ... -> [3, 2]
    assert list(g[4]) == [3, 2]


def test_torch_builder_matches_numpy_on_cpu():
    torch = pytest.importorskip("torch")
    cfg = synth.get_config("C0").scaled(n=1500, nq=4)
    x = synth.generate_base(cfg)
    cand_np = synth.knn_candidates(x, 32)
    from synth.graph import _knn_torch, _prune_torch
    xt = torch.as_tensor(x)
    cand_t = _knn_torch(xt, 32).numpy()
    assert (cand_np == cand_t).mean() > 0.999
    g_np = synth.rng_prune_fill(x, cand_np, 16)
    g_t = _prune_torch(xt, torch.as_tensor(cand_np), 16).numpy()
    assert (g_np == g_t).all()


def test_ground_truth_and_recall():
    x = np.array([[0.0, 0], [1, 0], [0, 2], [5, 5]], np.float32)
    q = np.array([[0.1, 0.0]], np.float32)
    gt = synth.ground_truth(x, q, 3)
    assert list(gt[0]) == [0, 1, 2]
    assert synth.recall_at_k(np.array([[0, 2, -1]]), gt, 3) == pytest.approx(2 / 3)
    gti = synth.ground_truth(x, q, 2, metric="ip")
    assert list(gti[0]) == [3, 1]
