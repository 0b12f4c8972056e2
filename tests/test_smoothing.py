"""Smoothing-threshold search on the GPU against golden
vectors produced by the reference itself (tests/golden/make_golden_smoothing.py,
smoothing.py:88-155, numerics.py:94-109)."""

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "smoothing_cases.npz")


def _cases():
    d = np.load(GOLD)
    for i in range(int(d["n_cases"])):
        m, k, n, g = (int(v) for v in d[f"c{i}_meta"])
        yield dict(i=i, m=m, k=k, n=n, g=g, pg=bool(d[f"c{i}_pg"]), x=d[f"c{i}_x"], w=d[f"c{i}_w"],
                   exact=d[f"c{i}_exact"], cand=d[f"c{i}_cand"], sigma=float(d[f"c{i}_sigma"]), sel=d[f"c{i}_sel"],
                   s=d[f"c{i}_s"], obj=float(d[f"c{i}_obj"]), grid=int(d[f"c{i}_grid"]))


def _seq_matmul(a, b):
    """numerics.py:94-109 restated (test-side check of the fixture)."""
    out = np.zeros((a.shape[0], b.shape[1]))
    for k in range(a.shape[1]):
        out += a[:, k:k + 1] * b[k:k + 1, :]
    return out


def test_golden_smoothing_fixture_consistent():
    """The fixture is self-consistent: its exact product is the sequential-k
    product, the plan's objective is the first minimum of the candidates, and
    s = max/sigma on exactly the selected channels."""
    for c in _cases():
        assert np.array_equal(_seq_matmul(c["x"], c["w"]).view(np.uint64), c["exact"].view(np.uint64))
        cand = c["cand"]
        assert c["obj"] == cand.min()
        mx = np.abs(c["x"]).max(axis=0)
        s = np.where(c["sel"], mx / c["sigma"], 1.0)
        assert np.array_equal(s.view(np.uint64), c["s"].view(np.uint64))


@pytest.mark.gpu
def test_gpu_matmul_ref_bit_exact():
    import torch

    import paper_2406_09904_b200 as Q

    for c in _cases():
        got = Q.matmul_ref(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["w"]).cuda()).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), c["exact"].view(np.uint64)), c["i"]
    rng = np.random.default_rng(5)
    for (m, k, n) in [(1, 1, 1), (65, 17, 129), (3, 0, 5), (70, 300, 2)]:
        a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
        got = Q.matmul_ref(a, b).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), _seq_matmul(a, b).view(np.uint64)), (m, k, n)
    with pytest.raises(Q.ShapeError):
        Q.matmul_ref(np.ones((2, 3)), np.ones((4, 2)))


@pytest.mark.gpu
def test_gpu_smoothing_objective_candidates():
    """Every candidate's objective within 1e-12 (relative) of the reference's:
    the error matrices are bit-identical, only the final sum's order differs."""
    import paper_2406_09904_b200 as Q

    for c in _cases():
        spec = Q.QuantSpec("per-group", c["g"]) if c["pg"] else Q.QuantSpec("per-channel")
        mx = Q.channel_maxima(c["x"])
        xmax = float(mx.max())
        got = [Q.smoothing_objective(c["x"], c["w"], np.ones(c["k"]), spec)]
        for i in range(c["grid"], 0, -1):
            sigma = (i / c["grid"]) * xmax
            got.append(Q.smoothing_objective(c["x"], c["w"],
                                             Q.smoothing_vector(mx, Q.select_outlier_channels(mx, sigma), sigma), spec))
        np.testing.assert_allclose(np.array(got), c["cand"], rtol=1e-12, atol=0)


@pytest.mark.gpu
def test_gpu_search_sigma_matches_reference_plan():
    import paper_2406_09904_b200 as Q

    for c in _cases():
        spec = Q.QuantSpec("per-group", c["g"]) if c["pg"] else Q.QuantSpec("per-channel")
        plan = Q.search_sigma(c["x"], c["w"], spec, grid_points=c["grid"])
        assert plan.sigma == c["sigma"], c["i"]
        assert plan.selected == tuple(int(t) for t in np.flatnonzero(c["sel"])), c["i"]
        assert np.array_equal(np.asarray(plan.s).view(np.uint64), c["s"].view(np.uint64)), c["i"]
        assert abs(plan.objective - c["obj"]) <= 1e-12 * c["obj"], c["i"]
    with pytest.raises(Q.DataError):
        Q.search_sigma(np.ones((2, 4)), np.ones((4, 2)), Q.QuantSpec("per-channel"), grid_points=1)
    z = Q.search_sigma(np.zeros((2, 4)), np.ones((4, 2)), Q.QuantSpec("per-channel"), grid_points=4)
    assert z.selected == () and z.sigma == 1.0


@pytest.mark.gpu
@pytest.mark.parametrize("g", [0, 64])
def test_gpu_search_sigma_random_vs_oracle(g):
    """Seeded random calibration sets (outlier channels, a zero channel) against
    the oracle restatement (oracle/qqq_oracle.py search_sigma, pinned to the
    reference goldens): same plan, objective within 1e-12."""
    import paper_2406_09904_b200 as Q
    from oracle import qqq_oracle as O

    rng = np.random.default_rng(100 + g)
    for (m, k, n) in [(8, 128, 32), (20, 192, 24)]:
        x = rng.standard_normal((m, k))
        x[:, rng.choice(k, 6, replace=False)] *= rng.uniform(8.0, 60.0, 6)
        x[:, 3] = 0.0
        w = rng.standard_normal((k, n)) * 0.1
        sigma, sel, s, obj = O.search_sigma(x, w, g, grid_points=10)
        spec = Q.QuantSpec("per-group", g) if g else Q.QuantSpec("per-channel")
        plan = Q.search_sigma(x, w, spec, grid_points=10)
        assert plan.sigma == sigma and plan.selected == sel, (m, k, n)
        assert np.array_equal(np.asarray(plan.s).view(np.uint64), s.view(np.uint64))
        assert abs(plan.objective - obj) <= 1e-12 * obj
