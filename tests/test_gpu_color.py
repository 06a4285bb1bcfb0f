"""Colour transfer on the device (csrc/kmeans.cuh + the solvers) against the
oracle (binding.kmeans, oracle/color_transfer.py) and the reference's own
criteria (test_apps.cpp:38-160).

k-means: same k-means++ picks (same std::mt19937_64 draws), centroids equal to
rounding (cluster sums are chunk-ordered on the device, sequential in the
oracle), identical assignments and weights."""
import numpy as np
import pytest

from oracle import binding
from oracle import color_transfer as ct
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu


def cloud(seed, n):
    return np.random.default_rng(seed).uniform(0.0, 1.0, (n, 3))


@pytest.mark.parametrize("n,k,seed", [(6, 6, 7), (500, 8, 11), (5000, 16, 3), (262144, 64, 21)])
def test_kmeans_matches_oracle(ctx, n, k, seed):
    pts = cloud(100 + seed, n)
    if n == 262144:  # a 512 x 512 "image": 8-bit colours
        pts = np.floor(pts * 255.0) / 255.0
    g = pot.kmeans_quantize(pts, k, seed, ctx=ctx)
    C, W, A, _ = binding.kmeans(pts, k, seed)
    np.testing.assert_allclose(g.centroids, C, rtol=0, atol=1e-12)
    assert np.array_equal(g.assignments, A)
    np.testing.assert_array_equal(g.weights, W)


def test_kmeans_reference_cases(ctx):
    pts = cloud(61, 6)  # :38-52
    h = pot.kmeans_quantize(pts, 6, 7, ctx=ctx)
    assert np.max(np.abs(h.weights - 1.0 / 6.0)) <= 1e-15
    for i in range(6):
        assert np.min(np.linalg.norm(h.centroids - pts[i], axis=1)) <= 1e-12
    rng = np.random.default_rng(62)  # :54-80
    pts = np.vstack([0.1 + rng.normal(0, 0.01, (100, 3)), 0.9 + rng.normal(0, 0.01, (100, 3))])
    h = pot.kmeans_quantize(pts, 2, 3, ctx=ctx)
    a, b = pts[:100].mean(axis=0), pts[100:].mean(axis=0)
    first, second = (a, b) if np.linalg.norm(h.centroids[0] - a) < np.linalg.norm(h.centroids[0] - b) else (b, a)
    assert np.linalg.norm(h.centroids[0] - first) <= 1e-3 and np.linalg.norm(h.centroids[1] - second) <= 1e-3
    with pytest.raises(pot.PotError) as e:  # :82-87
        pot.kmeans_quantize(cloud(63, 4), 5, 1, ctx=ctx)
    assert e.value.code == pot.ErrorCode.InvalidArgument
    with pytest.raises(pot.PotError) as e:
        pot.kmeans_quantize(np.zeros((0, 3)), 1, 1, ctx=ctx)
    assert e.value.code == pot.ErrorCode.EmptyInput


def test_barycentric_projection_rules():  # :89-124 (host glue of the API)
    plan = np.array([[0.2, 0.2], [0.0, 0.0]])
    src = np.array([[0.3, 0.3, 0.3], [0.9, 0.1, 0.5]])
    tgt = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]])
    out = pot.barycentric_projection(plan, src, tgt)
    assert np.linalg.norm(out[0] - 0.5) <= 1e-15 and np.array_equal(out[1], src[1])
    rng = np.random.default_rng(64)
    for _ in range(50):
        plan = rng.uniform(0, 1, (5, 5)) * (rng.uniform(0, 1, (5, 5)) < 0.6)
        s, t = cloud(int(rng.integers(1 << 30)), 5), cloud(int(rng.integers(1 << 30)), 5)
        out = pot.barycentric_projection(plan, s, t)
        live = plan.sum(axis=1) > 0
        assert np.all(out[live] >= t.min(axis=0) - 1e-12) and np.all(out[live] <= t.max(axis=0) + 1e-12)


def test_color_transfer_self_transfer_keeps_colors(ctx):  # :126-143
    hist = pot.kmeans_quantize(cloud(65, 400), 8, 11, ctx=ctx)
    cfg = pot.SolverConfig(epsilon=1e-3, log_every=1000000, max_iterations=100000)
    res = pot.color_transfer(hist, hist, 0.5, pot.SolverKind.Aspot, cfg, ctx=ctx)
    for i in range(8):
        if res.solve.plan.X[i].sum() > 1e-3:
            assert np.linalg.norm(res.recolored[i] - hist.centroids[i]) <= 0.05
    assert (res.instance.C * res.solve.plan.X).sum() <= 1e-3 + 1e-9


@pytest.mark.parametrize("kind,p", [(pot.SolverKind.TunedSinkhorn, 1.0), (pot.SolverKind.FeasibleSinkhorn, 1.0),
                                    (pot.SolverKind.TunedSinkhorn, 2.0)])
def test_color_transfer_matches_oracle(ctx, kind, p):
    """The acceptance-test pipeline shape (test_acceptance.cpp:255-300): two
    64-colour histograms of 'warm' / 'cool' images, budget 0.2."""
    rng = np.random.default_rng(7)
    warm = np.clip(rng.normal([0.8, 0.5, 0.3], 0.15, (20000, 3)), 0, 1)
    cool = np.clip(rng.normal([0.3, 0.5, 0.8], 0.15, (20000, 3)), 0, 1)
    src, tgt = pot.kmeans_quantize(warm, 64, 21, ctx=ctx), pot.kmeans_quantize(cool, 64, 22, ctx=ctx)
    cfg = pot.SolverConfig(epsilon=0.05, tuning_exponent_p=p, log_every=1000000)
    g = pot.color_transfer(src, tgt, 0.2, kind, cfg, ctx=ctx)
    rec, o, (r, c, C, s) = ct.color_transfer(src.centroids, src.weights, tgt.centroids, tgt.weights, 0.2, int(kind),
                                             epsilon=0.05, p=p)
    assert g.solve.iterations == o.iterations
    assert abs(g.instance.s - 0.2 * min(g.instance.r.sum(), g.instance.c.sum())) <= 1e-12
    assert g.solve.feasibility_gap <= 1e-9
    np.testing.assert_allclose(g.recolored, rec, rtol=0, atol=1e-8)
    out = pot.recolor_points(src.assignments, g.recolored)
    assert out.shape == (20000, 3) and out.dtype == np.uint8
