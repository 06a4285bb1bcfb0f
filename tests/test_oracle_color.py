"""Colour-transfer oracle (oracle/color_transfer.py, binding.kmeans) against
the reference's own tests (test_apps.cpp:38-160). CPU only."""
import numpy as np
import pytest

from oracle import binding
from oracle import color_transfer as ct


def cloud(seed, n):
    return np.random.default_rng(seed).uniform(0.0, 1.0, (n, 3))


def test_kmeans_each_point_its_own_centroid():  # :38-52
    pts = cloud(61, 6)
    C, W, A, _ = binding.kmeans(pts, 6, 7)
    assert np.max(np.abs(W - 1.0 / 6.0)) <= 1e-15
    for i in range(6):
        assert np.min(np.linalg.norm(C - pts[i], axis=1)) <= 1e-12


def test_kmeans_recovers_well_separated_blobs():  # :54-80
    rng = np.random.default_rng(62)
    pts = np.vstack([0.1 + rng.normal(0, 0.01, (100, 3)), 0.9 + rng.normal(0, 0.01, (100, 3))])
    C, W, A, _ = binding.kmeans(pts, 2, 3)
    a, b = pts[:100].mean(axis=0), pts[100:].mean(axis=0)
    first, second = (a, b) if np.linalg.norm(C[0] - a) < np.linalg.norm(C[0] - b) else (b, a)
    assert np.linalg.norm(C[0] - first) <= 1e-3 and np.linalg.norm(C[1] - second) <= 1e-3
    assert abs(W.sum() - 1.0) <= 1e-12


def test_kmeans_rejects_bad_arguments():  # :82-87
    pts = cloud(63, 4)
    with pytest.raises(binding.OracleError):
        binding.kmeans(pts, 5, 1)
    with pytest.raises(binding.OracleError):
        binding.kmeans(np.zeros((0, 3)), 1, 1)


def test_barycentric_row_average_and_zero_row():  # :89-105
    plan = np.array([[0.2, 0.2], [0.0, 0.0]])
    src = np.array([[0.3, 0.3, 0.3], [0.9, 0.1, 0.5]])
    tgt = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]])
    out = ct.barycentric_projection(plan, src, tgt)
    assert np.linalg.norm(out[0] - 0.5) <= 1e-15
    assert np.array_equal(out[1], src[1])


def test_color_transfer_self_and_budget():  # :126-160
    hist = binding.kmeans(cloud(65, 400), 8, 11)
    rec, res, (r, c, C, s) = ct.color_transfer(hist[0], hist[1], hist[0], hist[1], 0.5, 0, epsilon=1e-3,
                                               max_iterations=100000)
    for i in range(8):
        if res.plan[i].sum() > 1e-3:
            assert np.linalg.norm(rec[i] - hist[0][i]) <= 0.05
    assert (C * res.plan).sum() <= 1e-3 + 1e-9
    src, tgt = binding.kmeans(cloud(66, 300), 6, 1), binding.kmeans(cloud(67, 300), 6, 2)
    rec, res, (r, c, C, s) = ct.color_transfer(src[0], src[1], tgt[0], tgt[1], 0.2, 2, epsilon=0.05)
    assert abs(s - 0.2 * min(r.sum(), c.sum())) <= 1e-12
    assert abs(C.max() - 1.0) <= 1e-12
    assert res.feasibility_gap <= 1e-9
