"""The registration oracle (oracle/registration.py) against the reference's
own registration tests (test_apps.cpp:160-230 FitRigid*, Registration*).
CPU only; the C11 acceptance case (test_acceptance.cpp:403-452) runs with
the GPU parity test (tests/test_gpu_registration.py) where the oracle is the
comparison point."""
import numpy as np
import pytest

from oracle import binding
from oracle import registration as reg


def random_cloud(seed, n):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (n, 3))


def rotation_z(deg):
    a = np.deg2rad(deg)
    return np.array([[np.cos(a), -np.sin(a), 0.0], [np.sin(a), np.cos(a), 0.0], [0.0, 0.0, 1.0]])


def test_fit_rigid_identity_for_aligned_clouds():  # test_apps.cpp:160-168
    pts = random_cloud(67, 20)
    R, t = reg.fit_rigid(np.eye(20) / 20.0, pts, pts)
    assert np.linalg.norm(R - np.eye(3)) <= 1e-12
    assert np.linalg.norm(t) <= 1e-12


def test_fit_rigid_recovers_known_transform():  # :170-185
    cloud = random_cloud(68, 30)
    R0, t0 = rotation_z(37.0), np.array([0.4, -0.7, 0.2])
    moved = cloud @ R0.T + t0
    R, t = reg.fit_rigid(np.eye(30) / 30.0, moved, cloud)
    assert np.linalg.norm(R - R0) <= 1e-8 and np.linalg.norm(t - t0) <= 1e-8
    assert np.linalg.norm(R.T @ R - np.eye(3)) <= 1e-9
    assert abs(np.linalg.det(R) - 1.0) <= 1e-9


def test_fit_rigid_reflection_corrected():  # :187-195
    cloud = random_cloud(69, 25)
    mirrored = cloud.copy()
    mirrored[:, 2] *= -1.0
    R, _ = reg.fit_rigid(np.eye(25) / 25.0, mirrored, cloud)
    assert abs(np.linalg.det(R) - 1.0) <= 1e-9


def test_fit_rigid_errors_on_degenerate_input():  # :197-214
    pts = random_cloud(70, 10)
    with pytest.raises(binding.OracleError) as e:
        reg.fit_rigid(np.zeros((10, 10)), pts, pts)
    assert e.value.code == reg.ZERO_MASS_PLAN
    line = np.zeros((10, 3))
    line[:, 0] = 0.1 * np.arange(10)
    with pytest.raises(binding.OracleError) as e:
        reg.fit_rigid(np.eye(10) * 0.1, line, line)
    assert e.value.code == reg.DEGENERATE_SVD


def test_registration_identical_clouds_fixed_point():  # :216-230
    pts = random_cloud(71, 40)
    res = reg.register_point_clouds(pts, pts, kind=0, alpha=1.0, epsilon=0.01, max_iterations=5000)
    assert res.converged and len(res.rounds) <= 1
    assert np.linalg.norm(res.R - np.eye(3)) <= 1e-4 and np.linalg.norm(res.t) <= 1e-4


def test_apply_all_and_compose_match_matrix_algebra():
    rng = np.random.default_rng(3)
    A = (rotation_z(20.0), np.array([0.1, 0.2, 0.3]))
    B = (rotation_z(-50.0), np.array([-0.3, 0.0, 0.5]))
    pts = rng.normal(size=(7, 3))
    np.testing.assert_allclose(reg.apply_all(*A, pts), pts @ A[0].T + A[1], rtol=0, atol=1e-15)
    R, t = reg.compose(A, B)
    np.testing.assert_allclose(reg.apply_all(R, t, pts), reg.apply_all(*A, reg.apply_all(*B, pts)), atol=1e-14)
