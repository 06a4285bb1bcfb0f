"""GPU registration (csrc/registration.cuh) against the registration oracle
(oracle/registration.py) and the reference's own criteria
(test_apps.cpp:160-230, test_acceptance.cpp:403-452 C11).

fp64: identical number of rounds and inner iterations per round, transforms
equal to rounding (the fit reads the plan's row/column sums and moments
instead of a dense plan; Jacobi SVD vs LAPACK)."""
import numpy as np
import pytest

from oracle import binding
from oracle import registration as reg
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu


def random_cloud(seed, n, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (n, 3))


def rotation_z(deg):
    a = np.deg2rad(deg)
    return np.array([[np.cos(a), -np.sin(a), 0.0], [np.sin(a), np.cos(a), 0.0], [0.0, 0.0, 1.0]])


# ----------------------------------------------------------------- fit_rigid --
def test_fit_rigid_cases(ctx):
    pts = random_cloud(67, 20)
    T = pot.fit_rigid(np.eye(20) / 20.0, pts, pts, ctx=ctx)
    assert np.linalg.norm(T.R - np.eye(3)) <= 1e-12 and np.linalg.norm(T.t) <= 1e-12
    cloud = random_cloud(68, 30)
    R0, t0 = rotation_z(37.0), np.array([0.4, -0.7, 0.2])
    T = pot.fit_rigid(np.eye(30) / 30.0, cloud @ R0.T + t0, cloud, ctx=ctx)
    assert np.linalg.norm(T.R - R0) <= 1e-8 and np.linalg.norm(T.t - t0) <= 1e-8
    assert abs(np.linalg.det(T.R) - 1.0) <= 1e-9
    cloud = random_cloud(69, 25)
    mirrored = cloud.copy()
    mirrored[:, 2] *= -1.0
    assert abs(np.linalg.det(pot.fit_rigid(np.eye(25) / 25.0, mirrored, cloud, ctx=ctx).R) - 1.0) <= 1e-9


def test_fit_rigid_errors(ctx):
    pts = random_cloud(70, 10)
    with pytest.raises(pot.PotError) as e:
        pot.fit_rigid(np.zeros((10, 10)), pts, pts, ctx=ctx)
    assert e.value.code == pot.ErrorCode.ZeroMassPlan
    line = np.zeros((10, 3))
    line[:, 0] = 0.1 * np.arange(10)
    with pytest.raises(pot.PotError) as e:
        pot.fit_rigid(np.eye(10) * 0.1, line, line, ctx=ctx)
    assert e.value.code == pot.ErrorCode.DegenerateSvd


@pytest.mark.parametrize("m,n,seed", [(40, 40, 1), (60, 35, 2), (25, 50, 3)])
def test_fit_rigid_matches_oracle_on_random_couplings(ctx, m, n, seed):
    rng = np.random.default_rng(seed)
    pi = rng.uniform(0, 1, (m, n)) ** 4
    x, y = rng.normal(size=(m, 3)), rng.normal(size=(n, 3))
    T = pot.fit_rigid(pi, x, y, ctx=ctx)
    R, t = reg.fit_rigid(pi, x, y)
    np.testing.assert_allclose(T.R, R, rtol=0, atol=1e-12)
    np.testing.assert_allclose(T.t, t, rtol=0, atol=1e-12)


# -------------------------------------------------------------- registration --
def compare(ctx, ref, mov, kind, rtol_T=1e-8, **kw):
    cfg = pot.RegistrationConfig(alpha=kw.get("alpha", 0.4), gamma0=kw.get("gamma0", 4.4e-3),
                                 anneal_rate=kw.get("anneal_rate", 0.83),
                                 transform_threshold=kw.get("transform_threshold", 1e-5),
                                 max_registrations=kw.get("max_registrations", 60),
                                 solve=pot.SolverConfig(epsilon=kw.get("epsilon", 0.01), log_every=10 ** 9,
                                                        max_iterations=kw.get("max_iterations", 3000),
                                                        tuning_exponent_p=kw.get("p", 1.0), materialize_plan=False))
    g = pot.register_point_clouds(ref, mov, cfg, kind=kind, ctx=ctx)
    o = reg.register_point_clouds(ref, mov, kind=int(kind), alpha=cfg.alpha, gamma0=cfg.gamma0,
                                  anneal_rate=cfg.anneal_rate, transform_threshold=cfg.transform_threshold,
                                  max_registrations=cfg.max_registrations, epsilon=cfg.solve.epsilon,
                                  max_iterations=cfg.solve.max_iterations, p=cfg.solve.tuning_exponent_p)
    assert g.converged == o.converged
    assert len(g.rounds) == len(o.rounds)
    assert [r.inner_iterations for r in g.rounds] == [r.inner_iterations for r in o.rounds]
    for a, b in zip(g.rounds, o.rounds):
        assert a.round == b.round and a.gamma == b.gamma
        assert a.cost == pytest.approx(b.cost, rel=1e-7)
    np.testing.assert_allclose(g.transform.R, o.R, rtol=0, atol=rtol_T)
    np.testing.assert_allclose(g.transform.t, o.t, rtol=0, atol=rtol_T)
    return g, o


def test_identical_clouds_fixed_point(ctx):  # test_apps.cpp:216-230
    pts = random_cloud(71, 40)
    cfg = pot.RegistrationConfig(alpha=1.0, solve=pot.SolverConfig(epsilon=0.01, max_iterations=5000,
                                                                    log_every=10 ** 6, materialize_plan=False))
    res = pot.register_point_clouds(pts, pts, cfg, kind=pot.SolverKind.Aspot, ctx=ctx)
    assert res.converged and len(res.rounds) <= 1
    assert np.linalg.norm(res.transform.R - np.eye(3)) <= 1e-4 and np.linalg.norm(res.transform.t) <= 1e-4


def c11_clouds(m=200):
    rng = np.random.default_rng(1111)
    reference = rng.uniform(0.0, 1.0, (m, 3))
    R0, t0 = rotation_z(30.0), np.array([0.3, -0.2, 0.1])
    moving = reference[: m // 2] @ R0.T + t0  # 50 % overlap
    return reference, moving, R0, t0


@pytest.mark.slow
def test_c11_registration_recovery_matches_oracle(ctx):
    """test_acceptance.cpp:403-452 (m = 200, 30 degree rotation, 50 % overlap)
    through the GPU, vs the oracle round by round."""
    reference, moving, R0, t0 = c11_clouds()
    g, _ = compare(ctx, reference, moving, pot.SolverKind.Aspot)
    residual = g.transform.R @ R0
    angle = np.degrees(np.arccos(np.clip((np.trace(residual) - 1.0) / 2.0, -1.0, 1.0)))
    diameter = max(np.linalg.norm(reference[i] - reference[j]) for i in range(200) for j in range(i + 1, 200))
    t_err = np.linalg.norm(g.transform.t - (-R0.T @ t0)) / diameter
    assert len(g.rounds) <= 60 and angle <= 5.0 and t_err <= 0.05


def test_unequal_sizes_padding_matches_oracle(ctx):
    """m < n pads rows, m > n pads columns (registration.hpp:141-150)."""
    ref = random_cloud(5, 30, 0.0, 1.0)
    R0, t0 = rotation_z(15.0), np.array([0.05, 0.1, -0.05])
    mov = np.vstack([ref @ R0.T + t0, random_cloud(6, 12, 0.0, 1.0)])  # 42 moving points
    compare(ctx, ref, mov, pot.SolverKind.Aspot, max_registrations=6, epsilon=0.05, max_iterations=2000)
    compare(ctx, mov, ref, pot.SolverKind.Aspot, max_registrations=6, epsilon=0.05, max_iterations=2000)


@pytest.mark.parametrize("kind,p", [(pot.SolverKind.TunedSinkhorn, 2.0), (pot.SolverKind.FeasibleSinkhorn, 1.0)])
def test_sinkhorn_registration_matches_oracle(ctx, kind, p):
    ref = random_cloud(8, 50, 0.0, 1.0)
    mov = ref[:40] @ rotation_z(20.0).T + np.array([0.1, 0.0, 0.05])
    compare(ctx, ref, mov, kind, max_registrations=8, epsilon=0.05, p=p, max_iterations=5000)


def test_fp32_registration_recovers_rotation(ctx):
    """A C3-shaped problem at n = 2048 in fp32 (stored cost): the recovered
    transform inverts the known motion."""
    rng = np.random.default_rng(33)
    ref = rng.uniform(-1.0, 1.0, (2048, 3))
    R0, t0 = rotation_z(25.0), np.array([0.2, -0.1, 0.15])
    mov = ref @ R0.T + t0
    cfg = pot.RegistrationConfig(alpha=0.9, max_registrations=40,
                                 solve=pot.SolverConfig(epsilon=0.01, log_every=10 ** 9, max_iterations=3000,
                                                        materialize_plan=False))
    res = pot.register_point_clouds(ref, mov, cfg, kind=pot.SolverKind.Aspot, dtype=pot.DType.F32, ctx=ctx)
    angle = np.degrees(np.arccos(np.clip((np.trace(res.transform.R @ R0) - 1.0) / 2.0, -1.0, 1.0)))
    assert angle <= 1.0
    assert np.linalg.norm(res.transform.t - (-R0.T @ t0)) <= 0.02
    assert all(r.inner_iterations > 0 for r in res.rounds)


def test_registration_validation(ctx):
    pts = random_cloud(1, 10)
    with pytest.raises(pot.PotError) as e:
        pot.register_point_clouds(pts[:2], pts, ctx=ctx)
    assert e.value.code == pot.ErrorCode.EmptyInput
    with pytest.raises(pot.PotError) as e:
        pot.register_point_clouds(pts, pts, pot.RegistrationConfig(alpha=0.0), ctx=ctx)
    assert e.value.code == pot.ErrorCode.InvalidArgument
    with pytest.raises(pot.PotError) as e:
        pot.register_point_clouds(pts, pts, pot.RegistrationConfig(anneal_rate=1.0), ctx=ctx)
    assert e.value.code == pot.ErrorCode.InvalidArgument
    with pytest.raises(pot.PotError) as e:
        pot.register_point_clouds(pts[:, :2], pts, ctx=ctx)
    assert e.value.code == pot.ErrorCode.DimensionMismatch
    res = pot.register_point_clouds(np.zeros((5, 3)), np.zeros((5, 3)), ctx=ctx)  # coincident: cmax = 0
    assert res.converged and len(res.rounds) == 0
