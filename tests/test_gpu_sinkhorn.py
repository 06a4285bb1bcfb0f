"""GPU parity of the feasible / tuned Sinkhorn solvers (solvers.hpp:387-589)
against the CPU oracle, through the C-ABI. fp64: identical iteration
counts and statuses, objective rel <= 1e-6, violation <= 1e-7; fp32:
objective rel <= 1e-4, violation <= 1e-5."""
import math

import numpy as np
import pytest

from oracle import binding
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu

TOL_F64_OBJ, TOL_F64_VIOL = 1e-6, 1e-7
TOL_F32_OBJ, TOL_F32_VIOL = 1e-4, 1e-5


def inst_of(r, c, C, s, dtype=pot.DType.F64):
    return pot.Instance(r=r, c=c, s=s, C=C, dtype=dtype)


def run_pair(ctx, kind, r, c, C, s, eps, p=1.0, max_iterations=200000, gamma=None, dtype=pot.DType.F64, log_every=10 ** 9):
    cfg = pot.SolverConfig(epsilon=eps, tuning_exponent_p=p, max_iterations=max_iterations, gamma_override=gamma,
                           log_every=log_every)
    g = pot.solve(inst_of(r, c, C, s, dtype), kind, cfg, ctx=ctx)
    o = binding.solve(int(kind), r, c, s, C=C, epsilon=eps, p=p, max_iterations=max_iterations, gamma_override=gamma,
                      log_every=log_every)
    return g, o


@pytest.mark.parametrize("kind", [pot.SolverKind.FeasibleSinkhorn, pot.SolverKind.TunedSinkhorn])
@pytest.mark.parametrize("seed,n", [(29, 5), (30, 6), (31, 4), (32, 7), (33, 3)])
def test_sinkhorn_small_instances_match_oracle(ctx, kind, seed, n):
    r, c, C, s = binding.random_instance(seed, n)
    p = 2.0 if kind == pot.SolverKind.TunedSinkhorn else 1.0
    g, o = run_pair(ctx, kind, r, c, C, s, 0.1, p=p)
    assert int(g.status) == o.status == 0
    assert g.iterations == o.iterations
    assert g.gamma == o.gamma and g.tolerance == o.tolerance
    assert abs(g.final_error - o.final_error) <= 1e-9 * max(o.final_error, 1e-30) + 1e-14
    assert abs(g.cost - o.cost) <= TOL_F64_OBJ * max(abs(o.cost), 1e-12)
    assert g.feasibility_gap <= TOL_F64_VIOL
    np.testing.assert_allclose(g.plan.X, o.plan, rtol=1e-6, atol=1e-12)
    assert g.stopping_iterate == "extended-marginals"


def test_sinkhorn_c1_matches_oracle(ctx):
    """configs[0] recipe (n = 300 here; feasible Sinkhorn, eps = 1e-2)."""
    inst = pot.config_instance(1, n=300)
    g, o = run_pair(ctx, pot.SolverKind.FeasibleSinkhorn, inst.r, inst.c, inst.C, inst.s, 1e-2)
    assert int(g.status) == o.status and g.iterations == o.iterations
    assert abs(g.cost - o.cost) <= TOL_F64_OBJ * abs(o.cost)
    assert g.feasibility_gap <= TOL_F64_VIOL


@pytest.mark.parametrize("p", [2.0, 4.0])
def test_tuned_sinkhorn_c2_shape_fp64(ctx, p):
    """configs[1] recipe (colour clouds) at n = 512, eps = 1e-3, tuned p."""
    inst = pot.config_instance(2, n=512)
    g, o = run_pair(ctx, pot.SolverKind.TunedSinkhorn, inst.r, inst.c, inst.C, inst.s, 1e-3, p=p)
    assert int(g.status) == o.status and g.iterations == o.iterations
    assert abs(g.cost - o.cost) <= TOL_F64_OBJ * abs(o.cost)
    assert g.feasibility_gap <= TOL_F64_VIOL


def test_tuned_sinkhorn_c2_shape_fp32(ctx):
    inst = pot.config_instance(2, n=512, dtype=pot.DType.F32)
    g, o = run_pair(ctx, pot.SolverKind.TunedSinkhorn, inst.r, inst.c, inst.C, inst.s, 1e-3, p=4.0,
                    dtype=pot.DType.F32)
    assert int(g.status) == o.status
    assert abs(g.cost - o.cost) <= TOL_F32_OBJ * abs(o.cost)
    assert g.feasibility_gap <= TOL_F32_VIOL


def test_tuned_sinkhorn_points_fp32(ctx):
    """configs[2] shape on the fly (n = 1024), tuned p = 4."""
    inst = pot.config_instance(3, n=1024)
    cfg = pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=4.0, log_every=10 ** 9, materialize_plan=False)
    g = pot.tuned_sinkhorn_solve(inst, cfg, ctx=ctx)
    C = pot.dense_cost(inst.X, inst.Y, inst.cost_scale)
    o = binding.solve(2, inst.r, inst.c, inst.s, C=C, epsilon=1e-2, p=4.0, log_every=10 ** 9)
    assert int(g.status) == o.status == 0
    assert abs(g.cost - o.cost) <= TOL_F32_OBJ * abs(o.cost)
    assert g.feasibility_gap <= TOL_F32_VIOL


def test_sinkhorn_trace_records_match_oracle(ctx):
    """log_every = 1: every record carries the rounded cost of the extended
    plan (solvers.hpp:444-455)."""
    r, c, C, s = binding.random_instance(30, 6)
    g, o = run_pair(ctx, pot.SolverKind.FeasibleSinkhorn, r, c, C, s, 0.1, log_every=1)
    o = binding.solve(1, r, c, s, C=C, epsilon=0.1, log_every=1, record_rounded_cost=True)
    assert len(g.trace) == len(o.trace)
    for rec, orow in zip(g.trace, o.trace):
        assert rec.t == int(orow[0])
        assert rec.error == pytest.approx(orow[1], rel=1e-9, abs=1e-15)
        assert rec.phi == pytest.approx(orow[2], rel=1e-9, abs=1e-15)
        assert rec.rounded_cost == pytest.approx(orow[3], rel=1e-9, abs=1e-15)


def test_sinkhorn_single_point_and_zero_budget(ctx):
    """test_solvers.cpp:373-378, 480-490."""
    inst = inst_of(np.array([1.0]), np.array([0.8]), np.array([[3.0]]), 0.5)
    g = pot.feasible_sinkhorn_solve(inst, pot.SolverConfig(), ctx=ctx)
    assert g.plan.X[0, 0] == 0.5 and g.status == pot.SolveStatus.Converged
    r, c, C, s = binding.random_instance(34, 4)
    for kind in (pot.SolverKind.FeasibleSinkhorn, pot.SolverKind.TunedSinkhorn):
        g = pot.solve(inst_of(r, c, C, 0.0), kind, pot.SolverConfig(), ctx=ctx)
        assert np.abs(g.plan.X).max() == 0.0 and g.status == pot.SolveStatus.Converged


def test_tuned_gamma_prescription(ctx):
    """test_solvers.cpp:380-392: gamma = (2 eps / (49 H_min))^(1/p), eps' = 2 eps / 49."""
    r, c, C, s = binding.random_instance(30, 5)
    h = min(-(r * np.log(r)).sum(), -(c * np.log(c)).sum())
    for p in (1.0, 2.0, 4.0):
        g = pot.tuned_sinkhorn_solve(inst_of(r, c, C, s), 0.098, p, pot.SolverConfig(max_iterations=1), ctx=ctx)
        assert g.gamma == pytest.approx((2 * 0.098 / (49 * h)) ** (1 / p), rel=1e-13)
        assert g.tolerance == pytest.approx(2 * 0.098 / 49, rel=1e-12)


def test_tuned_unit_entropy_gamma(ctx):
    """test_solvers.cpp:394-415: H = 1, p = 1, eps = 0.098 -> gamma = 0.004."""
    lo, hi = 0.3, 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        x = mid / 3
        if -3 * x * math.log(x) < 1.0:
            lo = mid
        else:
            hi = mid
    a = 0.5 * (lo + hi)
    r = np.full(3, a / 3)
    C = np.ones((3, 3)) - np.eye(3)
    g = pot.tuned_sinkhorn_solve(inst_of(r, r.copy(), C, 0.25 * a), 0.098, 1.0, pot.SolverConfig(max_iterations=1),
                                 ctx=ctx)
    assert g.gamma == pytest.approx(0.004, abs=1e-12)
    assert g.tolerance == pytest.approx(0.004, abs=1e-12)


def test_tuned_rejects_zero_entropy(ctx):
    """test_solvers.cpp:446-461."""
    inst = inst_of(np.array([3.0, 2.0]), np.array([2.5, 2.5]), np.ones((2, 2)), 1.0)
    with pytest.raises(pot.PotError) as e:
        pot.tuned_sinkhorn_solve(inst, 0.1, 1.0, ctx=ctx)
    assert e.value.code == pot.ErrorCode.ZeroEntropy


def test_solvers_agree_within_two_epsilon(ctx):
    """test_solvers.cpp:463-478 on the device path."""
    for seed in (33, 34, 35):
        r, c, C, s = binding.random_instance(seed, 6)
        cfg = pot.SolverConfig(epsilon=0.1, log_every=10 ** 9, max_iterations=200000)
        a = pot.aspot_solve(inst_of(r, c, C, s), cfg, ctx=ctx).cost
        b = pot.feasible_sinkhorn_solve(inst_of(r, c, C, s), cfg, ctx=ctx).cost
        t = pot.tuned_sinkhorn_solve(inst_of(r, c, C, s), 0.1, 2.0, cfg, ctx=ctx).cost
        assert abs(a - b) <= 0.2 + 1e-9 and abs(a - t) <= 0.2 + 1e-9 and abs(b - t) <= 0.2 + 1e-9
