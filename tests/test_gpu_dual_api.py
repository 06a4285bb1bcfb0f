"""The reference's dual-level public API (dual.hpp, solvers.hpp helpers,
core.hpp validation) through the Python mirror: b_matrix / exponent_matrix
(device), dual_objective / dual_gradient / feasibility_error (device sums),
greenkhorn_step, aspot_setup, the AspotObserver hook — against the oracle
and the reference's hand values (test_dual.cpp, test_solvers.cpp)."""
import math

import numpy as np
import pytest

from oracle import binding
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu


def test_dual_functions_hand_values(ctx):
    """test_dual.cpp:54-160 on the 1 x 1 instance: phi = 3, grad = (1, 1, .5)."""
    ectx = pot.EntropicContext(np.zeros((1, 1)), 1.0, np.ones(1), np.ones(1), 0.5)
    z = pot.DualPoint.zero(1)
    assert pot.dual_objective(ectx, z, ctx=ctx) == 3.0
    g = pot.dual_gradient(ectx, z, ctx=ctx)
    assert g.u[0] == 1.0 and g.v[0] == 1.0 and g.w == 0.5
    assert pot.feasibility_error(ectx, z, ctx=ctx) == 2.5
    assert pot.b_matrix(ectx, z, ctx=ctx)[0, 0] == 1.0
    with pytest.raises(pot.PotError) as e:
        pot.b_matrix(ectx, pot.DualPoint(np.array([400.0]), np.array([400.0]), 0.0), ctx=ctx)
    assert e.value.code == pot.ErrorCode.Overflow


def test_b_matrix_matches_oracle_sums(ctx):
    r, c, C, s = binding.random_instance(11, 40)
    rng = np.random.default_rng(2)
    u, v, w = rng.uniform(-3, 1, 40), rng.uniform(-3, 1, 40), 0.3
    ectx = pot.EntropicContext(C, 0.05, r, c, s)
    z = pot.DualPoint(u, v, w)
    E = pot.exponent_matrix(ectx, z, ctx=ctx)
    np.testing.assert_array_equal(E, ((-C / 0.05 + u[:, None]) + v[None, :]) + w)
    B = pot.b_matrix(ectx, z, ctx=ctx)
    rc, row, col, tot, mx = binding.sweep(C, 0.05, u, v, w)
    np.testing.assert_allclose(B.sum(axis=1), row, rtol=1e-13)
    np.testing.assert_allclose(B.sum(axis=0), col, rtol=1e-13)


def test_greenkhorn_step_and_setup_match_oracle_solve(ctx):
    """The first iterations of ASPOT rebuilt from the public helpers equal the
    device solver's decision log (greenkhorn_step, aspot_setup, theta_next,
    dual_gradient, dual_objective: solvers.hpp:296-369)."""
    r, c, C, s = binding.random_instance(24, 5)
    inst = pot.Instance(r=r, c=c, s=s, C=C)
    st = pot.aspot_setup(inst, 0.1)
    ectx = pot.EntropicContext(C, st.gamma, st.mixed_r, st.mixed_c, s)
    n = 5
    z, zc, theta, gk = pot.DualPoint.zero(n), pot.DualPoint.zero(n), 1.0, 0
    step_denom = 3.0 * (st.mixed_r.sum() + st.mixed_c.sum() - s)
    phic = pot.dual_objective(ectx, zc, ctx=ctx)
    errs = []
    for _ in range(4):
        step = st.gamma / (step_denom * theta)
        zb = (1.0 - theta) * zc + theta * z
        g = pot.dual_gradient(ectx, zb, ctx=ctx)
        zg = zb + theta * ((zb - step * g) - z)
        zh = pot.greenkhorn_step(ectx, zg, pot.BlockRule.Greedy, gk, ctx=ctx)
        phih = pot.dual_objective(ectx, zh, ctx=ctx)
        best = zc if phic <= phih else zh
        zc = pot.greenkhorn_step(ectx, best, pot.BlockRule.Greedy, gk + 1, ctx=ctx)
        z, gk, theta = best, gk + 2, pot.theta_next(theta)
        phic = pot.dual_objective(ectx, zc, ctx=ctx)
        errs.append(pot.feasibility_error(ectx, zc, ctx=ctx))
    o = binding.solve(0, r, c, s, C=C, epsilon=0.1, max_iterations=4)
    np.testing.assert_allclose(errs, o.log[:4, 5], rtol=1e-10)


def test_aspot_observer_sees_every_iteration(ctx):
    inst = pot.config_instance(1, n=100)
    seen = []
    cfg = pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9)
    res = pot.aspot_solve(inst, cfg, ctx=ctx, observer=seen.append)
    plain = pot.aspot_solve(inst, cfg, ctx=ctx)
    assert res.iterations == plain.iterations == len(seen) and res.cost == plain.cost
    assert [it.t for it in seen] == list(range(1, res.iterations + 1))
    last = seen[-1]
    assert last.error == pytest.approx(res.final_error, rel=0, abs=0)
    assert last.phi_best <= last.phi_hat and last.z_check.u.shape == (100,)
    assert pot.feasibility_error(last.ctx, last.z_check, ctx=ctx) == pytest.approx(last.error, rel=1e-9)


def test_validation_report_lists_every_violation():
    inst = pot.Instance(r=np.array([1.0, -1.0]), c=np.ones(2), s=5.0, C=np.array([[0.0, -1.0], [1.0, 0.0]]))
    codes = [v.code for v in pot.validation_report(inst)]
    assert codes == [pot.ErrorCode.NegativeEntry, pot.ErrorCode.NegativeEntry, pot.ErrorCode.BudgetExceedsMass]
    with pytest.raises(pot.ValidationError) as e:
        pot.validate(inst)
    assert e.value.code == pot.ErrorCode.NegativeEntry and len(e.value.violations) == 3
    assert pot.solver_kind_from_name("sinkhorn") == pot.SolverKind.FeasibleSinkhorn
    assert pot.solver_kind_from_name("nope") is None
