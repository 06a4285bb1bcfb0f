"""Parity on all five BASELINE.json configs at their real sizes.

Where the CPU oracle can finish (configs[0], configs[1] Sinkhorn, batched
problems) the comparison is a full solve; where it cannot in seconds
(n = 16384, 65536) it is prefix parity of the first iterations plus
size-independent properties of the GPU's full solve (convergence to the
stated tolerance, exact feasibility of the rounded plan, plan mass = s).
The oracle runs on every host core here; its results are bit-identical for
any thread count (oracle/pot_oracle.hpp sweep / parallel_for)."""
import os

import numpy as np
import pytest

from oracle import binding
from tests import headline_golden
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu

TOL_F64_OBJ, TOL_F64_VIOL = 1e-6, 1e-7
TOL_F32_OBJ, TOL_F32_VIOL = 1e-4, 1e-5


@pytest.fixture(autouse=True)
def oracle_threads():
    binding.lib().oracle_set_threads(os.cpu_count() or 1)
    yield


def oracle_cost(inst):
    return inst.C if inst.C is not None else pot.dense_cost(inst.X, inst.Y, inst.cost_scale)


def check_properties(g, s, tol_viol):
    assert g.feasibility_gap <= tol_viol
    assert abs(g.plan.mass - s) <= tol_viol
    assert np.all(g.plan.row_slack >= -tol_viol) and np.all(g.plan.col_slack >= -tol_viol)
    if g.status == pot.SolveStatus.Converged:
        assert g.final_error <= g.tolerance


# ---------------------------------------------------------- configs[0] --
def test_c1_feasible_sinkhorn_full(ctx):
    """n = 1000 fp64 stored, feasible Sinkhorn to convergence (the ASPOT
    counterpart is test_gpu_aspot.py::test_aspot_c1_full_matches_oracle)."""
    inst = pot.config_instance(1)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9)
    g = pot.feasible_sinkhorn_solve(inst, cfg, ctx=ctx)
    o = binding.solve(1, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-2)
    assert int(g.status) == o.status == 0 and g.iterations == o.iterations
    assert abs(g.cost - o.cost) <= TOL_F64_OBJ * abs(o.cost)
    check_properties(g, inst.s, TOL_F64_VIOL)


# ---------------------------------------------------------- configs[1] --
@pytest.mark.slow
def test_c2_aspot_prefix_fp64(ctx):
    """n = 4096 fp64, eps = 1e-3: the first 12 iterations take identical
    decisions and E_t (the oracle cannot finish the full solve in seconds)."""
    inst = pot.config_instance(2)
    cfg = pot.SolverConfig(epsilon=1e-3, log_every=10 ** 9, max_iterations=12, collect_iter_log=True,
                           materialize_plan=False)
    g = pot.aspot_solve(inst, cfg, ctx=ctx, iter_log_cap=100)
    o = binding.solve(0, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-3, max_iterations=12, skip_plan=True)
    assert g.iterations == o.iterations == 12
    np.testing.assert_array_equal(g.iter_log[:, 1:5], o.log[:, 1:5])
    np.testing.assert_allclose(g.iter_log[:, 5], o.log[:, 5], rtol=1e-9)
    np.testing.assert_allclose(g.iter_log[:, 6], o.log[:, 6], rtol=1e-12)


@pytest.mark.slow
@pytest.mark.parametrize("dtype,p", [(pot.DType.F64, 4.0), (pot.DType.F32, 4.0), (pot.DType.F64, 2.0)])
def test_c2_tuned_sinkhorn_full(ctx, dtype, p):
    """n = 4096, eps = 1e-3, tuned gamma (p = 2, 4) to convergence."""
    inst = pot.config_instance(2, dtype=dtype)
    cfg = pot.SolverConfig(epsilon=1e-3, tuning_exponent_p=p, log_every=10 ** 9, materialize_plan=False)
    g = pot.tuned_sinkhorn_solve(inst, cfg, ctx=ctx)
    o = binding.solve(2, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-3, p=p, skip_plan=False, want_plan=False)
    assert int(g.status) == o.status == 0
    if dtype == pot.DType.F64:
        assert g.iterations == o.iterations
        assert abs(g.cost - o.cost) <= TOL_F64_OBJ * abs(o.cost)
        check_properties(g, inst.s, TOL_F64_VIOL)
    else:
        assert abs(g.iterations - o.iterations) <= max(2, 0.02 * o.iterations)
        assert abs(g.cost - o.cost) <= TOL_F32_OBJ * abs(o.cost)
        check_properties(g, inst.s, TOL_F32_VIOL)


@pytest.mark.slow
def test_c2_tuned_sinkhorn_p1_capped(ctx):
    """p = 1: gamma = 2 eps / (49 H_min) is tiny and the solve is long; both
    capped at 300 iterations: same status and trace (fp64)."""
    inst = pot.config_instance(2)
    cfg = pot.SolverConfig(epsilon=1e-3, tuning_exponent_p=1.0, log_every=50, max_iterations=300,
                           record_rounded_cost=False, materialize_plan=False)
    g = pot.tuned_sinkhorn_solve(inst, cfg, ctx=ctx)
    o = binding.solve(2, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-3, p=1.0, max_iterations=300, log_every=50,
                      skip_plan=True)
    assert int(g.status) == o.status and g.iterations == o.iterations
    assert g.gamma == o.gamma and g.tolerance == o.tolerance
    assert [r.t for r in g.trace] == [int(x) for x in o.trace[:, 0]]
    np.testing.assert_allclose([r.error for r in g.trace], o.trace[:, 1], rtol=1e-9)


@pytest.mark.slow
def test_c2_feasible_sinkhorn_capped(ctx):
    """n = 4096 fp64, eps = 1e-3, feasible Sinkhorn (the ASPOT gamma = 3.0e-5:
    thousands of iterations, beyond the oracle's budget in a test): both
    capped at 200 iterations, same status, trace errors to 1e-9 and the
    rounded plan of the capped iterate to the fp64 bars."""
    inst = pot.config_instance(2)
    cfg = pot.SolverConfig(epsilon=1e-3, log_every=25, max_iterations=200, record_rounded_cost=False,
                           materialize_plan=False)
    g = pot.feasible_sinkhorn_solve(inst, cfg, ctx=ctx)
    o = binding.solve(1, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-3, max_iterations=200, log_every=25,
                      want_plan=False)
    assert int(g.status) == o.status and g.iterations == o.iterations
    assert [r.t for r in g.trace] == [int(x) for x in o.trace[:, 0]]
    np.testing.assert_allclose([r.error for r in g.trace], o.trace[:, 1], rtol=1e-9)
    assert abs(g.cost - o.cost) <= TOL_F64_OBJ * abs(o.cost)
    check_properties(g, inst.s, TOL_F64_VIOL)


@pytest.mark.slow
def test_c2_aspot_prefix_fp32(ctx):
    """n = 4096 fp32 stored cost: 12 iterations against the fp64 oracle on the
    fp32-rounded C; decisions identical until the first fp32 near-tie of
    z_best, E_t and phi to the fp32 bars up to there."""
    inst = pot.config_instance(2, dtype=pot.DType.F32)
    cfg = pot.SolverConfig(epsilon=1e-3, log_every=10 ** 9, max_iterations=12, collect_iter_log=True,
                           materialize_plan=False)
    g = pot.aspot_solve(inst, cfg, ctx=ctx, iter_log_cap=100)
    o = binding.solve(0, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-3, max_iterations=12, skip_plan=True)
    assert g.iterations == o.iterations == 12
    diff = np.flatnonzero((g.iter_log[:, 1:5] != o.log[:, 1:5]).any(axis=1))
    k = int(diff[0]) if len(diff) else 12
    assert k >= 2
    np.testing.assert_allclose(g.iter_log[:k, 5], o.log[:k, 5], rtol=1e-4)
    np.testing.assert_allclose(g.iter_log[:k, 6:8], o.log[:k, 6:8], rtol=1e-6)
    if k < 12:
        assert abs(o.log[k - 1, 6] - o.log[k, 7]) <= 1e-5 * abs(o.log[k, 7]), (o.log, g.iter_log)


# ---------------------------------------------------------- configs[2] --
@pytest.mark.slow
def test_c3_aspot_prefix_and_full(ctx):
    """n = 16384 fp32 on the fly: first 3 iterations vs the fp64 oracle on the
    fp32-rounded coordinates (E_t, phi within fp32 tolerance), then the GPU's
    full solve converges with an exactly feasible rounded plan."""
    inst = pot.config_instance(3)
    if not inst.cost_scale:
        inst.cost_scale = pot.points_scale(inst.X, inst.Y)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, max_iterations=3, collect_iter_log=True,
                           materialize_plan=False)
    g = pot.aspot_solve(inst, cfg, ctx=ctx, iter_log_cap=10)
    o = binding.solve(0, inst.r, inst.c, inst.s, X=inst.X, Y=inst.Y, scale=inst.cost_scale, epsilon=1e-2,
                      max_iterations=3, skip_plan=True)
    assert g.iterations == o.iterations == 3
    # fp32 vs fp64: identical decisions until the first near-tie (z_best's
    # phi(z_check) <= phi_hat can resolve differently at fp32 precision);
    # E_t and phi agree to fp32 tolerance up to there
    diff = np.flatnonzero((g.iter_log[:, 2:5] != o.log[:, 2:5]).any(axis=1))
    k = int(diff[0]) if len(diff) else 3
    assert k >= 1
    np.testing.assert_allclose(g.iter_log[:k, 5], o.log[:k, 5], rtol=1e-3)  # E_t
    np.testing.assert_allclose(g.iter_log[:k, 6], o.log[:k, 6], rtol=1e-5)  # phi(z_check)
    if k < 3:  # iteration k compares phi(z_check_{k-1}) (col 6, row k-1) with phi_hat_k (col 7)
        assert abs(o.log[k - 1, 6] - o.log[k, 7]) <= 1e-5 * abs(o.log[k, 7]), (o.log, g.iter_log)
    full = pot.aspot_solve(inst, pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, materialize_plan=False), ctx=ctx)
    assert full.status == pot.SolveStatus.Converged
    check_properties(full, inst.s, TOL_F32_VIOL)


@pytest.mark.slow
def test_c3_tuned_sinkhorn_prefix_and_full(ctx):
    inst = pot.config_instance(3)
    if not inst.cost_scale:
        inst.cost_scale = pot.points_scale(inst.X, inst.Y)
    cfg = pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=4.0, log_every=1, max_iterations=2,
                           record_rounded_cost=False, materialize_plan=False)
    g = pot.tuned_sinkhorn_solve(inst, cfg, ctx=ctx)
    o = binding.solve(2, inst.r, inst.c, inst.s, X=inst.X, Y=inst.Y, scale=inst.cost_scale, epsilon=1e-2, p=4.0,
                      max_iterations=2, log_every=1, skip_plan=True)
    assert g.iterations == o.iterations == 2
    for rec, orow in zip(g.trace, o.trace):
        assert rec.t == int(orow[0])
        assert rec.error == pytest.approx(orow[1], rel=1e-3)
    full = pot.tuned_sinkhorn_solve(inst, pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=4.0, log_every=10 ** 9,
                                                            materialize_plan=False), ctx=ctx)
    assert full.status == pot.SolveStatus.Converged
    check_properties(full, inst.s, TOL_F32_VIOL)


# ---------------------------------------------------------- configs[3] --
@pytest.mark.slow
def test_c4_tuned_sinkhorn_full_and_prefix(ctx):
    """n = 65536 fp32 on the fly (n^2 = 2^32: 64-bit indexing), tuned p = 4:
    the first iteration vs the oracle (points mode), then the full solve."""
    inst = pot.config_instance(4)
    assert inst.cost_scale is None  # derived on the device (max over 2^32 pairs)
    cfg = pot.SolverConfig(epsilon=1e-3, tuning_exponent_p=4.0, log_every=1, max_iterations=1,
                           record_rounded_cost=False, materialize_plan=False)
    g = pot.tuned_sinkhorn_solve(inst, cfg, ctx=ctx)
    full = pot.tuned_sinkhorn_solve(inst, pot.SolverConfig(epsilon=1e-3, tuning_exponent_p=4.0, log_every=10 ** 9,
                                                            materialize_plan=False), ctx=ctx)
    assert full.status == pot.SolveStatus.Converged
    check_properties(full, inst.s, TOL_F32_VIOL)
    # the oracle needs the same cost normalisation the device derived: the
    # max over all pairs, computed here in chunks
    if headline_golden.live():  # ~1.5 min on 16 cores
        scale = pot.points_scale(inst.X, inst.Y, chunk=1024)
        o = binding.solve(2, inst.r, inst.c, inst.s, X=inst.X, Y=inst.Y, scale=scale, epsilon=1e-3, p=4.0,
                          max_iterations=1, log_every=1, skip_plan=True)
    else:  # the same call's result, committed (tests/golden/make_headline_golden.py)
        o = headline_golden.load("c4_tuned_prefix", inst.X, inst.Y, inst.r, inst.c, [inst.s])
    assert [int(x) for x in o.trace[:, 0]] == [rec.t for rec in g.trace]
    for rec, orow in zip(g.trace, o.trace):
        assert rec.error == pytest.approx(orow[1], rel=1e-3)


@pytest.mark.slow
def test_c4_aspot_runs_and_is_feasible(ctx):
    """n = 65536 ASPOT (eps = 1e-3): 50 iterations, exactly feasible plan."""
    inst = pot.config_instance(4)
    cfg = pot.SolverConfig(epsilon=1e-3, log_every=10 ** 9, max_iterations=50, materialize_plan=False)
    g = pot.aspot_solve(inst, cfg, ctx=ctx)
    assert g.iterations == 50 or g.status == pot.SolveStatus.Converged
    assert g.status != pot.SolveStatus.StepSizeUnderflow
    check_properties(g, inst.s, TOL_F32_VIOL)
    assert np.isfinite(g.cost) and g.cost > 0


# ---------------------------------------------------------- configs[4] --
@pytest.mark.slow
def test_c5_batched_problems_match_oracle(ctx):
    """256 x n = 2048 fp32 stored problems (per-problem seeds); here 4 of them
    through the batched entry point, each vs the oracle (ASPOT and tuned
    Sinkhorn p = 4)."""
    insts = [pot.config_instance(5, seed=1 + k) for k in range(4)]
    for kind, p in ((pot.SolverKind.Aspot, 1.0), (pot.SolverKind.TunedSinkhorn, 4.0)):
        cfg = pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=p, log_every=10 ** 9, materialize_plan=False)
        res = pot.solve_batched(kind, insts, cfg, ctx=ctx, concurrency=4)
        for inst, g in zip(insts, res):
            o = binding.solve(int(kind), inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-2, p=p, want_plan=False)
            assert int(g.status) == o.status == 0
            assert abs(g.cost - o.cost) <= TOL_F32_OBJ * abs(o.cost)
            assert abs(g.iterations - o.iterations) <= max(3, 0.05 * o.iterations)
            check_properties(g, inst.s, TOL_F32_VIOL)


def test_batched_matches_single_solves(ctx):
    """potgpu_solve_batched (workers on SM shares, own streams) against one
    solve per problem: fp64 decisions, iteration counts and statuses equal,
    costs to rounding."""
    insts = [pot.config_instance(1, n=300, seed=10 + k) for k in range(6)]
    cfg = pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9, materialize_plan=False)
    for kind in (pot.SolverKind.Aspot, pot.SolverKind.FeasibleSinkhorn):
        res = pot.solve_batched(kind, insts, cfg, ctx=ctx, concurrency=3)
        for inst, b in zip(insts, res):
            g = pot.solve(inst, kind, cfg, ctx=ctx)
            assert b.status == g.status and b.iterations == g.iterations, (kind, b.iterations, g.iterations)
            assert abs(b.cost - g.cost) <= 1e-9 * abs(g.cost)
