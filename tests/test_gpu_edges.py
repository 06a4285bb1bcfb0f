"""Edge cases of the fp32 kernels: sizes that are not multiples of the
512-column strip (padding columns), partial 32-row tiles, tiny n, zero
marginal entries, coincident points — fp32 results against the fp64 oracle
on the same fp32-rounded inputs, and the invariants every rounded plan must
satisfy."""
import numpy as np
import pytest

from oracle import binding
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu

TOL_F32_OBJ, TOL_F32_VIOL = 1e-4, 1e-5


def points_instance(n, seed, zero_frac=0.0, dup=False):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (n, 3))
    Y = X + rng.normal(0, 0.2, (n, 3)) if dup is False else X.copy()
    r = rng.uniform(0.2, 1, n)
    c = rng.uniform(0.2, 1, n)
    if zero_frac:
        r[rng.uniform(0, 1, n) < zero_frac] = 0.0
    r /= r.sum()
    c /= c.sum() / 1.2
    return pot.Instance(r=r, c=c, s=0.8, X=X, Y=Y, dtype=pot.DType.F32)


def check(g, inst):
    assert g.feasibility_gap <= TOL_F32_VIOL
    assert abs(g.plan.mass - inst.s) <= TOL_F32_VIOL
    assert np.all(g.plan.row_slack >= -TOL_F32_VIOL) and np.all(g.plan.col_slack >= -TOL_F32_VIOL)


@pytest.mark.parametrize("n,seed", [(3, 1), (33, 2), (511, 3), (513, 4), (1000, 5)])
@pytest.mark.parametrize("kind", [pot.SolverKind.Aspot, pot.SolverKind.TunedSinkhorn])
def test_points_odd_sizes_match_oracle(ctx, n, seed, kind):
    inst = points_instance(n, seed)
    inst.cost_scale = pot.points_scale(inst.X, inst.Y)
    p = 2.0 if kind == pot.SolverKind.TunedSinkhorn else 1.0
    cfg = pot.SolverConfig(epsilon=5e-2, tuning_exponent_p=p, log_every=10 ** 9)
    g = pot.solve(inst, kind, cfg, ctx=ctx)
    C = pot.dense_cost(inst.X, inst.Y, inst.cost_scale)
    o = binding.solve(int(kind), inst.r, inst.c, inst.s, C=C, epsilon=5e-2, p=p, log_every=10 ** 9)
    assert int(g.status) == o.status
    assert abs(g.iterations - o.iterations) <= max(3, 0.05 * o.iterations)
    assert abs(g.cost - o.cost) <= 5 * TOL_F32_OBJ * abs(o.cost) + 1e-9
    check(g, inst)


@pytest.mark.parametrize("n", [7, 600, 1027])
def test_dense_fp32_odd_sizes_match_oracle(ctx, n):
    r, c, C, s = binding.random_instance(900 + n, n)
    inst = pot.Instance(r=r, c=c, s=s, C=C.astype(np.float32).astype(np.float64), dtype=pot.DType.F32)
    cfg = pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9)
    g = pot.aspot_solve(inst, cfg, ctx=ctx)
    o = binding.solve(0, r, c, s, C=inst.C, epsilon=5e-2, log_every=10 ** 9)
    assert int(g.status) == o.status
    assert abs(g.cost - o.cost) <= 5 * TOL_F32_OBJ * abs(o.cost) + 1e-9
    check(g, inst)


def test_zero_marginal_entries_and_coincident_points(ctx):
    inst = points_instance(300, 9, zero_frac=0.2)
    inst.cost_scale = pot.points_scale(inst.X, inst.Y)
    for kind in (pot.SolverKind.Aspot, pot.SolverKind.TunedSinkhorn, pot.SolverKind.FeasibleSinkhorn):
        g = pot.solve(inst, kind, pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9), ctx=ctx)
        assert g.status == pot.SolveStatus.Converged
        check(g, inst)
        zero_rows = inst.r == 0
        assert np.all(np.abs(g.plan.X[zero_rows]) <= TOL_F32_VIOL)
    dup = points_instance(200, 10, dup=True)  # Y == X: a zero-cost diagonal
    dup.cost_scale = pot.points_scale(dup.X, dup.Y)
    g = pot.aspot_solve(dup, pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9), ctx=ctx)
    assert g.status == pot.SolveStatus.Converged
    check(g, dup)


def test_max_iterations_one_and_session_pause(ctx):
    inst = pot.config_instance(3, n=1024)
    g = pot.aspot_solve(inst, pot.SolverConfig(epsilon=1e-2, max_iterations=1, log_every=1,
                                               materialize_plan=False), ctx=ctx)
    assert g.iterations == 1 and g.status == pot.SolveStatus.MaxIterationsExceeded
    assert [t.t for t in g.trace] == [0, 1]
    assert all(t.rounded_cost is not None and np.isfinite(t.rounded_cost) for t in g.trace)
    check(g, inst)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, materialize_plan=False, record_rounded_cost=False)
    s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
    done = 0
    for k in (1, 2, 5, 10):
        _, it, fin = s.iterate(k)
        assert it == k and not fin
        done += it
    a = s.finish()
    b = pot.aspot_solve(inst, pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, max_iterations=done,
                                               materialize_plan=False, record_rounded_cost=False), ctx=ctx)
    assert a.final_error == b.final_error and a.cost == b.cost


@pytest.mark.parametrize("dtype", [pot.DType.F64, pot.DType.F32])
def test_dense_layouts_give_identical_solves(ctx, dtype):
    """The dense cost read from C order, Fortran order (Eigen's column-major
    MatrixXd) and padded row / column views (leading dimension > n): the
    device sees the same values, so the solves agree bit for bit. n x ldc
    spans more than one pinned staging chunk, the last one partial."""
    n = 1100
    base = pot.config_instance(1, n=n, seed=4, dtype=dtype)
    cfg = pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9, max_iterations=60)
    ref = pot.aspot_solve(base, cfg, ctx=ctx)
    wide = np.full((n, n + 37), np.nan)
    wide[:, :n] = base.C
    tall = np.full((n + 11, n), np.nan)
    tall[:n, :] = base.C
    for C in (np.asfortranarray(base.C), wide[:, :n], np.asfortranarray(tall)[:n, :]):
        inst = pot.Instance(r=base.r, c=base.c, s=base.s, C=C, dtype=dtype)
        g = pot.aspot_solve(inst, cfg, ctx=ctx)
        assert g.iterations == ref.iterations and g.status == ref.status
        assert g.cost == ref.cost and g.final_error == ref.final_error
        assert np.array_equal(g.plan.row_slack, ref.plan.row_slack)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_device_cost_scale_is_the_exact_fp64_max(ctx, seed):
    """The on-the-fly cost scale derived on the device (two fp32 passes, then
    fp64 on the candidate pairs) equals 1 / max_ij |x_i - y_j|^2 in the fp64
    formula the host uses, so a solve with the scale derived on the device
    and one with the host's scale are bit-identical. Seed 2 adds many pairs
    that tie or nearly tie for the maximum."""
    rng = np.random.default_rng(seed)
    n = 3000
    X = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
    Y = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
    if seed == 2:  # corners: many (near-)maximal pairs
        X[:50] = np.float32(-1.0)
        Y[:50] = np.float32(1.0)
        Y[50:60] = np.nextafter(np.float32(1.0), np.float32(0.0))
    r = np.full(n, 1.0 / n)
    cfg = pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9, max_iterations=30, materialize_plan=False)
    a = pot.aspot_solve(pot.Instance(r=r, c=r, s=0.9, X=X, Y=Y, cost_scale=None, dtype=pot.DType.F32), cfg, ctx=ctx)
    b = pot.aspot_solve(pot.Instance(r=r, c=r, s=0.9, X=X, Y=Y, cost_scale=pot.points_scale(X, Y),
                                     dtype=pot.DType.F32), cfg, ctx=ctx)
    assert a.iterations == b.iterations and a.cost == b.cost and a.final_error == b.final_error
