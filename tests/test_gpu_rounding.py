"""round_pot / round_balanced on user plans (csrc/dense_round.cuh) against the
oracle (rounding.hpp restatement): every path of the projection — mass cap,
row clip, column clip, deficit fill, zero rows / columns, the empty plan —
and the error codes. The device sums are fixed-order trees, the oracle's
sequential/compensated: agreement to ~1e-15 relative."""
import numpy as np
import pytest

from oracle import binding
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu


def case(seed, n, density=1.0, scale=1.0):
    rng = np.random.default_rng(seed)
    r, c, C, s = binding.random_instance(seed, n)
    X = rng.uniform(0, scale, (n, n)) * (rng.uniform(0, 1, (n, n)) < density)
    return pot.Instance(r=r, c=c, s=s, C=C), X


@pytest.mark.parametrize("seed,n,density,scale", [(1, 5, 1.0, 1.0), (2, 37, 0.3, 0.01), (3, 100, 1.0, 10.0),
                                                  (4, 257, 0.05, 0.1), (5, 8, 0.0, 1.0), (6, 600, 0.5, 0.001)])
def test_round_pot_matches_oracle(ctx, seed, n, density, scale):
    inst, X = case(seed, n, density, scale)
    g = pot.round_pot(X, inst, ctx=ctx)
    o = binding.round_pot(X, inst.C, inst.r, inst.c, inst.s)
    np.testing.assert_allclose(g.X, o, rtol=1e-13, atol=1e-16)
    assert abs(g.mass - inst.s) <= 1e-12
    assert np.all(g.row_slack >= -1e-12) and np.all(g.col_slack >= -1e-12)


@pytest.mark.parametrize("seed,rows,cols", [(7, 6, 6), (8, 50, 80), (9, 300, 200)])
def test_round_balanced_matches_oracle(ctx, seed, rows, cols):
    rng = np.random.default_rng(seed)
    r = rng.uniform(0.1, 1, rows)
    c = rng.uniform(0.1, 1, cols)
    c *= r.sum() / c.sum()
    X = rng.uniform(0, 0.01, (rows, cols))
    g = pot.round_balanced(X, r, c, ctx=ctx)
    o = binding.round_balanced(X, r, c)
    np.testing.assert_allclose(g, o, rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(g.sum(axis=1), r, rtol=1e-12)
    np.testing.assert_allclose(g.sum(axis=0), c, rtol=1e-12)


def test_rounding_errors(ctx):
    inst, X = case(10, 5)
    with pytest.raises(pot.PotError) as e:
        pot.round_pot(X[:4], inst, ctx=ctx)
    assert e.value.code == pot.ErrorCode.DimensionMismatch
    bad = pot.Instance(r=inst.r, c=inst.c, s=10.0, C=inst.C)
    with pytest.raises(pot.PotError) as e:
        pot.round_pot(X, bad, ctx=ctx)
    assert e.value.code == pot.ErrorCode.BudgetExceedsMass
    with pytest.raises(pot.PotError) as e:
        pot.round_balanced(X, np.ones(5), 2 * np.ones(5), ctx=ctx)
    assert e.value.code == pot.ErrorCode.UnbalancedMarginals


def test_device_resident_inputs_match_host_inputs(ctx):
    """device_ptrs = 1 (CUDA arrays, e.g. torch tensors; zero-copy for C):
    the same solve as from host buffers."""
    import torch
    inst = pot.config_instance(1, n=300)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9)
    a = pot.aspot_solve(inst, cfg, ctx=ctx)
    dev = pot.Instance(r=torch.tensor(inst.r, device="cuda"), c=torch.tensor(inst.c, device="cuda"), s=inst.s,
                       C=torch.tensor(inst.C, device="cuda"))
    b = pot.aspot_solve(dev, cfg, ctx=ctx)
    assert a.iterations == b.iterations and a.cost == b.cost
    pts = pot.config_instance(3, n=1024)
    cfg32 = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, materialize_plan=False)
    a = pot.aspot_solve(pts, cfg32, ctx=ctx)
    devp = pot.Instance(r=torch.tensor(pts.r, device="cuda"), c=torch.tensor(pts.c, device="cuda"), s=pts.s,
                        X=torch.tensor(pts.X, device="cuda"), Y=torch.tensor(pts.Y, device="cuda"),
                        cost_scale=pts.cost_scale, dtype=pot.DType.F32)
    b = pot.aspot_solve(devp, cfg32, ctx=ctx)
    assert a.iterations == b.iterations and a.cost == b.cost
