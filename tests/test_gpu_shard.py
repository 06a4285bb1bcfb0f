"""Row-sharded solves (csrc/shard.cuh) on one GPU.

The multi-GPU data path is: each rank sweeps its row block, a gather kernel
folds the block's partials into [rows | cols | max slots], one SUM
all-reduce, then replicated O(n) logic. Here the same kernels run with S
shards in one process (potgpu_comm_init_local; the all-reduce is the
fixed-order device sum over shards) and through a single-rank NCCL
communicator (the NCCL calls captured in the per-iteration CUDA graphs).
Bars as for the unsharded path: fp64 identical decisions / iteration counts
vs the oracle (ties aside), objective rel 1e-6, violation 1e-7; fp32 1e-4 /
1e-5. Only column sums are reassociated by sharding; row sums and the max
exponent are bit-identical (exact zeros elsewhere in the reduced vector)."""
import numpy as np
import pytest

from oracle import binding
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu

TOL_F64_OBJ, TOL_F64_VIOL = 1e-6, 1e-7
TOL_F32_OBJ, TOL_F32_VIOL = 1e-4, 1e-5

_ctxs = {}


def sctx(shards, nccl=False):
    """A context running `shards` row shards (cached per configuration)."""
    key = (shards, nccl)
    if key not in _ctxs:
        c = pot.Context(0)
        if nccl:
            c.init_comm(0, 1, pot.nccl_unique_id())
        c.shard_local(shards)
        _ctxs[key] = c
    return _ctxs[key]


def inst_of(r, c, C, s, dtype=pot.DType.F64):
    return pot.Instance(r=r, c=c, s=s, C=C, dtype=dtype)


@pytest.fixture(autouse=True)
def _need_gpu(ctx):
    yield


def test_comm_info():
    assert sctx(3).comm_info() == (0, 1, 3)
    assert sctx(2, nccl=True).comm_info() == (0, 1, 2)


@pytest.mark.parametrize("n,shards", [(5, 2), (5, 7), (257, 3), (1000, 4), (1000, 1)])
def test_sharded_sweep_matches_oracle(n, shards):
    """B(z) sums through the gather + reduction (n < shards: empty shards)."""
    rng = np.random.default_rng(n + shards)
    r, c, C, s = binding.random_instance(300 + n, n)
    gamma = 0.05
    u, v, w = rng.uniform(-3, 1, n), rng.uniform(-3, 1, n), float(rng.uniform(-1, 1))
    rc, row, col, tot, mx = binding.sweep(C, gamma, u, v, w)
    ev = pot.dual_eval(inst_of(r, c, C, s), gamma, u, v, w, ctx=sctx(shards, nccl=(shards == 1)))
    np.testing.assert_allclose(ev.row, row, rtol=1e-13, atol=0)
    np.testing.assert_allclose(ev.col, col, rtol=1e-13, atol=0)
    assert abs(ev.total - tot) <= 1e-13 * tot
    assert ev.max_exponent == pytest.approx(mx, rel=0, abs=1e-12)


def test_sharded_overflow_detected_in_any_shard():
    """The max-exponent slot of the shard that overflows reaches every rank."""
    n = 64
    C = np.zeros((n, n))
    u = np.zeros(n)
    u[50] = 800.0  # row 50 lives in the last of 4 shards
    inst = inst_of(np.ones(n), np.ones(n), C, 0.5)
    with pytest.raises(pot.PotError) as e:
        pot.dual_eval(inst, 1.0, u, np.zeros(n), 0.0, ctx=sctx(4))
    assert e.value.code == pot.ErrorCode.Overflow


def aspot_vs_oracle(cx, r, c, C, s, cfg, max_tie_flips=0):
    cfg.collect_iter_log = True
    g = pot.aspot_solve(inst_of(r, c, C, s), cfg, ctx=cx, iter_log_cap=200000)
    o = binding.solve(0, r, c, s, C=C, epsilon=cfg.epsilon, gamma_override=cfg.gamma_override,
                      max_iterations=cfg.max_iterations, block_rule=int(cfg.block_rule), log_every=10 ** 9)
    assert int(g.status) == o.status and g.iterations == o.iterations
    flips = np.flatnonzero((g.iter_log[:, 1:5] != o.log[:, 1:5]).any(axis=1))
    assert len(flips) <= max_tie_flips, (flips, g.iter_log[flips], o.log[flips])
    assert abs(g.cost - o.cost) <= TOL_F64_OBJ * max(abs(o.cost), 1e-12)
    assert g.feasibility_gap <= TOL_F64_VIOL
    if g.plan.X is not None and o.plan is not None:
        np.testing.assert_allclose(g.plan.X, o.plan, rtol=1e-6, atol=1e-12)
    return g, o


@pytest.mark.parametrize("seed,n,eps,shards", [(24, 5, 0.1, 2), (25, 6, 0.05, 3), (13, 4, 0.02, 5)])
def test_sharded_aspot_small_matches_oracle(seed, n, eps, shards):
    r, c, C, s = binding.random_instance(seed, n)
    aspot_vs_oracle(sctx(shards), r, c, C, s, pot.SolverConfig(epsilon=eps, log_every=10 ** 9))


@pytest.mark.parametrize("shards,nccl", [(3, False), (1, True), (2, True)])
def test_sharded_aspot_c1_matches_oracle(shards, nccl):
    """configs[0] recipe at n = 300, full solve, plan materialised."""
    inst = pot.config_instance(1, n=300)
    aspot_vs_oracle(sctx(shards, nccl), inst.r, inst.c, inst.C, inst.s, pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9))


def test_sharded_aspot_trace_matches_unsharded(ctx):
    """Per-record rounded costs (the sharded output stage) vs one GPU."""
    inst = pot.config_instance(1, n=200)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=5)
    a = pot.aspot_solve(inst, cfg, ctx=ctx)
    b = pot.aspot_solve(inst, cfg, ctx=sctx(3))
    assert a.iterations == b.iterations and len(a.trace) == len(b.trace)
    for x, y in zip(a.trace, b.trace):
        assert x.t == y.t
        assert y.error == pytest.approx(x.error, rel=1e-9)
        assert y.rounded_cost == pytest.approx(x.rounded_cost, rel=1e-9)
    np.testing.assert_allclose(b.plan.X, a.plan.X, rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("kind", [pot.SolverKind.FeasibleSinkhorn, pot.SolverKind.TunedSinkhorn])
@pytest.mark.parametrize("shards,nccl", [(3, False), (2, True)])
def test_sharded_sinkhorn_matches_oracle(kind, shards, nccl):
    inst = pot.config_instance(1, n=300)
    p = 2.0 if kind == pot.SolverKind.TunedSinkhorn else 1.0
    cfg = pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=p, log_every=10 ** 9)
    g = pot.solve(inst, kind, cfg, ctx=sctx(shards, nccl))
    o = binding.solve(int(kind), inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-2, p=p, log_every=10 ** 9)
    assert int(g.status) == o.status == 0 and g.iterations == o.iterations
    assert abs(g.final_error - o.final_error) <= 1e-8 * o.final_error
    assert abs(g.cost - o.cost) <= TOL_F64_OBJ * abs(o.cost)
    assert g.feasibility_gap <= TOL_F64_VIOL
    np.testing.assert_allclose(g.plan.X, o.plan, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("kind", [pot.SolverKind.Aspot, pot.SolverKind.TunedSinkhorn])
def test_sharded_fp32_points_matches_unsharded(ctx, kind):
    """configs[2] shape at n = 2048 (fp32, on-the-fly cost), 4 shards vs one.
    The fp32 column sums are reassociated by sharding, and the unsharded
    default also takes the one-sided / K1'' passes the sharded path does not.
    Late in the solve the greedy Greenkhorn block choice (solvers.hpp:54-69)
    cycles through near-ties of its rho-scores; fp32 noise can delay one choice
    by an iteration, after which two solves stay one iteration out of phase:
    E_t and the rounded cost oscillate with that phase (E_t by ~20 %, the cost
    by ~0.3 %), the dual objective does not. Measured on B200
    (tools/k1pp_small.py, tools/k1pp_logs.py, profiles/r02/k1pp_small_2048.jsonl):
    the default stops at 1851, the sharded, unfused and fp64 oracle solves at
    1846; phi agrees to 7e-7 at EVERY iteration across all of them; solves
    that stay in phase agree in cost to 5e-5 (profiles/r02/shard_meas.jsonl).
    So: iteration counts within 2 %, phi at equal iteration counts to 1e-6,
    the cost to the fp32 bar when the stops coincide and to 5e-3 otherwise."""
    inst = pot.config_instance(3, n=2048)
    p = 4.0 if kind == pot.SolverKind.TunedSinkhorn else 1.0

    def cfg(cap=10 ** 6):
        return pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=p, log_every=10 ** 9, materialize_plan=False,
                                max_iterations=cap)
    a = pot.solve(inst, kind, cfg(), ctx=ctx)
    b = pot.solve(inst, kind, cfg(), ctx=sctx(4))
    assert a.status == b.status == pot.SolveStatus.Converged
    assert abs(a.iterations - b.iterations) <= max(2, 0.02 * a.iterations)
    assert b.feasibility_gap <= TOL_F32_VIOL and abs(b.plan.mass - inst.s) <= TOL_F32_VIOL
    if a.iterations == b.iterations:
        assert abs(a.cost - b.cost) <= TOL_F32_OBJ * abs(a.cost)
    else:  # the iterate of the earlier stop, on both paths
        k = min(a.iterations, b.iterations)
        a = pot.solve(inst, kind, cfg(k), ctx=ctx)
        b = pot.solve(inst, kind, cfg(k), ctx=sctx(4))
        assert a.iterations == b.iterations == k
        assert abs(a.cost - b.cost) <= 5e-3 * abs(a.cost)
    if kind == pot.SolverKind.Aspot:
        assert abs(a.phi - b.phi) <= 1e-6 * abs(a.phi)


def test_sharded_fp32_aspot_prefix_trajectory(ctx):
    """The same n = 2048 fp32 ASPOT solve for a fixed 150 iterations, 4 shards
    vs one: decisions, E_t and phi agree until the first decision that
    differs, which must be a near-tie of phi(z_check) <= phi_hat at fp32
    precision (as for fp32 vs the fp64 oracle, test_gpu_configs.py C3)."""
    inst = pot.config_instance(3, n=2048)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, max_iterations=150, collect_iter_log=True,
                           materialize_plan=False, record_rounded_cost=False)
    a = pot.aspot_solve(inst, cfg, ctx=ctx, iter_log_cap=200)
    b = pot.aspot_solve(inst, cfg, ctx=sctx(4), iter_log_cap=200)
    diff = np.flatnonzero((a.iter_log[:, 1:5] != b.iter_log[:, 1:5]).any(axis=1))
    k = int(diff[0]) if len(diff) else len(a.iter_log)
    assert k >= 1
    np.testing.assert_allclose(b.iter_log[:k, 5], a.iter_log[:k, 5], rtol=1e-3)
    np.testing.assert_allclose(b.iter_log[:k, 6], a.iter_log[:k, 6], rtol=1e-5)
    if k < len(a.iter_log):  # the first differing decision is a near-tie of z_best (solvers.hpp:342)
        assert abs(a.iter_log[k - 1, 6] - a.iter_log[k, 7]) <= 1e-5 * abs(a.iter_log[k, 7])


def test_sharded_session_steps_match_unsharded(ctx):
    """The bench's session path: k iterations at a time, E_t agrees."""
    inst = pot.config_instance(3, n=2048)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, max_iterations=40, collect_iter_log=True,
                           materialize_plan=False, record_rounded_cost=False)
    res = []
    for cx in (ctx, sctx(2, nccl=True)):
        s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=cx, iter_log_cap=64)
        for _ in range(4):
            s.iterate(10)
        res.append(s.finish())
    a, b = res
    assert a.iterations == b.iterations == 40
    np.testing.assert_allclose(b.iter_log[:, 5], a.iter_log[:, 5], rtol=1e-3)
