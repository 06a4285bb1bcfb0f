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


@pytest.mark.parametrize("side_stream", [False, True])
def test_device_inputs_are_ordered_after_their_producer(ctx, side_stream):
    """A cost still being written by torch when the solve is called (a long
    sleep kernel ahead of it on the producer's stream) is read only after it
    is complete: potgpu_problem.producer_stream."""
    import torch
    inst = pot.config_instance(1, n=512)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, max_iterations=30)
    a = pot.aspot_solve(inst, cfg, ctx=ctx)
    C_host = torch.tensor(inst.C)
    stream = torch.cuda.Stream() if side_stream else torch.cuda.current_stream()
    with torch.cuda.stream(stream):
        C = torch.zeros((512, 512), dtype=torch.float64, device="cuda")
        torch.cuda._sleep(200_000_000)  # ~0.1 s of device time before the copy lands
        C.copy_(C_host.pin_memory().to("cuda", non_blocking=True))
        dev = pot.Instance(r=torch.tensor(inst.r, device="cuda"), c=torch.tensor(inst.c, device="cuda"), s=inst.s, C=C)
        b = pot.aspot_solve(dev, cfg, ctx=ctx)
    assert a.iterations == b.iterations and a.cost == b.cost


@pytest.mark.parametrize("cost", ["points", "dense32"])
def test_fp32_output_stage_matches_oracle_rounding(ctx, cost):
    """The fp32 ASPOT output stage (device round_pot: column-clip sweep +
    fused final sums / <C, X> pass) against the oracle's round_pot of the
    fp64 B(z_check) rebuilt in numpy from the returned potentials: the
    stage's own error, not the solver's. Cost within 1e-5 relative (B200:
    2.3e-6 / 2.7e-6 for dense / points — the column clip's fp32 column sums
    feed the deficit fill, whose mass is a cancellation s - sum(rowX3)),
    slacks within 1e-8; north_star's fp32 objective bar is 1e-4."""
    pts = pot.config_instance(3, n=1500)
    f32 = lambda x: np.asarray(x, dtype=np.float32).astype(np.float64)  # noqa: E731
    C = pot.dense_cost(f32(pts.X), f32(pts.Y), pts.cost_scale)
    inst = pts if cost == "points" else pot.Instance(r=pts.r, c=pts.c, s=pts.s, C=C, dtype=pot.DType.F32)
    if cost == "dense32":
        C = f32(C)
    g = pot.aspot_solve(inst, pot.SolverConfig(epsilon=2e-2, log_every=10 ** 9, max_iterations=300,
                                               materialize_plan=False), ctx=ctx)
    E = (-C / g.gamma + g.u[:, None]) + g.v[None, :] + g.w
    X = binding.round_pot(np.exp(E), C, inst.r, inst.c, inst.s)
    ocost, omass = float(np.sum(C * X)), float(X.sum())
    assert abs(g.cost - ocost) <= 1e-5 * abs(ocost), (g.cost, ocost)
    np.testing.assert_allclose(g.plan.row_slack, inst.r - X.sum(axis=1), rtol=0, atol=1e-8)
    np.testing.assert_allclose(g.plan.col_slack, inst.c - X.sum(axis=0), rtol=0, atol=1e-8)
    assert abs(g.plan.mass - omass) <= 1e-9


@pytest.mark.parametrize("kind", ["aspot", "tuned", "feasible"])
@pytest.mark.parametrize("cost", ["points", "dense32"])
def test_fused_fp32_output_stage_matches_dense_plan(ctx, kind, cost):
    """The fused fp32 output pass (no dense plan) against the dense-plan path
    of the same solve (k_plan_cost, fp64 exponentials, materialize_plan=True)
    and numpy's <C, X> of that plan. dense32: both paths sum the same fp32
    exponents (1e-6). points: the fused pass forms the exponent in fp64
    (k_rowcost_pts64) while the dense-plan path takes its final row sums from
    the solver's fp32 sweep and the deficit fill moves with them (measured
    2.7e-5 on B200 for the Sinkhorn plans; the oracle comparison above pins
    the fused pass itself to 1e-6)."""
    pts = pot.config_instance(3, n=1500)
    if cost == "dense32":
        inst = pot.Instance(r=pts.r, c=pts.c, s=pts.s, C=pot.dense_cost(pts.X, pts.Y, pts.cost_scale),
                            dtype=pot.DType.F32)
    else:
        inst = pts
    sk = {"aspot": pot.SolverKind.Aspot, "tuned": pot.SolverKind.TunedSinkhorn,
          "feasible": pot.SolverKind.FeasibleSinkhorn}[kind]
    base = dict(epsilon=2e-2, tuning_exponent_p=4.0, log_every=10 ** 9, max_iterations=300)
    a = pot.solve(inst, sk, pot.SolverConfig(materialize_plan=False, **base), ctx=ctx)
    b = pot.solve(inst, sk, pot.SolverConfig(materialize_plan=True, **base), ctx=ctx)
    assert a.iterations == b.iterations
    f32 = lambda x: np.asarray(x, dtype=np.float32).astype(np.float64)  # noqa: E731
    C = pot.dense_cost(f32(pts.X), f32(pts.Y), pts.cost_scale) if cost == "points" else f32(inst.C)
    ref = float(np.sum(C * b.plan.X))
    assert abs(b.cost - ref) <= 1e-9 * abs(ref), (b.cost, ref)
    tol, atol = (1e-6, 1e-9) if cost == "dense32" else (1e-4, 1e-8)
    assert abs(a.cost - ref) <= tol * abs(ref), (a.cost, ref)
    np.testing.assert_allclose(a.plan.row_slack, b.plan.row_slack, rtol=0, atol=atol)
    np.testing.assert_allclose(a.plan.col_slack, b.plan.col_slack, rtol=0, atol=atol)
    assert a.feasibility_gap <= 1e-5


DEVICE_ROUND_SNIPPET = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
from paper_2601_17196_b200 import pot
out = {}
pts = pot.config_instance(3, n=1200)
cases = {"f64": pot.config_instance(1, n=700),
         "dense32": pot.Instance(r=pts.r, c=pts.c, s=pts.s, C=pot.dense_cost(pts.X, pts.Y, pts.cost_scale),
                                 dtype=pot.DType.F32),
         "points": pts}
for name, inst in cases.items():
    cfg = pot.SolverConfig(epsilon=2e-2, log_every=10 ** 9, max_iterations=400, materialize_plan=False)
    g = pot.aspot_solve(inst, cfg)
    out[name] = {"it": g.iterations, "cost": g.cost, "gap": g.feasibility_gap, "mass": g.plan.mass,
                 "rs": g.plan.row_slack.tolist(), "cs": g.plan.col_slack.tolist()}
print(json.dumps(out))
"""


def test_device_rounding_matches_host_rounding():
    """round_pot of the ASPOT plan on the device (plan.cuh enqueue_round_device:
    single-block O(n) kernels around the two sweeps, one download) against
    the host-orchestrated implicit rounding ($POTGPU_DEVICE_ROUND=0), fp64
    stored, fp32 stored and fp32 points."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("1", "0"):
        env = dict(os.environ, POTGPU_DEVICE_ROUND=flag)
        r = subprocess.run([sys.executable, "-c", DEVICE_ROUND_SNIPPET % root], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[flag] = json.loads(r.stdout.strip().splitlines()[-1])
    for name in ("f64", "dense32", "points"):
        d, h = res["1"][name], res["0"][name]
        assert d["it"] == h["it"]
        tol = 1e-12 if name == "f64" else (1e-6 if name == "dense32" else 1e-5)
        assert abs(d["cost"] - h["cost"]) <= tol * abs(h["cost"]), (name, d["cost"], h["cost"])
        assert abs(d["mass"] - h["mass"]) <= 1e-12
        atol = 1e-14 if name == "f64" else 1e-8
        np.testing.assert_allclose(d["rs"], h["rs"], rtol=0, atol=atol)
        np.testing.assert_allclose(d["cs"], h["cs"], rtol=0, atol=atol)
        assert d["gap"] <= (1e-7 if name == "f64" else 1e-5)


TAIL_SNIPPET = r"""
import json, sys
sys.path.insert(0, %r)
from paper_2601_17196_b200 import pot
out = {}
for name, inst in (("f64", pot.config_instance(1, n=600)), ("points", pot.config_instance(3, n=1500))):
    cfg = pot.SolverConfig(epsilon=2e-2, log_every=3, max_iterations=90, materialize_plan=False,
                           record_rounded_cost=True)
    g = pot.aspot_solve(inst, cfg, trace_cap=1000)
    out[name] = {"t": [r.t for r in g.trace], "rc": [r.rounded_cost for r in g.trace], "cost": g.cost}
print(json.dumps(out))
"""


def test_record_rounding_tail_matches_host_rounding():
    """record_rounded_cost with records inside the loop: the per-record
    round_pot runs as a gated device tail of the attempt graph (no pause,
    no host round trip); every record's cost equals the paused host-driven
    rounding ($POTGPU_NO_ROUND_TAIL=1)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("", "1"):
        env = dict(os.environ)
        if flag:
            env["POTGPU_NO_ROUND_TAIL"] = flag
        r = subprocess.run([sys.executable, "-c", TAIL_SNIPPET % root], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[flag] = json.loads(r.stdout.strip().splitlines()[-1])
    for name, tol in (("f64", 1e-13), ("points", 1e-9)):
        a, b = res[""][name], res["1"][name]
        assert a["t"] == b["t"] and len(a["t"]) >= 5
        assert all(x is not None for x in a["rc"])
        np.testing.assert_allclose(a["rc"], b["rc"], rtol=tol)
