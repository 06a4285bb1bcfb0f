"""The device path against the committed golden vectors (tests/golden/):
fp64 solves on the reference's fixture instances (same iteration counts,
statuses and ASPOT decision logs; objective within the fp64 bar), and the
reference tests' hand-valued known answers through potgpu_dual_eval."""
import json
import os

import numpy as np
import pytest

from paper_2601_17196_b200 import pot

from .golden.make_golden import SOLVERS, instance_digest, log_digest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL_F64_OBJ, TOL_F64_VIOL = 1e-6, 1e-7


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("case", load("solves.json")["cases"], ids=lambda c: f"n{c['n']}s{c['seed']}")
def test_device_matches_golden_solves(ctx, case):
    inst = pot.make_synthetic_instance(case["n"], case["seed"], case["mass_r"], case["mass_c"], case["s_frac"])
    assert instance_digest(inst.r, inst.c, inst.C, inst.s) == case["instance_sha256"]
    for kind, name, p in SOLVERS:
        g = case["results"][name]
        cfg = pot.SolverConfig(epsilon=case["epsilon"], tuning_exponent_p=p, log_every=10 ** 9,
                               collect_iter_log=kind == 0)
        d = pot.solve(inst, pot.SolverKind(kind), cfg, ctx=ctx, iter_log_cap=100000)
        assert (int(d.status), d.iterations) == (g["status"], g["iterations"]), name
        assert abs(d.cost - g["cost"]) <= TOL_F64_OBJ * abs(g["cost"]), name
        assert d.feasibility_gap <= TOL_F64_VIOL
        assert np.allclose(d.plan.X.sum(axis=1), g["plan_row_sums"], rtol=1e-6, atol=1e-12)
        if kind == 0:
            assert log_digest(d.iter_log) == g["decision_log_sha256"]


def test_device_reference_kats(ctx):
    k = load("reference_kats.json")
    for e in k["b_matrix"]:
        inst = pot.Instance(r=np.ones(1), c=np.ones(1), s=0.5, C=np.array([[e["c0"]]]))
        de = pot.dual_eval(inst, e["gamma"], [e["u"]], [e["v"]], e["w"], ctx=ctx)
        assert abs(de.total - e["B"]) <= e["tol"], e["cite"]
    for e in k["overflow"]:
        inst = pot.Instance(r=np.ones(1), c=np.ones(1), s=0.5, C=np.array([[e["c0"]]]))
        with pytest.raises(pot.PotError) as ex:
            pot.dual_eval(inst, e["gamma"], [e["u"]], [e["v"]], e["w"], ctx=ctx)
        assert ex.value.code == pot.ErrorCode.Overflow, e["cite"]
    z = k["at_zero"]
    inst = pot.Instance(r=np.ones(1), c=np.ones(1), s=0.5, C=np.array([[z["c0"]]]))
    de = pot.dual_eval(inst, z["gamma"], [0.0], [0.0], 0.0, ctx=ctx)
    assert de.phi == z["phi"] and de.error == z["error"] and de.grad_w == z["grad_w"], z["cite"]
