"""Golden vectors (tests/golden/): the CPU oracle against its committed
outputs on the reference's own fixture generator (drift pin), and against the
reference tests' hand-valued known answers. No GPU."""
import json
import os

import numpy as np
import pytest

from oracle import binding

from .golden.make_golden import CASES, SOLVERS, instance_digest, log_digest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("case", load("solves.json")["cases"], ids=lambda c: f"n{c['n']}s{c['seed']}")
def test_oracle_reproduces_golden_solves(case):
    r, c, C, s = binding.make_synthetic(case["n"], case["seed"], case["mass_r"], case["mass_c"], case["s_frac"])
    assert instance_digest(r, c, C, s) == case["instance_sha256"]  # the fixture generator's draw order
    for kind, name, p in SOLVERS:
        g = case["results"][name]
        o = binding.solve(kind, r, c, s, C=C, epsilon=case["epsilon"], p=p, log_every=10 ** 9)
        assert (o.status, o.iterations) == (g["status"], g["iterations"]), name
        assert o.cost == g["cost"] and o.final_error == g["final_error"], name
        assert np.array_equal(o.plan.sum(axis=1), np.array(g["plan_row_sums"])), name
        if kind == 0:
            assert log_digest(o.log) == g["decision_log_sha256"]


def test_golden_cases_match_generator_list():
    got = [(c["n"], c["seed"], c["mass_r"], c["mass_c"], c["s_frac"], c["epsilon"]) for c in load("solves.json")["cases"]]
    assert got == [tuple(x) for x in CASES]


def scalar(c0):
    return np.array([[c0]]), np.ones(1), np.ones(1), 0.5


def test_oracle_reference_kats():
    k = load("reference_kats.json")
    for e in k["b_matrix"]:
        C, _, _, _ = scalar(e["c0"])
        rc, row, col, tot, mx = binding.sweep(C, e["gamma"], np.array([e["u"]]), np.array([e["v"]]), e["w"])
        assert rc == 0 and abs(tot - e["B"]) <= e["tol"], e["cite"]
    for e in k["overflow"]:
        C, _, _, _ = scalar(e["c0"])
        rc = binding.sweep(C, e["gamma"], np.array([e["u"]]), np.array([e["v"]]), e["w"])[0]
        assert rc != 0, e["cite"]


def test_headline_fixtures_match_their_instances():
    """tests/golden/headline.json (the oracle's answers at n = 65536, read by
    the GPU parity tests instead of a 9-minute oracle run): every entry's
    digest is the digest of the instance the recipe builds today."""
    from tests import headline_golden
    from paper_2601_17196_b200 import pot
    inst = pot.config_instance(4)
    a = headline_golden.load("c4_aspot_prefix", inst.X, inst.Y, inst.r, inst.c, [inst.s])
    assert a.iterations == 3 and a.log.shape == (3, 9) and a.scale > 0
    t = headline_golden.load("c4_tuned_prefix", inst.X, inst.Y, inst.r, inst.c, [inst.s])
    assert t.iterations == 1 and [int(x) for x in t.trace[:, 0]] == [0, 1]
