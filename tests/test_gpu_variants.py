"""Every run-time selectable variant of the device path (environment
switches read once per process, so each runs in a subprocess) solves the
same small problems as the default build: the fp64 dense ASPOT path with
the same decisions and objective to rounding, the fp32 on-the-fly path
within the fp32 bar. Covers the CUDA-graph WHILE loop, the full z_check' sweep instead of the one-sided one, PDL off, the
evaluation's threads per index, and the measured points-sweep variants."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import json, sys
sys.path.insert(0, %r)
from paper_2601_17196_b200 import pot
ctx = pot.Context(0)
out = {}
d = pot.config_instance(1, n=300, seed=5)
g = pot.aspot_solve(d, pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9, materialize_plan=False), ctx=ctx)
out["dense"] = [int(g.status), g.iterations, g.cost, g.feasibility_gap]
p = pot.config_instance(3, n=700, seed=5)
g = pot.aspot_solve(p, pot.SolverConfig(epsilon=5e-2, log_every=10 ** 9, max_iterations=200, materialize_plan=False), ctx=ctx)
out["points"] = [int(g.status), g.iterations, g.cost, g.feasibility_gap]
g = pot.tuned_sinkhorn_solve(p, 5e-2, 2.0, pot.SolverConfig(log_every=10 ** 9, materialize_plan=False), ctx=ctx)
out["sinkhorn"] = [int(g.status), g.iterations, g.cost, g.feasibility_gap]
print(json.dumps(out))
""" % ROOT


def run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SNIPPET], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def baseline():
    return run({})


@pytest.mark.parametrize("env", [
    {"POTGPU_GRAPH_LOOP": "1"},
    {"POTGPU_ONE_SIDED": "0"},
    {"POTGPU_K1PP": "0"},
    {"POTGPU_PTS1_TWO": "0"},
    {"POTGPU_PDL": "0"},
    {"POTGPU_EVAL_TPI": "1"},
    {"POTGPU_EVAL_BLOCKS_PER_SM": "1"},
    {"POTGPU_PTS_PAIRS": "3"},
    {"POTGPU_PTS_PAIRS": "5"},
    {"POTGPU_PTS_PAIRS": "8"},
    {"POTGPU_SWEEP_WAVES": "4"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_matches_default(baseline, env):
    got = run(env)
    st, it, cost, gap = got["dense"]
    assert (st, it) == tuple(baseline["dense"][:2])
    assert abs(cost - baseline["dense"][2]) <= 1e-9 * abs(baseline["dense"][2]) and gap <= 1e-7
    for key in ("points", "sinkhorn"):
        st, it, cost, gap = got[key]
        b = baseline[key]
        assert st == b[0] and abs(cost - b[2]) <= 1e-4 * abs(b[2]) and gap <= 1e-5, (key, got[key], b)
