"""Sweep / attempt counters of a small fp64 ASPOT solve (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2601_17196_b200 import pot  # noqa: E402

ctx = pot.Context(0)
inst = pot.config_instance(1, n=256)
for rrc in (True, False):
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, collect_iter_log=True, record_rounded_cost=rrc)
    g = pot.aspot_solve(inst, cfg, ctx=ctx, iter_log_cap=100000)
    print("record_rounded_cost", rrc, "iterations", g.iterations, "sweeps", g.sweeps, "attempts", g.attempts,
          "halvings", int(g.iter_log[:, 1].sum()), "trace", len(g.trace))
