"""A small fp32 on-the-fly ASPOT solve (both one-sided blocks, K1'') and a
tuned Sinkhorn solve for compute-sanitizer (memcheck / racecheck) runs:
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

ctx = pot.Context(0)
for n in (700, 1300):
    inst = pot.config_instance(3, n=n, seed=3)
    cfg = pot.SolverConfig(epsilon=2e-2, log_every=10 ** 9, max_iterations=60, materialize_plan=False,
                           collect_iter_log=True)
    r = pot.aspot_solve(inst, cfg, ctx=ctx, iter_log_cap=1000)
    mix = collections.Counter(int(row[4]) for row in r.iter_log)
    print(n, r.status.name, r.iterations, r.cost, r.feasibility_gap, "block_check mix", dict(mix), flush=True)
    t = pot.tuned_sinkhorn_solve(inst, 2e-2, 2.0, pot.SolverConfig(log_every=10 ** 9, materialize_plan=False), ctx=ctx)
    print(n, "tuned", t.status.name, t.iterations, t.cost, flush=True)
