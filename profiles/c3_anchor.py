"""C3 (n = 16384) fp32 headline solve against an fp64 GPU anchor on the same
fp32-rounded coordinates (stored fp64 logK, 2.1 GB), and the C4 (n = 65536)
ASPOT / tuned Sinkhorn full solves. Prints one JSON line per measurement.
Run on the GPU box; the numbers feed DESIGN.md §7 and BASELINE.md §4."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

ctx = pot.Context(0)


def summ(tag, r, extra=None):
    d = {"tag": tag, "status": r.status.name, "iterations": r.iterations, "cost": r.cost, "phi": r.phi,
         "final_error": r.final_error, "tolerance": r.tolerance, "gap": r.feasibility_gap, "mass": r.plan.mass,
         "wall_s": r.wall_seconds, "loop_s": r.loop_seconds}
    d.update(extra or {})
    print(json.dumps(d), flush=True)
    return d


inst = pot.config_instance(3)
inst.cost_scale = pot.points_scale(inst.X, inst.Y)
anchor = pot.Instance(r=inst.r, c=inst.c, s=inst.s, X=inst.X, Y=inst.Y, cost_scale=inst.cost_scale,
                      dtype=pot.DType.F64, stored=True)
cfg = lambda **k: pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, materialize_plan=False,  # noqa: E731
                                   record_rounded_cost=False, collect_iter_log=True, **k)
a = pot.aspot_solve(anchor, cfg(), ctx=ctx, iter_log_cap=100000)
summ("c3_fp64_anchor", a)
f = pot.aspot_solve(inst, cfg(), ctx=ctx, iter_log_cap=100000)
la, lf = a.iter_log, f.iter_log
m = min(len(la), len(lf))
diff = np.flatnonzero((la[:m, 1:5] != lf[:m, 1:5]).any(axis=1))
first = int(diff[0]) if len(diff) else m
summ("c3_fp32", f, {"first_decision_diff": first, "n_decision_diff": int(len(diff)),
                    "E_rel_at_first": float(abs(lf[max(first - 1, 0), 5] / la[max(first - 1, 0), 5] - 1))})
g = pot.aspot_solve(inst, cfg(max_iterations=a.iterations), ctx=ctx, iter_log_cap=100000)
summ("c3_fp32_at_anchor_iterations", g)
for K in (100, 500, 1000):
    a2 = pot.aspot_solve(anchor, cfg(max_iterations=K), ctx=ctx, iter_log_cap=100000)
    g2 = pot.aspot_solve(inst, cfg(max_iterations=K), ctx=ctx, iter_log_cap=100000)
    summ(f"c3_fp64_K{K}", a2)
    summ(f"c3_fp32_K{K}", g2, {"cost_rel": abs(g2.cost / a2.cost - 1), "phi_rel": abs(g2.phi / a2.phi - 1)})
del anchor

if os.environ.get("C4", "1") == "1":
    c4 = pot.config_instance(4)
    t0 = time.perf_counter()
    r = pot.aspot_solve(c4, pot.SolverConfig(epsilon=1e-3, log_every=10 ** 9, materialize_plan=False,
                                             record_rounded_cost=False, max_iterations=200000), ctx=ctx)
    summ("c4_aspot_full", r, {"host_s": time.perf_counter() - t0})
    for p in (4.0, 2.0):
        t0 = time.perf_counter()
        r = pot.tuned_sinkhorn_solve(c4, pot.SolverConfig(epsilon=1e-3, tuning_exponent_p=p, log_every=10 ** 9,
                                                          materialize_plan=False, record_rounded_cost=False,
                                                          max_iterations=200000), ctx=ctx)
        summ(f"c4_tuned_p{p:g}", r, {"host_s": time.perf_counter() - t0})
