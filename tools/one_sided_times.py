"""One-sided pass time (both blocks), full sweep time and ASPOT it/s of the
current build at C3 / C4, one JSON line (A/B of sweep_pts1_f32 variants)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
ctx = pot.Context(0)
out = {"tag": tag}
for cid in (3, 4):
    inst = pot.config_instance(cid)
    cfg = pot.SolverConfig(epsilon=1e-3 if cid == 4 else 1e-2, log_every=10 ** 9, max_iterations=10 ** 7,
                           record_rounded_cost=False, materialize_plan=False)
    s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
    s.iterate(3)
    ms, it, _ = s.iterate(60 if cid != 4 else 8)
    out[f"C{cid}_it_s"] = round(it / ms * 1e3, 1)
    out[f"C{cid}_sweep_ms"] = round(s.time_sweep(10)[0], 4)
    out[f"C{cid}_one_u_ms"] = round(s.time_one_sided(0, 10), 4)
    out[f"C{cid}_one_v_ms"] = round(s.time_one_sided(1, 10), 4)
    s.close()
print(json.dumps(out))
