"""Debug probe for the cluster batch kernel (not a test): a few configs[4]
problems with a bounded iteration count, per cluster size / fusion switch
given in the environment; prints iterations, status, sweeps, cost."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
insts = [pot.config_instance(5, seed=1 + i) for i in range(k)]
cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, max_iterations=int(os.environ.get("MAXIT", "1500")),
                       materialize_plan=False, record_rounded_cost=False, collect_iter_log=True)
t0 = time.perf_counter()
res = pot.solve_batched(pot.SolverKind.Aspot, insts, cfg, iter_log_cap=5000)
dt = time.perf_counter() - t0
for r in res:
    lg = r.iter_log
    print(json.dumps({"it": r.iterations, "status": int(r.status), "sweeps": r.sweeps, "attempts": r.attempts,
                      "cost": r.cost, "err": r.final_error,
                      "keep": float(lg[:, 3].mean()) if len(lg) else None,
                      "bh_w": float((lg[:, 2] == 2).mean()) if len(lg) else None,
                      "bc_w": float((lg[:, 4] == 2).mean()) if len(lg) else None}))
print("wall", dt)
