"""K1'' / one-sided / sharded variants of one fp32 points solve at a small n,
with the fp64 oracle on the same instance: stopping iteration, cost and the
first iteration at which the decision logs or E_t part ways (GPU box)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SNIPPET = r"""
import json, sys
sys.path.insert(0, %r)
from paper_2601_17196_b200 import pot
cfg_id, n, iters, eps, shards = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
inst = pot.config_instance(cfg_id, n=n)
ctx = pot.Context(0)
if shards > 1:
    ctx.shard_local(shards)
cfg = pot.SolverConfig(epsilon=eps, log_every=10 ** 9, max_iterations=iters or 10 ** 6, record_rounded_cost=False,
                       materialize_plan=False, collect_iter_log=True)
r = pot.aspot_solve(inst, cfg, ctx=ctx, iter_log_cap=100000)
print(json.dumps({"status": int(r.status), "iterations": r.iterations, "cost": r.cost, "gap": r.feasibility_gap,
                  "sweeps": r.sweeps, "log": r.iter_log.tolist()}))
""" % ROOT


def run(env_extra, *args):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SNIPPET] + [str(a) for a in args], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        print(r.stderr[-2000:])
        raise SystemExit(1)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    d["log"] = np.array(d["log"])
    return d


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-2
    res = {}
    for name, env, sh in (("default", {}, 1), ("k1pp0", {"POTGPU_K1PP": "0"}, 1), ("onesided0", {"POTGPU_ONE_SIDED": "0"}, 1),
                          ("shard4", {}, 4), ("shard2", {}, 2)):
        res[name] = run(env, cfg_id, n, 0, eps, sh)
    sys.path.insert(0, ROOT)
    from paper_2601_17196_b200 import pot
    from oracle import binding
    inst = pot.config_instance(cfg_id, n=n)
    C = pot.dense_cost(inst.X, inst.Y, inst.cost_scale)
    o = binding.solve(0, inst.r, inst.c, inst.s, C=C, epsilon=eps, log_every=10 ** 9, want_plan=False)
    print(json.dumps({"oracle": {"iterations": o.iterations, "cost": o.cost}}))
    ol = np.asarray(o.log)
    base = res["onesided0"]
    for name, d in res.items():
        k = min(len(d["log"]), len(base["log"]))
        dec = np.where(np.any(d["log"][:k, 2:5] != base["log"][:k, 2:5], axis=1))[0]
        rel = np.abs(d["log"][:k, 5] - base["log"][:k, 5]) / np.abs(base["log"][:k, 5])
        ko = min(len(d["log"]), len(ol))
        deco = np.where(np.any(d["log"][:ko, 2:5] != ol[:ko, 2:5], axis=1))[0]
        relo = np.abs(d["log"][:ko, 5] - ol[:ko, 5]) / np.abs(ol[:ko, 5])
        print(json.dumps({"variant": name, "iterations": d["iterations"], "cost": d["cost"], "gap": d["gap"], "sweeps": d["sweeps"],
                          "rel_cost_vs_oracle": abs(d["cost"] - o.cost) / abs(o.cost),
                          "first_decision_diff_vs_full": int(dec[0]) if len(dec) else None,
                          "max_rel_Et_vs_full": float(rel.max()), "rel_Et_at": [float(rel[min(i, k - 1)]) for i in (10, 100, 500, 1000, k - 1)],
                          "first_decision_diff_vs_oracle": int(deco[0]) if len(deco) else None,
                          "rel_Et_vs_oracle_at": [float(relo[min(i, ko - 1)]) for i in (10, 100, 500, 1000, ko - 1)],
                          "last_Et": d["log"][-3:, 5].tolist()}))


if __name__ == "__main__":
    main()
