#!/usr/bin/env python
"""Regenerate tests/golden/solves.json: golden vectors of the CPU oracle
(oracle/, the restatement of the reference's solvers; test infrastructure)
on instances of the reference's own fixture generator make_synthetic_instance
(synthetic.hpp:15-54, regenerated bit-identically from (n, seed, masses)).
The reference itself cannot be built here (no Eigen), so these
vectors pin the oracle against drift and give the GPU tests fixed answers.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding  # noqa: E402

# (n, seed, mass_r, mass_c, s_frac, epsilon): make_scaling_instance's masses
# (synthetic.hpp:58-60) and the acceptance-test style small cases
CASES = [
    (12, 1, 1.0, 1.0, 0.5, 0.05),
    (24, 7, 5.0, 3.0, 0.2, 0.05),
    (40, 3, 1.0, 1.2, 0.8, 0.02),
    (64, 11, 2.0, 1.5, 0.6, 0.05),
]
SOLVERS = [(0, "aspot", 1.0), (1, "feasible_sinkhorn", 1.0), (2, "tuned_sinkhorn", 2.0)]


def instance_digest(r, c, C, s):
    h = hashlib.sha256()
    for a in (r, c, C, np.array([s])):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def log_digest(log):
    ints = np.ascontiguousarray(log[:, :5], dtype=np.int64)  # t, halvings, block_hat, zbest_is_check, block_check
    return hashlib.sha256(ints.tobytes()).hexdigest()


def main():
    out = {"generator": "tests/golden/make_golden.py", "oracle": "oracle/pot_oracle.hpp (fp64, -ffp-contract=off)",
           "cases": []}
    for n, seed, mr, mc, sf, eps in CASES:
        r, c, C, s = binding.make_synthetic(n, seed, mr, mc, sf)
        case = {"n": n, "seed": seed, "mass_r": mr, "mass_c": mc, "s_frac": sf, "epsilon": eps,
                "instance_sha256": instance_digest(r, c, C, s), "s": s, "results": {}}
        for kind, name, p in SOLVERS:
            o = binding.solve(kind, r, c, s, C=C, epsilon=eps, p=p, log_every=10 ** 9)
            res = {"status": o.status, "iterations": o.iterations, "gamma": o.gamma, "tolerance": o.tolerance,
                   "final_error": o.final_error, "cost": o.cost, "feasibility_gap": o.feasibility_gap,
                   "mass": o.mass, "plan_row_sums": [float(x) for x in o.plan.sum(axis=1)],
                   "plan_col_sums": [float(x) for x in o.plan.sum(axis=0)]}
            if kind == 0:
                res["decision_log_sha256"] = log_digest(o.log)
                res["decisions_head"] = [[int(v) for v in row[:5]] for row in o.log[:12]]
            case["results"][name] = res
        out["cases"].append(case)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "solves.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
