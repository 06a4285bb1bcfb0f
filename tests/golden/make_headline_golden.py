#!/usr/bin/env python
"""Regenerate tests/golden/headline.json: the CPU oracle's answers for the
parity tests at the BASELINE sizes, which take the oracle minutes (too long
for every GPU-suite run): configs[3] ASPOT 3-iteration prefix (n = 65536,
points mode), configs[2] fp64 ASPOT 20-iteration prefix (n = 16384, points
mode), configs[1] tuned Sinkhorn p = 1 capped at 300 iterations, configs[3]
tuned Sinkhorn 1-iteration prefix, configs[4] (4 problems) ASPOT and tuned
Sinkhorn to convergence. Each entry carries a digest of its input so a test
fails loudly if the instance recipe changes.

    python tests/golden/make_headline_golden.py   # ~30 min on 8 cores
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding  # noqa: E402
from paper_2601_17196_b200 import pot  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "headline.json")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()[:16]


def res(o):
    return {"status": int(o.status), "iterations": int(o.iterations), "cost": float(o.cost), "phi": float(o.phi),
            "final_error": float(o.final_error), "feasibility_gap": float(o.feasibility_gap),
            "gamma": float(o.gamma), "tolerance": float(o.tolerance),
            "log": np.asarray(o.log).tolist(), "trace": np.asarray(o.trace).tolist()}


def main():
    binding.lib().oracle_set_threads(os.cpu_count() or 1)
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    todo = sys.argv[1:] or ["c4_aspot_prefix", "c3_anchor_prefix", "c2_tuned_p1_capped", "c4_tuned_prefix", "c5"]
    for name in todo:
        t0 = time.time()
        if name == "c4_aspot_prefix":
            inst = pot.config_instance(4)
            scale = pot.points_scale(inst.X, inst.Y, chunk=1024)
            o = binding.solve(0, inst.r, inst.c, inst.s, X=inst.X, Y=inst.Y, scale=scale, epsilon=1e-3,
                              max_iterations=3, skip_plan=True)
            out[name] = dict(res(o), scale=scale, digest=digest(inst.X, inst.Y, inst.r, inst.c, [inst.s]))
        elif name == "c3_anchor_prefix":
            inst = pot.config_instance(3)
            scale = pot.points_scale(inst.X, inst.Y)
            o = binding.solve(0, inst.r, inst.c, inst.s, X=inst.X, Y=inst.Y, scale=scale, epsilon=1e-2,
                              max_iterations=20, skip_plan=True)
            out[name] = dict(res(o), scale=scale, digest=digest(inst.X, inst.Y, inst.r, inst.c, [inst.s]))
        elif name == "c2_tuned_p1_capped":
            inst = pot.config_instance(2)
            o = binding.solve(2, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-3, p=1.0, max_iterations=300,
                              log_every=50, skip_plan=True)
            out[name] = dict(res(o), digest=digest(inst.C, inst.r, inst.c, [inst.s]))
        elif name == "c4_tuned_prefix":
            inst = pot.config_instance(4)
            scale = pot.points_scale(inst.X, inst.Y, chunk=1024)
            o = binding.solve(2, inst.r, inst.c, inst.s, X=inst.X, Y=inst.Y, scale=scale, epsilon=1e-3, p=4.0,
                              max_iterations=1, log_every=1, skip_plan=True)
            out[name] = dict(res(o), scale=scale, digest=digest(inst.X, inst.Y, inst.r, inst.c, [inst.s]))
        elif name == "c5":
            insts = [pot.config_instance(5, seed=1 + k) for k in range(4)]
            for kind, p, tag in ((0, 1.0, "aspot"), (2, 4.0, "tuned")):
                out[f"c5_{tag}"] = []
                for inst in insts:
                    o = binding.solve(kind, inst.r, inst.c, inst.s, C=inst.C, epsilon=1e-2, p=p, want_plan=False)
                    out[f"c5_{tag}"].append(dict(res(o), digest=digest(inst.C, inst.r, inst.c, [inst.s])))
        print(name, f"{time.time() - t0:.0f}s", flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f)


if __name__ == "__main__":
    main()
