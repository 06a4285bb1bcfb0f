#!/usr/bin/env python
"""Cost of the reference's default trace fidelity (log_every = 1 with
record_rounded_cost, core.hpp:248; every record carries round_pot's cost)
against a plain solve, at configs[2] (n = 16384), K iterations; the
per-record rounding runs as a device tail of the attempt graph.

    python profiles/record_overhead.py [--k 200]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=200)
    ap.add_argument("--config", type=int, default=3)
    args = ap.parse_args()
    ctx = pot.Context(0)
    inst = pot.config_instance(args.config)
    eps = 1e-2 if args.config != 4 else 1e-3
    out = {}
    for name, le, rc in (("plain", 10 ** 9, False), ("log_every_1", 1, True), ("log_every_10", 10, True)):
        cfg = pot.SolverConfig(epsilon=eps, log_every=le, max_iterations=args.k, record_rounded_cost=rc,
                               materialize_plan=False)
        pot.aspot_solve(inst, cfg, ctx=ctx, trace_cap=args.k + 2)  # warm
        t0 = time.perf_counter()
        g = pot.aspot_solve(inst, cfg, ctx=ctx, trace_cap=args.k + 2)
        out[name] = {"wall_s": time.perf_counter() - t0, "loop_s": g.loop_seconds, "records": len(g.trace),
                     "last_rounded_cost": g.trace[-1].rounded_cost}
    out["ratio_log_every_1"] = out["log_every_1"]["wall_s"] / out["plain"]["wall_s"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
