#!/usr/bin/env python
"""Where the end-to-end time of one public-API call goes (C3, K iterations):
session begin (upload, validation, setup, first evaluation, graph capture),
iterate(K), finish (rounding + download), host wall clock around each.

    python profiles/e2e_breakdown.py [--k 20]
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
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--config", type=int, default=3)
    args = ap.parse_args()
    ctx = pot.Context(0)
    inst = pot.config_instance(args.config)
    cfg = pot.SolverConfig(epsilon=1e-2 if args.config != 4 else 1e-3, log_every=10 ** 9, max_iterations=args.k,
                           record_rounded_cost=False, materialize_plan=False)
    pot.aspot_solve(inst, cfg, ctx=ctx)  # warm (module load, first-touch allocations)
    out = {}
    for rep in range(2):
        t0 = time.perf_counter()
        s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
        t1 = time.perf_counter()
        ms, it, fin = s.iterate(-1)
        t2 = time.perf_counter()
        r = s.finish()
        t3 = time.perf_counter()
        s.close()
        t4 = time.perf_counter()
        full = pot.aspot_solve(inst, cfg, ctx=ctx)
        t5 = time.perf_counter()
        out = {"begin_ms": (t1 - t0) * 1e3, "iterate_ms": (t2 - t1) * 1e3, "iterate_device_ms": ms,
               "iterations": it, "finish_ms": (t3 - t2) * 1e3, "close_ms": (t4 - t3) * 1e3,
               "aspot_solve_ms": (t5 - t4) * 1e3, "wall_seconds_reported": full.wall_seconds,
               "e2e_it_per_s": full.iterations / (t5 - t4)}
        print(json.dumps(out))


if __name__ == "__main__":
    main()
