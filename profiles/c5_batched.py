#!/usr/bin/env python
"""BASELINE configs[4] as the reference quotes it: 256 independent problems,
n = 2048, fp32 stored C (per-problem seeds), solved to convergence through
the batched public entry point (potgpu_solve_batched), reported as
problems/s (host wall time of the whole call: upload of the 256 fp32 costs,
setup, the solves, rounding, download), with the stored-C sweep traffic it
implies (sweeps x n^2 x 4 B / wall) against the HBM roofline.

    python profiles/c5_batched.py [--count 256] [--concurrency 8,16,32] > gpurun_out/c5.jsonl
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
    ap.add_argument("--count", type=int, default=256)
    ap.add_argument("--concurrency", default="8,16,32")
    ap.add_argument("--solvers", default="aspot,tuned")
    args = ap.parse_args()
    ctx = pot.Context(0)
    t0 = time.perf_counter()
    insts = [pot.config_instance(5, seed=1 + k) for k in range(args.count)]
    gen_s = time.perf_counter() - t0
    n = insts[0].size()
    peaks_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    hbm = json.load(open(peaks_path)).get("hbm_gbs", 6650.0) if os.path.exists(peaks_path) else 6650.0
    for name in args.solvers.split(","):
        kind, p = (pot.SolverKind.Aspot, 1.0) if name == "aspot" else (pot.SolverKind.TunedSinkhorn, 4.0)
        cfg = pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=p, log_every=10 ** 9, materialize_plan=False,
                               record_rounded_cost=False)
        pot.solve_batched(kind, insts[:4], cfg, ctx=ctx, concurrency=4)  # warm: modules, caches
        for conc in (int(c) for c in args.concurrency.split(",")):
            t0 = time.perf_counter()
            res = pot.solve_batched(kind, insts, cfg, ctx=ctx, concurrency=conc)
            wall = time.perf_counter() - t0
            iters = sum(r.iterations for r in res)
            sweeps = sum(r.sweeps for r in res)
            conv = sum(1 for r in res if r.status == pot.SolveStatus.Converged)
            side = n + 1 if kind != pot.SolverKind.Aspot else n  # Sinkhorn sweeps the dummy-augmented plan
            gbs = sweeps * side * side * 4 / wall / 1e9
            print(json.dumps({"config": "configs[4]", "solver": name, "count": args.count, "n": n,
                              "concurrency": conc, "wall_s": wall, "problems_per_s": args.count / wall,
                              "iterations": iters, "iterations_per_s": iters / wall, "sweeps": sweeps,
                              "converged": conv, "sweep_gb_s": gbs, "hbm_frac": gbs / hbm,
                              "instance_gen_s": gen_s}), flush=True)


if __name__ == "__main__":
    main()
