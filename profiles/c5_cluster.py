#!/usr/bin/env python
"""configs[4] through the one-problem-per-cluster kernel (csrc/batch_cluster.cuh):
wall time of the batched call and, from POTGPU_TRACE_SETUP, the host
upload/setup time and the kernel's device time, for cluster sizes and
resident-cluster caps. Kernel-side sweep traffic = sweeps x n^2 x 4 B.

    python profiles/c5_cluster.py [--count 256] > gpurun_out/c5_cluster.jsonl
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
    ap.add_argument("--variants", default="0:0,2:0,4:0,1:0")
    args = ap.parse_args()
    ctx = pot.Context(0)
    insts = [pot.config_instance(5, seed=1 + k) for k in range(args.count)]
    n = insts[0].size()
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, materialize_plan=False, record_rounded_cost=False)
    os.environ["POTGPU_TRACE_SETUP"] = "1"
    pot.solve_batched(pot.SolverKind.Aspot, insts[:8], cfg, ctx=ctx)  # warm
    for v in args.variants.split(","):
        cs, cap = v.split(":")
        os.environ["POTGPU_BC_CS"] = cs  # 0: automatic
        os.environ["POTGPU_BC_CLUSTERS"] = cap
        t0 = time.perf_counter()
        res = pot.solve_batched(pot.SolverKind.Aspot, insts, cfg, ctx=ctx)
        wall = time.perf_counter() - t0
        sweeps = sum(r.sweeps for r in res)
        iters = sum(r.iterations for r in res)
        print(json.dumps({"cs": int(cs), "cap": int(cap), "wall_s": wall, "problems_per_s": args.count / wall,
                          "iterations": iters, "sweeps": sweeps, "sweep_bytes": sweeps * n * n * 4,
                          "converged": sum(1 for r in res if r.status == pot.SolveStatus.Converged)}), flush=True)


if __name__ == "__main__":
    main()
