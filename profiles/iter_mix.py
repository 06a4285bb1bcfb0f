#!/usr/bin/env python
"""Mix of the ASPOT iteration paths at a config (GPU box): how often z_hat's
and z_check''s Greenkhorn blocks are u / v / w, how often z_best = z_check,
and the sweeps per iteration -- the inputs of the sweep-count design.

    python profiles/iter_mix.py [--config 3] [--iters 0 (to convergence)]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--iters", type=int, default=0)
    args = ap.parse_args()
    inst = pot.config_instance(args.config, n=args.n) if args.n else pot.config_instance(args.config)
    eps = {1: 1e-2, 2: 1e-3, 3: 1e-2, 4: 1e-3, 5: 1e-2}[args.config]
    cfg = pot.SolverConfig(epsilon=eps, log_every=10 ** 9, max_iterations=args.iters or 10 ** 6,
                           record_rounded_cost=False, materialize_plan=False, collect_iter_log=True)
    r = pot.aspot_solve(inst, cfg, iter_log_cap=200000)
    lg = r.iter_log
    mix = collections.Counter()
    for row in lg:
        mix[(int(row[2]), int(row[3]), int(row[4]))] += 1
    out = {"config": args.config, "n": inst.size(), "iterations": r.iterations, "sweeps": getattr(r, "sweeps", None),
           "mix (block_hat, zbest_is_check, block_check)": {str(k): v for k, v in sorted(mix.items())}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
