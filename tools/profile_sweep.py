"""Small driver for ncu: sets up a BASELINE workload and runs a few ASPOT
iterations + sweep launches (no timing printed is a bench value)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--stored", action="store_true")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
inst = pot.config_instance(args.config, n=args.n)
if args.stored:
    inst.stored = True
cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, record_rounded_cost=False, materialize_plan=False)
s = pot.Session(pot.SolverKind.Aspot, inst, cfg)
s.iterate(args.iters)
ms, el, by = s.time_sweep(args.reps)
print(f"sweep {ms:.4f} ms/launch, {el / ms / 1e6:.1f} Gelem/s, {by / ms / 1e6:.1f} GB/s")
s.close()
