"""Small driver for ncu: sets up a BASELINE workload, runs a few ASPOT
iterations, then brackets `reps` UNGATED sweep launches of the current point
(Session.time_sweep) with cudaProfilerStart/Stop, so that
`ncu --profile-from-start off` captures a real hot-loop launch and never one
of the loop's gated early-exit launches. No timing printed here is a bench
value.

    ncu --profile-from-start off --set full ... python tools/profile_sweep.py --config 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402  (cudaProfilerStart/Stop)
from paper_2601_17196_b200 import pot  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--stored", action="store_true")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
torch.cuda.init()
inst = pot.config_instance(args.config, n=args.n)
if args.stored:
    inst.stored = True
    inst.dtype = pot.DType.F32
cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, record_rounded_cost=False, materialize_plan=False)
s = pot.Session(pot.SolverKind.Aspot, inst, cfg)
s.iterate(args.iters)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ms, el, by = s.time_sweep(args.reps)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"sweep {ms:.4f} ms/launch, {el / ms / 1e6:.1f} Gelem/s, {by / ms / 1e6:.1f} GB/s")
s.close()
