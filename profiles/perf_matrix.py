#!/usr/bin/env python
"""Device iterations/s of every solver on every BASELINE config (resident
problem, session API, CUDA-event time of k iterations after warm-up), plus
the sweep-kernel time. A regression table for kernel / grid changes:

    python profiles/perf_matrix.py [--iters 50] [--shards S] > gpurun_out/perf.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

CASES = [  # (config, n, dtype, solver, epsilon, p)
    (1, 1000, pot.DType.F64, pot.SolverKind.Aspot, 1e-2, 1.0),
    (1, 1000, pot.DType.F64, pot.SolverKind.FeasibleSinkhorn, 1e-2, 1.0),
    (2, 4096, pot.DType.F64, pot.SolverKind.Aspot, 1e-3, 1.0),
    (2, 4096, pot.DType.F64, pot.SolverKind.TunedSinkhorn, 1e-3, 4.0),
    (2, 4096, pot.DType.F32, pot.SolverKind.TunedSinkhorn, 1e-3, 4.0),
    (3, 16384, pot.DType.F32, pot.SolverKind.Aspot, 1e-2, 1.0),
    (3, 16384, pot.DType.F32, pot.SolverKind.TunedSinkhorn, 1e-2, 4.0),
    (4, 65536, pot.DType.F32, pot.SolverKind.Aspot, 1e-3, 1.0),
    (4, 65536, pot.DType.F32, pot.SolverKind.TunedSinkhorn, 1e-3, 4.0),
    (5, 2048, pot.DType.F32, pot.SolverKind.Aspot, 1e-2, 1.0),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--shards", type=int, default=1)
    args = ap.parse_args()
    ctx = pot.Context(0)
    if args.shards > 1:
        ctx.shard_local(args.shards)
    for cid, n, dt, kind, eps, p in CASES:
        inst = pot.config_instance(cid, n=n, dtype=dt)
        cfg = pot.SolverConfig(epsilon=eps, tuning_exponent_p=p, log_every=10 ** 9, max_iterations=10 ** 7,
                               record_rounded_cost=False, materialize_plan=False)
        s = pot.Session(kind, inst, cfg, ctx=ctx)
        s.iterate(3)
        ms, it, fin = s.iterate(args.iters)
        sweep_ms, elems, byts = s.time_sweep(10)
        _, _, sweeps = s.stats()
        s.close()
        print(json.dumps({"config": cid, "n": n, "dtype": dt.name, "solver": kind.name, "iters": it,
                          "it_per_s": it / (ms * 1e-3) if ms > 0 else None, "ms_per_it": ms / max(it, 1),
                          "sweep_ms": sweep_ms, "sweep_gelem_s": elems / (sweep_ms * 1e-3) / 1e9,
                          "sweep_gb_s": byts / (sweep_ms * 1e-3) / 1e9 if byts else None, "finished": fin}))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
