"""Sharded (local shards) vs unsharded fp32 ASPOT at the configs[2] shape,
n = 2048: stopping iteration and rounded cost (feeds the tolerance of
tests/test_gpu_shard.py). Not a test."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

ctx = pot.Context(0)
shard_ctx = {}
for s in (2, 4):
    c = pot.Context(0)
    c.shard_local(s)
    shard_ctx[s] = c
for seed in (1, 2, 3, 4):
    inst = pot.config_instance(3, n=2048, seed=seed)
    cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, materialize_plan=False)
    a = pot.aspot_solve(inst, cfg, ctx=ctx)
    out = {"seed": seed, "it1": a.iterations, "cost1": a.cost}
    for s, c in shard_ctx.items():
        b = pot.aspot_solve(inst, cfg, ctx=c)
        out[f"it{s}"] = b.iterations
        out[f"rel{s}"] = abs(b.cost / a.cost - 1)
        # the same iteration count as the unsharded stop
        b2 = pot.aspot_solve(inst, pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, materialize_plan=False,
                                                    max_iterations=a.iterations), ctx=c)
        out[f"rel{s}_same_it"] = abs(b2.cost / a.cost - 1)
    print(json.dumps(out), flush=True)
