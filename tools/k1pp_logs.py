"""Dump the ASPOT iteration logs of the K1'' / unfused / full-sweep / sharded
variants of one fp32 points solve (GPU box) to gpurun_out/k1pp_logs.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from k1pp_small import run  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-2
out = {}
for name, env, sh in (("default", {}, 1), ("k1pp0", {"POTGPU_K1PP": "0"}, 1), ("onesided0", {"POTGPU_ONE_SIDED": "0"}, 1),
                      ("shard4", {}, 4), ("shard2", {}, 2)):
    d = run(env, cfg_id, n, 0, eps, sh)
    out[name] = d["log"]
    print(name, d["iterations"], d["cost"], d["sweeps"], flush=True)
np.savez_compressed("gpurun_out/k1pp_logs.npz", **out)
