"""Quick device check of the tensor-core points sweep against the CUDA-core
one (run on the GPU box): sweep time of each and the first iterations'
E_t / phi. Not a test; tests/test_gpu_carry.py is."""
import json
import os
import subprocess
import sys

SNIP = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
from paper_2601_17196_b200 import pot
ctx = pot.Context(0)
n = int(sys.argv[1])
inst = pot.config_instance(3, n=n)
cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, max_iterations=10 ** 6, record_rounded_cost=False,
                       materialize_plan=False, collect_iter_log=True)
s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx, iter_log_cap=1000)
ms, it, fin = s.iterate(30)
c1 = s.carry_stats()
sw = s.time_sweep(20)
r = s.finish()
print(json.dumps({"ms30": ms, "carry": c1, "sweep_ms": sw[0], "log": r.iter_log[:30, 5:8].tolist()}))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

for n in (4096, 16384):
    out = {}
    for name, env in (("tc", {}), ("cuda", {"POTGPU_TC": "0"})):
        e = dict(os.environ)
        e.update(env)
        r = subprocess.run([sys.executable, "-c", SNIP, str(n)], env=e, capture_output=True, text=True, timeout=600)
        if r.returncode != 0:
            print(name, n, "FAILED", r.stderr[-3000:])
            continue
        out[name] = json.loads(r.stdout.strip().splitlines()[-1])
        print(name, n, "sweep ms", out[name]["sweep_ms"], "30 it ms", out[name]["ms30"], "carry", out[name]["carry"])
    if len(out) == 2:
        import numpy as np
        a, b = np.array(out["tc"]["log"]), np.array(out["cuda"]["log"])
        print("max rel diff E/phi_check/phi_hat:", (np.abs(a - b) / np.abs(b)).max(axis=0))
