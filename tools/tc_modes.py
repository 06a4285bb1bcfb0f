"""sweep_tc_f32 timing experiments ($POTGPU_TC_DEBUG, each in its own
process): 0 normal, 1 no exponentials (max pass), 2 no MMA (consumers
alone on stale TMEM), 3 no MUFU (FADD instead). Not a test."""
import os
import subprocess
import sys

SNIP = r"""
import sys
sys.path.insert(0, %r)
from paper_2601_17196_b200 import pot
inst = pot.config_instance(3, n=16384)
cfg = pot.SolverConfig(epsilon=1e-2, log_every=10 ** 9, record_rounded_cost=False, materialize_plan=False)
s = pot.Session(pot.SolverKind.Aspot, inst, cfg)
s.iterate(3)
print(s.time_sweep(20)[0])
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for mode in ("0", "1", "2", "3"):
    e = dict(os.environ)
    e["POTGPU_TC_DEBUG"] = mode
    r = subprocess.run([sys.executable, "-c", SNIP], env=e, capture_output=True, text=True, timeout=300)
    print("mode", mode, r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-500:])
