"""Per-launch device time of the default fp32 points sweep at C3 / C4 sizes
(Session.time_sweep, after a few iterations). Not a test, not a bench line."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

for cfgid, n in ((3, 16384), (4, 65536)):
    inst = pot.config_instance(cfgid, n=n)
    cfg = pot.SolverConfig(epsilon=1e-2 if cfgid == 3 else 1e-3, log_every=10 ** 9, record_rounded_cost=False,
                           materialize_plan=False)
    s = pot.Session(pot.SolverKind.Aspot, inst, cfg)
    ms_it, it, _ = s.iterate(20)
    ms = s.time_sweep(20)[0]
    print(f"C{cfgid} n={n}: sweep {ms:.4f} ms ({n * n / ms / 1e6:.0f} Gex2/s), 20 iterations {ms_it:.3f} ms")
    s.close()
