"""Five C4 ASPOT iterations through the session API (launch-list target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402

ctx = pot.Context(0)
inst = pot.config_instance(4)
cfg = pot.SolverConfig(epsilon=1e-3, log_every=10 ** 9, max_iterations=10 ** 6, record_rounded_cost=False,
                       materialize_plan=False)
s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
s.iterate(2)
print(s.iterate(3))
