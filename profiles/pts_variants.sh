# points-sweep column pairs per lane (POTGPU_PTS_PAIRS), C3 and C4 sweep times
for v in 8 2; do
  POTGPU_PTS_PAIRS=$v python - <<'PY'
import os, json
from paper_2601_17196_b200 import pot
ctx = pot.Context(0)
out = {"pairs": int(os.environ["POTGPU_PTS_PAIRS"])}
for cid, eps in ((3, 1e-2), (4, 1e-3)):
    inst = pot.config_instance(cid)
    cfg = pot.SolverConfig(epsilon=eps, log_every=10**9, max_iterations=10**7, record_rounded_cost=False, materialize_plan=False)
    s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
    s.iterate(3)
    ms, it, _ = s.iterate(30 if cid == 3 else 5)
    sw = s.time_sweep(20)[0]
    s.close()
    out[f"C{cid}_sweep_ms"] = round(sw, 4); out[f"C{cid}_it_s"] = round(it / ms * 1e3, 1)
print(json.dumps(out))
PY
done
