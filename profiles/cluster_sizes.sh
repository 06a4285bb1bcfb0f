# points sweep: row-partial cluster merge size (POTGPU_PTS_CLUSTER), iteration rate C3/C4 and sweep time
for c in 1 8 4 2 8; do
  POTGPU_PTS_CLUSTER=$c python - <<'PY'
import os, json
from paper_2601_17196_b200 import pot
ctx = pot.Context(0)
out = {"cluster": int(os.environ["POTGPU_PTS_CLUSTER"])}
for cid, eps, k in ((3, 1e-2, 60), (4, 1e-3, 6)):
    inst = pot.config_instance(cid)
    cfg = pot.SolverConfig(epsilon=eps, log_every=10**9, max_iterations=10**7, record_rounded_cost=False, materialize_plan=False)
    s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
    s.iterate(3)
    ms, it, _ = s.iterate(k)
    sw = s.time_sweep(20)[0]
    s.close()
    out[f"C{cid}_sweep_ms"] = round(sw, 4); out[f"C{cid}_it_s"] = round(it / ms * 1e3, 1)
print(json.dumps(out))
PY
done
