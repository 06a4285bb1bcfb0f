for t in 4 2 1 4 1; do
  POTGPU_EVAL_TPI=$t timeout 300 python profiles/perf_matrix.py --iters 60 2>&1 | python -c "
import sys,json
out=[]
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if d['solver']=='Aspot': out.append(f\"C{d['config']}:{round(d['it_per_s'] or 0,0)}\")
print('tpi=$t', ' '.join(out))
"
done
