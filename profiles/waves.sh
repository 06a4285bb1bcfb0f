for w in 1 2 4 8 16; do
  POTGPU_SWEEP_WAVES=$w python bench.py --no-cpu --no-tte --steps 50 > gpurun_out/bench_w$w.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/bench_w$w.json')); print('waves $w', round(d['value'],1), 'it/s sweep_ms', round(d['roofline']['ms_per_launch'],4), 'stored_ms', round(d['roofline_stored']['ms_per_launch'],4))"
done
