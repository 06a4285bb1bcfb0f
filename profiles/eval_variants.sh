set -u
OUT=gpurun_out; mkdir -p $OUT
for b in 0 1 2 4; do
  if [ $b = 0 ]; then unset POTGPU_EVAL_BLOCKS_PER_SM; else export POTGPU_EVAL_BLOCKS_PER_SM=$b; fi
  python profiles/sweep_times.py --tag evalbps$b >> $OUT/times.jsonl 2>&1
done
unset POTGPU_EVAL_BLOCKS_PER_SM
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 120 --csv --log-file $OUT/launches_warm2.csv \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_warm2.log 2>&1; echo "warm rc=$?"
timeout 900 python -m pytest tests/test_gpu_aspot.py tests/test_gpu_edges.py tests/test_gpu_dual_api.py -x -q > $OUT/gpu_tests_ctl.log 2>&1; echo tests rc=$?; tail -2 $OUT/gpu_tests_ctl.log
cat $OUT/times.jsonl
