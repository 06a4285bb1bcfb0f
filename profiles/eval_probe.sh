#!/bin/bash
# Warm per-kernel durations of a few C3 ASPOT attempts (no cache flush between
# kernels) and full captures of the two k_point_eval modes (sweep partials /
# scaled). Run on the GPU box from the repo root.
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv --log-file $OUT/launches_warm.csv \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_warm.log 2>&1; echo "warm rc=$?"
for spec in "28 eval_scaled" "26 eval_full"; do
  set -- $spec
  $NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_point_eval" --launch-skip $1 --launch-count 1 -o $OUT/$2 -f \
    python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_$2.log 2>&1; echo "$2 rc=$?"
done
