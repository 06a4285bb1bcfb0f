#!/bin/bash
# Profile recipe (B200_PROFILING.md): bench line, launch list, one full ncu
# capture of each hot kernel. Run on the GPU box from the repo root:
#   gpurun -- 'bash profiles/run_profile.sh'
# Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/rNN/.
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
# launch list of a short bench (per-launch times are cold-cache, serialised)
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
# full captures: the on-the-fly sweep mid-loop, the stored sweep, the point evaluation
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:sweep_pts2_f32" --launch-skip 12 --launch-count 1 -o $OUT/sweep_points -f \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_points.log 2>&1; echo "points rc=$?"
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:sweep_f32<potgpu::SrcDenseF32>" --launch-skip 4 --launch-count 1 -o $OUT/sweep_stored -f \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_stored.log 2>&1; echo "stored rc=$?"
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_point_eval" --launch-skip 20 --launch-count 1 -o $OUT/point_eval -f \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_eval.log 2>&1; echo "eval rc=$?"
