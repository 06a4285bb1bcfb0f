#!/bin/bash
# Profile recipe (B200_PROFILING.md): bench line, launch list, one full ncu
# capture of each hot kernel. Run on the GPU box from the repo root:
#   gpurun -- 'bash profiles/run_profile.sh'
# Outputs land in gpurun_out/ (scratch); profiles/summarize_ncu.py copies the
# summaries to profiles/rNN/.
#
# The full captures use `--profile-from-start off`: tools/profile_sweep.py
# brackets UNGATED sweep launches of a mid-solve point (Session.time_sweep,
# after 20 iterations) with cudaProfilerStart/Stop, so the capture can never
# land on one of the loop's gated early-exit launches (round-1 mistake).
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
FULL="--set full --clock-control none --import-source on --kernel-name-base demangled --profile-from-start off --launch-count 1"
python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
# launch list of a short bench (per-launch times are cold-cache, serialised)
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
# full captures: the on-the-fly sweep, the stored sweep, the point evaluation
$NCU $FULL -k "regex:sweep_pts" -o $OUT/sweep_points -f \
  python tools/profile_sweep.py --config 3 > $OUT/ncu_points.log 2>&1; echo "points rc=$?"
$NCU $FULL -k "regex:sweep_f32" -o $OUT/sweep_stored -f \
  python tools/profile_sweep.py --config 3 --stored > $OUT/ncu_stored.log 2>&1; echo "stored rc=$?"
# the fused one-sided pass (z_check' + the next z_bar, K1''): launches inside the loop; the
# summariser keeps the longest (the gated early-exit launches are a few us)
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:sweep_pts1" --launch-skip 4 --launch-count 6 -o $OUT/sweep_pts1 -f \
  python bench.py --steps 6 --warmup 6 --no-tte --no-cpu > $OUT/ncu_pts1.log 2>&1; echo "pts1 rc=$?"
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_point_eval" --launch-skip 20 --launch-count 1 -o $OUT/point_eval -f \
  python bench.py --steps 3 --warmup 3 --no-tte --no-cpu > $OUT/ncu_eval.log 2>&1; echo "eval rc=$?"
