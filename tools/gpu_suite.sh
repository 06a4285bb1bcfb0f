#!/bin/bash
# The GPU suite file by file, each under its own timeout, with per-test
# durations (finds slow or hanging tests without losing the whole run).
#   gpurun -- 'bash tools/gpu_suite.sh [timeout_per_file]'
T=${1:-900}
mkdir -p gpurun_out
: > gpurun_out/suite_summary.txt
for f in tests/test_gpu_*.py; do
  s=$(date +%s)
  timeout -s INT $T python -m pytest "$f" -m gpu -q -p no:cacheprovider --durations=8 > "gpurun_out/suite_$(basename $f .py).log" 2>&1
  rc=$?
  e=$(( $(date +%s) - s ))
  echo "$f rc=$rc ${e}s $(tail -1 gpurun_out/suite_$(basename $f .py).log)" | tee -a gpurun_out/suite_summary.txt
done
