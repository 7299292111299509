#!/bin/bash
# the full single-conv sweep (vcnn-bench/1) + compute-sanitizer over every kernel family
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out/sweep gpurun_out/sanitizer
timeout -s KILL 1500 python scripts/sweep.py --out gpurun_out/sweep > gpurun_out/sweep/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep/sweep.log
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/$tool.log
done
tail -n 3 gpurun_out/sweep/sweep.log; for t in memcheck racecheck synccheck; do echo "== $t"; tail -n 4 gpurun_out/sanitizer/$t.log; done
