#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_run.py)
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/$tool.log
done
for t in memcheck racecheck synccheck; do echo "== $t"; tail -n 4 gpurun_out/sanitizer/$t.log; done
