#!/bin/bash
# quick iteration: GPU tests (subset via TESTS), bench line, launch list
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest ${TESTS:-tests -m gpu} -x -q -rf --tb=short > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --details gpurun_out/bench_details.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-infer"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c ${LCOUNT:-40} --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
tail -n 4 gpurun_out/pytest_quick.log; tail -c 600 gpurun_out/bench.log; tail -n 14 gpurun_out/launches_summary.txt
