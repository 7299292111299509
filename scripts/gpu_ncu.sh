#!/bin/bash
# ncu: per-launch durations of one training step; with FULL=1 also a full
# capture of the tcgen05 kernels (SKIP / COUNT / KREGEX select them).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph ${BENCH_ARGS}"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c ${LCOUNT:-60} --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
if [ -n "$FULL" ]; then
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:${KREGEX:-tc_gemm} -s ${SKIP:-0} -c ${COUNT:-6} -o gpurun_out/prof $B > gpurun_out/ncu_full.log 2>&1
fi
