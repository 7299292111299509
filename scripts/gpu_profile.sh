#!/bin/bash
# Evidence run: bench line, ncu launch list of one eager step, and one
# `ncu --set full` capture of the dominant kernels.  Bounded by timeouts.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout -s KILL 400 python bench.py --steps 50 --warmup 10 --details gpurun_out/bench_details.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c ${LCOUNT:-60} --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-direct_conv|SlabWgrad} -c ${COUNT:-5} -o gpurun_out/prof $B > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/bench.log gpurun_out/bench_ref.log
