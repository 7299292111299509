#!/bin/bash
# One GPU session: device info, smoke, gpu tests, short bench, launch list.
# Every step is bounded by its own timeout so a hung kernel cannot wedge the box.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout -s KILL 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -rf --tb=line ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 400 python bench.py --steps 30 --warmup 5 --details gpurun_out/bench_details.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$NCU" ]; then bash scripts/gpu_ncu.sh; fi
if false; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_launch.log 2>&1
fi
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log
