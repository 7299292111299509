#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/debug_net.py > gpurun_out/debug.log 2>&1; echo "debug rc=$?" >> gpurun_out/debug.log
timeout -s KILL 900 python -m pytest tests/test_gpu_ops.py -m gpu -q --tb=line > gpurun_out/pytest_ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops.log
tail -5 gpurun_out/debug.log
