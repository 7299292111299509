#!/bin/bash
# Round-end evidence: the single-conv sweep (vcnn-bench/1), the other BASELINE
# configs' bench lines, sanitizer.  Each step bounded.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out/sweep gpurun_out/configs
timeout -s KILL 1500 python scripts/sweep.py --out gpurun_out/sweep > gpurun_out/sweep/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep/sweep.log
for c in "deconv121 --batch 16" "denoise16 --batch 128" "single-conv --batch 128 --channels 64 --ksize 5"; do
  n=$(echo $c | cut -d' ' -f1)
  timeout -s KILL 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-faithful --no-roofline-run --details gpurun_out/configs/$n.details.json > gpurun_out/configs/$n.log 2>&1
done
tail -n 2 gpurun_out/sweep/sweep.log; for f in gpurun_out/configs/*.log; do tail -n 1 $f | cut -c1-200; done
