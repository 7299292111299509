#!/bin/bash
# Other BASELINE configs (parity-test cases, not bench lines): one short bench
# line + per-op details each, and a cold launch list per config.  Bounded.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out/sweep
run() {  # name, bench args
  local n=$1; shift
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
      --details gpurun_out/sweep/$n.details.json >> gpurun_out/sweep/lines.jsonl 2> gpurun_out/sweep/$n.err
  if [ -n "$LAUNCHES" ]; then
    timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c ${LCOUNT:-40} --csv \
      --log-file gpurun_out/sweep/$n.launches.csv python bench.py --steps 2 --warmup 1 --no-e2e \
      --no-cpu-baseline --no-graph --no-infer "$@" > /dev/null 2>&1
    python scripts/launches.py gpurun_out/sweep/$n.launches.csv > gpurun_out/sweep/$n.launches.txt 2>&1
  fi
}
all() {
  run lenet-caffe --config lenet-caffe --batch 100
  run scale1-analog --config scale1-analog --batch 100
  run denoise16 --config denoise16 --batch 128
  run deconv121 --config deconv121 --batch 16
  run cifar3-b1024 --config cifar3 --batch 1024
  for ck in "32 5" "64 5" "128 3" "256 3" "128 7" "64 11"; do
    set -- $ck
    run sc-c$1-k$2 --config single-conv --channels $1 --ksize $2 --batch 128
  done
}
eval "${SWEEP:-all}"
