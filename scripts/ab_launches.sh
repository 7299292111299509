#!/bin/bash
# A/B of the per-kernel launch durations of the CIFAR-3 b128 step (ncu, serialised)
# usage: ENVA="..." ENVB="..." bash scripts/ab_launches.sh
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-infer --no-faithful --no-roofline-run"
for v in A B; do
  eval "env \${ENV$v} timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c ${LCOUNT:-40} --csv --log-file gpurun_out/launches_$v.csv $B" > /dev/null 2>&1
  python scripts/launches.py gpurun_out/launches_$v.csv > gpurun_out/launches_$v.txt 2>&1
  echo "== $v (${ENVA:+A=$ENVA} ${ENVB:+B=$ENVB})"; tail -n 14 gpurun_out/launches_$v.txt
done
for v in A B; do eval "env \${ENV$v} timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-faithful --no-roofline-run --no-infer" 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v value', round(l['value']), 'e2e', round(l['e2e']['value']))"; done
