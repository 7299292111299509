#!/bin/bash
# bench value A/B under env settings (3 alternating runs each)
cd "$(dirname "$0")/.." || exit 1
for r in 1 2 3; do
for cfg in "${ENVA:-X=1}" "${ENVB:-X=1}"; do
  env $cfg timeout -s KILL 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-faithful --no-roofline-run --no-infer 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', 'value', round(l['value']), 'e2e', round(l['e2e']['value']), 'ms', round(l['ms_per_step']*1000,1))"
done; done
