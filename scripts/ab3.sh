#!/bin/bash
# step time (one- and multi-step graphs) and bench value of the current build
cd "$(dirname "$0")/.." || exit 1
for r in 1 2 3; do
  timeout -s KILL 120 python scripts/dbg_l0.py 2>&1 | tail -1
  timeout -s KILL 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-faithful --no-roofline-run --no-infer 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', round(l['value']), 'e2e', round(l['e2e']['value']), 'ms', round(l['ms_per_step']*1000,1))"
done
