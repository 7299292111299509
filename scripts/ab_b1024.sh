#!/bin/bash
# A/B of the b1024 conv GEMM table (bench.py's roofline run) under two env settings
cd "$(dirname "$0")/.." || exit 1
for cfg in "${ENVA:-X=1}" "${ENVB:-X=1}"; do
  echo "== $cfg"
  env $cfg timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-faithful --no-infer 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(l['value']))
for r in l.get('conv_gemm_roofline_b1024', []): print('  b1024', r['gemm'], r['us'], 'us', r['tflops'], 'TF/s', r['frac_of_peak'])
"
done
