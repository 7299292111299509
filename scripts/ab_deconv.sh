#!/bin/bash
# deconv-121 b16 step + top ops under env settings
cd "$(dirname "$0")/.." || exit 1
for c in "${ENVA:-X=1}" "${ENVB:-X=1}"; do
  env $c timeout -s KILL 300 python bench.py --config deconv121 --batch 16 --steps 10 --warmup 3 --no-cpu-baseline --no-faithful --no-roofline-run --no-infer --details gpurun_out/d.json 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(l['value']), 'img/s', round(l['ms_per_step']*1000,1), 'us')"
  python -c "
import json; d=json.load(open('gpurun_out/d.json'))
for r in sorted(d['ops'], key=lambda r:-r['us'])[:4]: print('  ', r['layer'], r['op'], round(r['us'],1), 'us', round(r.get('tflops',0),1), 'TF/s')
"
done
