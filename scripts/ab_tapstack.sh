cd /root/repo
for cfg in "VCNN_TAPSTACK=0" "VCNN_TS_R=0" "VCNN_TS_R=6" "VCNN_TS_R=6 VCNN_TS_NBUF=2" "VCNN_TS_R=4 VCNN_TS_NBUF=2" "VCNN_TS_NBUF=2"; do
  env $cfg timeout -s KILL 120 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/l.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-infer --no-faithful --no-roofline-run > /dev/null 2>&1
  echo "== $cfg: $(python scripts/launches.py gpurun_out/l.csv 2>/dev/null | grep direct_conv | head -2 | awk '{print $1}' | tr '\n' ' ')"
  env $cfg timeout -s KILL 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-faithful --no-roofline-run --no-infer 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   value', round(l['value']), 'e2e', round(l['e2e']['value']))"
done
