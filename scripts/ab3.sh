#!/bin/bash
# A/B of an env switch: single- vs multi-step graph step time + bench value
cd "$(dirname "$0")/.." || exit 1
for r in 1 2; do
for cfg in "${ENVA:-X=1}" "${ENVB:-X=1}"; do
  env TAG=$cfg $cfg timeout -s KILL 120 python scripts/dbg_l0.py 2>&1 | tail -1
done; done
bash scripts/ab_value.sh
