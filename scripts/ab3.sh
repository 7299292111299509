#!/bin/bash
# layer-0 weight-gradient placement A/B (single- vs multi-step graphs + bench)
cd "$(dirname "$0")/.." || exit 1
for r in 1 2; do
for cfg in VCNN_L0_SIDE=1 X=1; do
  env TAG=$cfg $cfg timeout -s KILL 120 python scripts/dbg_l0.py 2>&1 | tail -1
done; done
ENVA=VCNN_L0_SIDE=1 ENVB=X=1 bash scripts/ab_value.sh
