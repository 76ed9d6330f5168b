#!/bin/bash
# A/B of the row processing order (Morton patches vs the caller's numbering),
# and of the staged edge tiles, on every call of the BASELINE configs.
# usage (under gpurun): bash tools/ab_order.sh [grid]
g=${1:-2048}
for ord in morton identity; do
  for tiles in 1 0; do
    for call in psd plain hvp hvp_psd energy; do
      r=$(MG_ROW_ORDER=$ord MG_EDGE_TILES=$tiles timeout 300 python bench.py --only --grid $g --profile-call $call --steps 20 2>&1 | tail -1)
      echo "order=$ord tiles=$tiles grid=$g $r"
    done
  done
  MG_ROW_ORDER=$ord timeout 900 python tools/bench_configs.py --sub 10 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('order=$ord', d['config'], d['call'], round(d['ms'],4), round(d['hbm_frac'],3))"
done
