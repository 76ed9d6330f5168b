#!/bin/bash
# BASELINE configs 3-4 (tools/bench_configs.py) against every ab_libs/lib_*.so
# and the default library. usage (under gpurun): bash tools/ab_cfg.sh <sub> <config> [...]
sub=$1; shift
for lib in "" ab_libs/lib_*.so; do
  MG_LIB=$lib timeout 900 python tools/bench_configs.py --sub $sub --configs "$@" 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('${lib:-base}', d['config'], d['call'], round(d['ms'],4), round(d['kernel_ms'] or 0,4), round(d['hbm_frac'],3))"
done
