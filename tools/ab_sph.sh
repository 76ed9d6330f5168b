# sphere configs (icosphere(sub)) against every ab_libs/lib_*.so and the default library
sub=${1:-10}
for lib in "" ab_libs/lib_*.so; do
  MG_LIB=$lib timeout 900 python tools/bench_configs.py --sub $sub --configs sphere 2>/dev/null | grep '^{' | python -c "
import json,sys
for d in map(json.loads, sys.stdin): print('${lib:-base}', d['call'], round(d['kernel_ms'],4), round(d['hbm_frac'],3))"
done
