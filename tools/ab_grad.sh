# A/B of the flat gradient row kernels: config-5 gradient (cloth 7072^2) and the
# smoothing gradient (icosphere(10)), twice, against every ab_libs/lib_*.so and the
# default library. usage (under gpurun): bash tools/ab_grad.sh
for r in 1 2; do
  for lib in "" ab_libs/lib_*.so; do
    MG_LIB=$lib timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import bench, os
out = bench.run_config5(6555.5, 'measured', 7072)
print(os.environ.get('MG_LIB') or 'base', round(out['cloth7072_grad']['kernel_ms'], 4))
" 2>&1 | tail -1
    MG_LIB=$lib timeout 900 python tools/bench_configs.py --sub 10 --configs smooth 2>/dev/null | grep '^{' | python -c "
import json,sys
for d in map(json.loads, sys.stdin):
    if d['call'] == 'eval_terms_grad': print('${lib:-base}', 'smooth_grad', round(d['kernel_ms'],4))"
  done
done
