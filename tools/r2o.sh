mkdir -p gpurun_out
tag=${1:-r2o}
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_parity_gpu.py tests/test_distributed_gpu.py tests/test_drivers_gpu.py tests/test_jit_gpu.py -x -q > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for v in 1 0; do
  MG_FV_CTA=$v timeout 900 python tools/bench_configs.py --sub 10 --configs sphere 2>/dev/null | grep '^{' | python -c "
import json,sys
for d in map(json.loads, sys.stdin): print('cta=$v', d['config'], d['call'], round(d['kernel_ms'],4), round(d['hbm_frac'],3))"
done > gpurun_out/ab_${tag}.txt 2>&1
tail -3 gpurun_out/pytest_${tag}.log; cat gpurun_out/ab_${tag}.txt
