# face CTA kernel: parity + A/B timing against the per-row kernel
mkdir -p gpurun_out
tag=${1:-r2j}
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_parity_gpu.py tests/test_distributed_gpu.py tests/test_distributed_mp_gpu.py tests/test_drivers_gpu.py -x -q > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for v in 1 0; do
  MG_FV_CTA=$v timeout 900 python tools/bench_configs.py --sub 10 --configs dirichlet 2>/dev/null | grep '^{' | python -c "
import json,sys
for d in map(json.loads, sys.stdin): print('cta=$v', d['call'], round(d['kernel_ms'],4), round(d['hbm_frac'],3))"
done > gpurun_out/ab_${tag}.txt
tail -3 gpurun_out/pytest_${tag}.log; cat gpurun_out/ab_${tag}.txt
