# face CTA kernel: parity + A/B (incl. gradient-only problems)
mkdir -p gpurun_out
tag=${1:-r2m}
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_parity_gpu.py tests/test_distributed_gpu.py tests/test_distributed_mp_gpu.py tests/test_drivers_gpu.py tests/test_jit_gpu.py -x -q > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for v in 1 0; do
  MG_FV_CTA=$v timeout 900 python tools/bench_configs.py --sub 10 --configs dirichlet 2>/dev/null | grep '^{' | python -c "
import json,sys
for d in map(json.loads, sys.stdin): print('cta=$v', d['call'], round(d['kernel_ms'],4), round(d['hbm_frac'],3))"
  MG_FV_CTA=$v timeout 600 python - <<'PY'
import os, sys, numpy as np, torch, bench
import paper_2509_00406_b200 as mg
from paper_2509_00406_b200.apps import distortion_problem, rest_geometry
pos, faces, uv = mg.punctured_icosphere_arrays(10)
mesh = mg.Mesh(pos, faces)
ri, ar = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in rest_geometry(mesh))
p = distortion_problem(mesh, ri, ar, with_hessian=False)
p.x = uv.ravel()
ms, kms = bench.time_with_kernel(p, lambda: p.eval_terms(sync=False), 10, 3)
print(f"cta={os.environ['MG_FV_CTA']} grad_only {kms:.4f}")
PY
done > gpurun_out/ab_${tag}.txt 2>&1
tail -3 gpurun_out/pytest_${tag}.log; cat gpurun_out/ab_${tag}.txt
