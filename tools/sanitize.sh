#!/bin/bash
# compute-sanitizer passes over the round-2 kernels (TMA-staged rings, CTA face
# lists, energy probe, fp32 storage, traced row modules, device PCG).
# usage (under gpurun): bash tools/sanitize.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
CS=compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 1 python -m pytest -x -q \
  tests/test_parity_gpu.py tests/test_odd_sizes_gpu.py tests/test_fp32_gpu.py tests/test_jit_gpu.py tests/test_solvers_gpu.py \
  -k "cloth8 or spring_pinned or dirichlet_ico2 or sphere_ico2 or smooth_ico2 or rectangles or icosphere or float32 or device_cg or rows" \
  > gpurun_out/memcheck_${tag}.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_${tag}.log
cat > /tmp/race.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2509_00406_b200 as mg
from paper_2509_00406_b200.apps import ClothConfig, cloth_problem, default_pins, lumped_masses, distortion_problem, rest_geometry
n = 64
pos, faces = mg.grid_arrays(n, 1.0 / (n - 1)); mesh = mg.Mesh(pos, faces)
rng = np.random.default_rng(0)
p = cloth_problem(ClothConfig(grid_n=n, spacing=1.0 / (n - 1)), mesh, pos + 1e-4 * rng.normal(size=pos.shape),
                  masses=lumped_masses(mesh, 1.0), pinned=default_pins(n))
p.precompute_sparsity(); p.x = (pos + 1e-4 * rng.normal(size=pos.shape)).ravel()
v = torch.from_numpy(rng.normal(size=p.num_dofs)).cuda()
p.eval_terms(psd_floor=1e-9); p.eval_terms(); p.hvp(p.x_device, v); p.hvp(p.x_device, v, psd_floor=1e-9); p.eval_energy_only(p.x_device)
q, qf, uv = mg.punctured_icosphere_arrays(3); qm = mg.Mesh(q, qf)
ri, ar = rest_geometry(qm); d = distortion_problem(qm, ri, ar, with_hessian=True); d.precompute_sparsity(); d.x = uv.ravel()
w = torch.from_numpy(rng.normal(size=d.num_dofs)).cuda()
d.eval_terms(); d.eval_terms(psd_floor=1e-9); d.hvp(d.x_device, w); d.hvp(d.x_device, w, psd_floor=1e-9)
torch.cuda.synchronize(); print("racecheck workload done")
PY
timeout 1500 $CS --tool racecheck --racecheck-report hazard python /tmp/race.py > gpurun_out/racecheck_${tag}.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_${tag}.log
timeout 1500 $CS --tool synccheck python /tmp/race.py > gpurun_out/synccheck_${tag}.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/synccheck_${tag}.log
tail -4 gpurun_out/memcheck_${tag}.log; tail -4 gpurun_out/racecheck_${tag}.log; tail -4 gpurun_out/synccheck_${tag}.log
