import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
import paper_2509_00406_b200 as mg
from paper_2509_00406_b200.apps import distortion_problem, rest_geometry, initial_sphere, sphere_problem, tangent_bases
torch.cuda.set_device(0)
def sphere(sub=9):
    pos, faces = mg.icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    base = initial_sphere(mesh); b1, b2 = tangent_bases(base)
    p = sphere_problem(mesh, base, b1, b2)
    p.x = 1e-3 * np.random.default_rng(0).normal(size=2 * len(pos))
    vd = torch.from_numpy(np.random.default_rng(1).normal(size=2 * len(pos))).cuda(); y = torch.empty_like(vd)
    return p, vd, y
def timed(p, vd, y, tag):
    fn = lambda: p.hvp(p.x_device, vd, out=y)
    print(tag, bench.time_with_kernel(p, fn, 10, 3))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print("   host submit ms/call", (t1 - t0) * 100, "total", (t2 - t0) * 100)
p, vd, y = sphere(); timed(p, vd, y, "sphere fresh")
pos, faces, uv = mg.punctured_icosphere_arrays(9)
mesh = mg.Mesh(pos, faces); ri, ar = rest_geometry(mesh)
d = distortion_problem(mesh, ri, ar, with_hessian=True); d.precompute_sparsity(); d.x = uv.ravel()
timed(p, vd, y, "sphere with dirichlet alive")
d.eval_terms(); timed(p, vd, y, "sphere after dirichlet eval")
del d; timed(p, vd, y, "sphere after dirichlet del")
