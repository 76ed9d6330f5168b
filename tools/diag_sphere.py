import sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2509_00406_b200 as mg
from paper_2509_00406_b200.apps import initial_sphere, sphere_problem, tangent_bases
torch.cuda.set_device(0)
def sphere(sub=9):
    pos, faces = mg.icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    base = initial_sphere(mesh); b1, b2 = tangent_bases(base)
    p = sphere_problem(mesh, base, b1, b2)
    p.x = 1e-3 * np.random.default_rng(0).normal(size=2 * len(pos))
    vd = torch.from_numpy(np.random.default_rng(1).normal(size=2 * len(pos))).cuda(); y = torch.empty_like(vd)
    return p, vd, y
p, vd, y = sphere()
print("fresh", bench.time_with_kernel(p, lambda: p.hvp(p.x_device, vd, out=y), 10, 3))
print("fresh again", bench.time_with_kernel(p, lambda: p.hvp(p.x_device, vd, out=y), 10, 3))
q, x, v = bench.build_engine_cloth(1024, "deterministic")
print("after cloth build", bench.time_with_kernel(p, lambda: p.hvp(p.x_device, vd, out=y), 10, 3))
del q; torch.cuda.empty_cache()
print("after cloth del", bench.time_with_kernel(p, lambda: p.hvp(p.x_device, vd, out=y), 10, 3))
p2, vd2, y2 = sphere()
print("second sphere", bench.time_with_kernel(p2, lambda: p2.hvp(p2.x_device, vd2, out=y2), 10, 3))
