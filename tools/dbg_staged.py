import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_00406_b200 as mg
from paper_2509_00406_b200.apps import ClothConfig, cloth_problem, default_pins, lumped_masses
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
pos, faces = mg.grid_arrays(n, 1.0 / (n - 1))
mesh = mg.Mesh(pos, faces)
rng = np.random.default_rng(3)
target = pos + 0.01 / (n - 1) * rng.normal(size=pos.shape)
x = (pos + 0.01 / (n - 1) * rng.normal(size=pos.shape)).ravel()
cfg = ClothConfig(grid_n=n, spacing=1.0 / (n - 1))
p = cloth_problem(cfg, mesh, target, masses=lumped_masses(mesh, 1.0), pinned=default_pins(n))
p.x = x
e = p.eval_terms()
v = torch.from_numpy(rng.normal(size=x.size)).cuda()
mv = p.hess.matvec(v)
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    hv = p.hvp(p.x_device, v)
    d = (hv - mv).abs()
    bad = torch.nonzero(d > 1e-8 * float(mv.abs().max())).flatten()
    print(k, "bad entries", bad.numel(), (bad[:10] // 3).tolist(), float(d.max()))
    torch.cuda.synchronize()
