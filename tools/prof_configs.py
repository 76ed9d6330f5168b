"""One warm-up call, then exactly one call of each BASELINE config 3/4 call,
for ncu (deterministic launch list). usage:
  ncu --set full ... -k regex:'k_rows|k_face|k_sphere' python tools/prof_configs.py --sub 10
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

FLOOR = 1e-9


def main():
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import (distortion_problem, edge_length_problem, initial_sphere, rest_geometry,
                                            sphere_problem, tangent_bases)

    ap = argparse.ArgumentParser()
    ap.add_argument("--sub", type=int, default=10)
    ap.add_argument("--configs", nargs="+", default=["dirichlet", "sphere", "smooth"])
    args = ap.parse_args()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if "dirichlet" in args.configs:
        pos, faces, uv = mg.punctured_icosphere_arrays(args.sub)
        mesh = mg.Mesh(pos, faces)
        ri, ar = (dev(a) for a in rest_geometry(mesh))
        p = distortion_problem(mesh, ri, ar, with_hessian=True)
        p.precompute_sparsity()
        p.x = uv.ravel()
        v = dev(np.random.default_rng(1).normal(size=p.num_dofs))
        p.eval_terms()  # warm-up
        torch.cuda.synchronize()
        p.eval_terms()
        p.eval_terms(psd_floor=FLOOR)
        p.hvp(p.x_device, v)
        p.hvp(p.x_device, v, psd_floor=FLOOR)
        torch.cuda.synchronize()
        del p
    if "sphere" in args.configs or "smooth" in args.configs:
        pos, faces = mg.icosphere_arrays(args.sub)
        mesh = mg.Mesh(pos, faces)
    if "sphere" in args.configs:
        base = initial_sphere(mesh)
        b1, b2 = tangent_bases(base)
        p = sphere_problem(mesh, dev(base), dev(b1), dev(b2))
        p.x = 1e-5 * np.random.default_rng(0).normal(size=p.num_dofs)
        v = dev(np.random.default_rng(1).normal(size=p.num_dofs))
        p.eval_terms()
        torch.cuda.synchronize()
        p.eval_terms()
        p.hvp(p.x_device, v)
        p.hvp(p.x_device, v, psd_floor=FLOOR)
        torch.cuda.synchronize()
        del p
    if "smooth" in args.configs:
        p = edge_length_problem(mesh)
        p.x = pos.ravel()
        v = dev(np.random.default_rng(1).normal(size=p.num_dofs))
        p.eval_terms()
        torch.cuda.synchronize()
        p.eval_terms()
        p.hvp(p.x_device, v)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
