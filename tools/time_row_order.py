"""Icosphere configs (smoothing HVP / gradient, sphere HVP, Dirichlet HVP) with
the rows in Morton order (the default for non-grid meshes) against the
caller's numbering (row_order="identity").
usage: python tools/time_row_order.py [--sub 10]"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import (distortion_problem, edge_length_problem, initial_sphere, rest_geometry,
                                            sphere_problem, tangent_bases)

    ap = argparse.ArgumentParser()
    ap.add_argument("--sub", type=int, default=10)
    args = ap.parse_args()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    pos, faces = mg.icosphere_arrays(args.sub)
    for order in ("morton", "identity"):
        mesh = mg.Mesh(pos, faces, row_order=order)
        p = edge_length_problem(mesh)
        p.x = pos.ravel()
        vd = dev(np.random.default_rng(1).normal(size=p.num_dofs))
        y = torch.empty_like(vd)
        for name, fn in (("smooth_hvp", lambda: p.hvp(p.x_device, vd, out=y)), ("smooth_grad", lambda: p.eval_terms(sync=False))):
            ms, kms = bench.time_with_kernel(p, fn, 20, 5)
            print(json.dumps({"order": mesh.row_order_used()[0], "call": name, "ms": ms, "kernel_ms": kms}), flush=True)
        del p
        base = initial_sphere(mesh)
        b1, b2 = tangent_bases(base)
        p = sphere_problem(mesh, dev(base), dev(b1), dev(b2))
        p.x = 1e-5 * np.random.default_rng(0).normal(size=p.num_dofs)
        vd = dev(np.random.default_rng(1).normal(size=p.num_dofs))
        y = torch.empty_like(vd)
        ms, kms = bench.time_with_kernel(p, lambda: p.hvp(p.x_device, vd, out=y), 20, 5)
        print(json.dumps({"order": mesh.row_order_used()[0], "call": "sphere_hvp", "ms": ms, "kernel_ms": kms}), flush=True)
        del p
        bench.gc_cuda()


if __name__ == "__main__":
    main()
