"""Cloth HVP (unclamped / clamped) on the 2048^2 grid with the rows forced into
Morton order (what a non-grid mesh gets): the staged row kernel against the
edge tile kernel (MG_EDGE_TILES=0 / 1 in the environment).
usage: MG_EDGE_TILES=1 python tools/time_morton_hvp.py"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import ClothConfig, cloth_problem, default_pins, lumped_masses

    n = 2048
    pos, faces, target, x, v = bench.cloth_inputs(n)
    mesh = mg.Mesh(pos, faces, row_order="morton")
    cfg = ClothConfig(grid_n=n, spacing=1.0 / (n - 1))
    p = cloth_problem(cfg, mesh, torch.from_numpy(target).cuda(),
                      masses=torch.from_numpy(lumped_masses(mesh, cfg.mass_density)).cuda(),
                      pinned=default_pins(n))
    p.x = x
    vd = torch.from_numpy(v).cuda()
    y = torch.empty_like(vd)
    for name, fn in (("hvp", lambda: p.hvp(p.x_device, vd, out=y)),
                     ("hvp_psd", lambda: p.hvp(p.x_device, vd, psd_floor=1e-9, out=y)),
                     ("grad", lambda: p.eval_terms(sync=False))):
        ms, kms = bench.time_with_kernel(p, fn, 30, 5)
        print(json.dumps({"tiles": os.environ.get("MG_EDGE_TILES", "1"), "call": name, "ms": ms, "kernel_ms": kms,
                          "row_order": mesh.row_order_used()[0]}))


if __name__ == "__main__":
    main()
