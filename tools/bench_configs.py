"""Time BASELINE configs 3 and 4 (symmetric Dirichlet grad+Hessian, sphere and
smoothing HVP) on one GPU: per call device ms, main-kernel ms, faces/s and the
HBM fraction of the algorithmic bytes. One JSON line per call.

usage: python tools/bench_configs.py [--sub 10] [--steps 10] [--configs dirichlet sphere smooth]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

FLOOR = 1e-9


def report(cfg, call, p, fn, steps, units, unit_name, nbytes, peak, extra=None):
    ms, kms = bench.time_with_kernel(p, fn, steps, 3)
    t = kms if kms else ms
    line = {"config": cfg, "call": call, "ms": ms, "kernel_ms": kms, unit_name + "_per_s": units / (ms * 1e-3),
            "algorithmic_bytes": nbytes, "hbm_frac": nbytes / (t * 1e-3) / 1e9 / peak}
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)


def run_dirichlet(s, steps, peak):
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import distortion_problem, rest_geometry

    t0 = time.perf_counter()
    pos, faces, uv = mg.punctured_icosphere_arrays(s)
    mesh = mg.Mesh(pos, faces)
    rest_inv, areas = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in rest_geometry(mesh))
    p = distortion_problem(mesh, rest_inv, areas, with_hessian=True)
    p.precompute_sparsity()
    p.x = uv.ravel()
    setup = time.perf_counter() - t0
    V, F, nnzb = len(pos), len(faces), p.hess.nnz_blocks
    v = torch.from_numpy(np.random.default_rng(1).normal(size=2 * V)).cuda()
    y = torch.empty_like(v)
    b_hess = 16 * V + 12 * F + 32 * F + 8 * F + 16 * V + 32 * nnzb
    b_hvp = 16 * V + 16 * V + 12 * F + 32 * F + 8 * F + 16 * V
    ex = {"V": V, "F": F, "nnzb": nnzb, "setup_s": setup}
    report("dirichlet", "eval_terms", p, lambda: p.eval_terms(sync=False), steps, F, "faces", b_hess, peak, ex)
    report("dirichlet", "eval_terms_psd", p, lambda: p.eval_terms(psd_floor=FLOOR, sync=False), steps, F, "faces",
           b_hess, peak)
    report("dirichlet", "hvp", p, lambda: p.hvp(p.x_device, v, out=y), steps, F, "faces", b_hvp, peak)
    report("dirichlet", "hvp_psd", p, lambda: p.hvp(p.x_device, v, psd_floor=FLOOR, out=y), steps, F, "faces",
           b_hvp, peak)


def run_sphere(s, steps, peak):
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import initial_sphere, sphere_problem, tangent_bases

    t0 = time.perf_counter()
    pos, faces = mg.icosphere_arrays(s)
    mesh = mg.Mesh(pos, faces)
    base = initial_sphere(mesh)
    b1, b2 = tangent_bases(base)
    base, b1, b2 = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (base, b1, b2))
    p = sphere_problem(mesh, base, b1, b2, with_hessian=False)
    V, F = len(pos), len(faces)
    p.x = 1e-5 * np.random.default_rng(0).normal(size=2 * V)  # tangent noise well below the edge length (no flips)
    setup = time.perf_counter() - t0
    v = torch.from_numpy(np.random.default_rng(1).normal(size=2 * V)).cuda()
    y = torch.empty_like(v)
    b_grad = 16 * V + 72 * V + 12 * F + 16 * V
    b_hvp = 16 * V + 16 * V + 72 * V + 12 * F + 16 * V
    ex = {"V": V, "F": F, "setup_s": setup}
    report("sphere", "eval_terms_grad", p, lambda: p.eval_terms(sync=False), steps, F, "faces", b_grad, peak, ex)
    report("sphere", "hvp", p, lambda: p.hvp(p.x_device, v, out=y), steps, F, "faces", b_hvp, peak)
    report("sphere", "hvp_psd", p, lambda: p.hvp(p.x_device, v, psd_floor=FLOOR, out=y), steps, F, "faces", b_hvp,
           peak)


def run_smooth(s, steps, peak):
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import edge_length_problem

    t0 = time.perf_counter()
    pos, faces = mg.icosphere_arrays(s)
    mesh = mg.Mesh(pos, faces)
    p = edge_length_problem(mesh, with_hessian=False)
    p.x = pos.ravel()
    V, F = len(pos), len(faces)
    E = 3 * F // 2
    setup = time.perf_counter() - t0
    v = torch.from_numpy(np.random.default_rng(1).normal(size=3 * V)).cuda()
    y = torch.empty_like(v)
    ex = {"V": V, "E": E, "setup_s": setup}
    report("smooth", "eval_terms_grad", p, lambda: p.eval_terms(sync=False), steps, E, "edges",
           24 * V + 8 * E + 24 * V, peak, ex)
    report("smooth", "hvp", p, lambda: p.hvp(p.x_device, v, out=y), steps, E, "edges", 24 * V + 8 * E + 24 * V, peak)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sub", type=int, default=10)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--configs", nargs="+", default=["dirichlet", "sphere", "smooth"])
    a = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    peak, _ = bench.peaks()
    for c in a.configs:
        {"dirichlet": run_dirichlet, "sphere": run_sphere, "smooth": run_smooth}[c](a.sub, a.steps, peak)


if __name__ == "__main__":
    main()
