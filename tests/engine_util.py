"""Build engine (CUDA) problems from golden fixtures."""

from __future__ import annotations

import numpy as np

from golden_util import build_terms

_KIND = {"V": "VERTEX", "EV": "EDGE", "FV": "FACE"}


def engine_mesh(d):
    import paper_2509_00406_b200 as mg

    if len(d["faces"]):
        return mg.Mesh(d["positions"], d["faces"])
    return mg.Mesh(d["positions"], np.zeros((0, 3)), edges=d["edges"])


def engine_problem(d, accumulation="deterministic", mesh=None, device_attrs=False, dtype=None):
    import torch

    import paper_2509_00406_b200 as mg

    mesh = mesh if mesh is not None else engine_mesh(d)
    p = mg.Problem(mesh, int(d["n"]), with_hessian=bool(d["with_hessian"]),
                   fixed_vertices=d["fixed"].tolist(), accumulation=accumulation, dtype=dtype)
    attr = (lambda a: torch.from_numpy(a).cuda()) if device_attrs else (lambda a: a)
    for op, term in build_terms(d, attr):
        p.add_term(getattr(mg.Element, _KIND[op]), getattr(mg.Op, op), term)
    return p
