"""Loading golden fixtures and building equivalent oracle / engine problems."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
FLOOR = 1e-9


def cases():
    """Problem fixtures (solver trajectories, solver_*.npz, are separate)."""
    return sorted(p.stem for p in GOLDEN.glob("*.npz") if not p.stem.startswith(("solver_", "vv_", "drivers", "traj_")))


def solver_cases():
    return sorted(p.stem for p in GOLDEN.glob("solver_*.npz"))


def load(name):
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["spec"] = json.loads(str(d["spec"]))
    d["name"] = name
    return d


def states(d):
    return sorted({int(k[1:].split("_")[0]) for k in d if k.startswith("s") and k.endswith("_x")})


def build_terms(d, attr=lambda a: a):
    """Builtin term objects from a fixture spec. `attr` maps each attribute
    array (e.g. to a CUDA tensor)."""
    from paper_2509_00406_b200 import terms as T

    out = []
    for s in d["spec"]:
        a = {k: attr(np.ascontiguousarray(d[v])) for k, v in s["attrs"].items()}
        t = s["type"]
        if t == "Spring":
            term = T.Spring(a["rest_len2"], s["coef"])
        elif t == "Inertia":
            term = T.Inertia(a["masses"], a["target"])
        elif t == "Gravity":
            term = T.Gravity(a["masses"], np.asarray(s["gravity"], dtype=np.float64), s["h2"])
        elif t == "EdgeLength":
            term = T.EdgeLength()
        elif t == "SymDirichlet":
            term = T.SymDirichlet(a["rest_inv"], a["areas"])
        elif t == "SphereBarrierStretch":
            term = T.SphereBarrierStretch(a["base"], a["b1"], a["b2"], s["include_barrier"], s["include_stretch"])
        else:
            raise KeyError(t)
        out.append((s["op"], term))
    return out


def oracle_problem(d, workers=1, accumulation="deterministic"):
    from oracle import OracleProblem

    return OracleProblem(len(d["positions"]), d["faces"], d["edges"], int(d["n"]), build_terms(d),
                         with_hessian=bool(d["with_hessian"]), fixed_vertices=d["fixed"].tolist(),
                         workers=workers, accumulation=accumulation)


def rel(cand, ref):
    """max|cand-ref| / max|ref| over finite entries; NaN masks must agree."""
    cand = np.asarray(cand, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert cand.shape == ref.shape, (cand.shape, ref.shape)
    nan_c, nan_r = ~np.isfinite(cand), ~np.isfinite(ref)
    if not np.array_equal(nan_c, nan_r):
        return float("inf")
    if not (~nan_r).any():
        return 0.0
    scale = float(np.max(np.abs(ref[~nan_r])))
    diff = float(np.max(np.abs(cand[~nan_r] - ref[~nan_r])))
    if scale == 0.0:
        return diff
    return diff / scale


def rel_scalar(a, b):
    a, b = float(a), float(b)
    if np.isnan(a) or np.isnan(b):
        return 0.0 if (np.isnan(a) and np.isnan(b)) else float("inf")
    if a == b:
        return 0.0
    return abs(a - b) / max(abs(b), 1e-300)
