"""Golden vectors for a VV (vertex one-ring) callback term, from the
UNMODIFIED reference `meshgrad` (run in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_vv.py

The callback (ring_energy below, repeated verbatim in tests/test_vv_gpu.py) is
a nonlinear, non-convex neighbourhood energy: the Hessian couples distance-2
vertices through the center (ref problem.py:340-353) and the PSD clamp has
work to do. Pinned vertices exercise the masked lift.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import meshgrad as mg  # noqa: E402
from meshgrad.active import sqrt  # noqa: E402
from meshgrad.mesh import Element, Op  # noqa: E402

FLOOR = 1e-9


def make_ring_energy(w):
    def ring_energy(vertex, nbrs, x):
        c = x[vertex]
        total = 0.0
        for nb in nbrs:
            d = c - x[nb]
            r = sqrt(d.norm2() + 0.01)
            total = total + (r - 0.3) * (r - 0.3) * w[vertex.index]
        return total

    return ring_energy


def main():
    mesh = mg.generate_grid(5, 0.25)
    n = 3
    rng = np.random.default_rng(11)
    w = 1.0 + rng.random(mesh.num_vertices)
    fixed = [0, 7]
    p = mg.Problem(mesh, n, fixed_vertices=fixed)
    p.add_term(Element.VERTEX, Op.VV, make_ring_energy(w))
    out = {"positions": mesh.positions, "faces": mesh.faces, "n": np.array(n), "w": w,
           "fixed": np.array(fixed, dtype=np.int64)}
    for s in range(2):
        x = mesh.positions.ravel() + 0.08 * rng.normal(size=n * mesh.num_vertices)
        v = rng.normal(size=n * mesh.num_vertices)
        p.x = x.copy()
        out[f"s{s}_x"] = x
        out[f"s{s}_energy"] = np.array(p.eval_terms())
        out[f"s{s}_grad"] = p.grad.copy()
        out[f"s{s}_hess"] = p.hess.values.copy()
        out[f"s{s}_psd_energy"] = np.array(p.eval_terms(psd_floor=FLOOR))
        out[f"s{s}_psd_hess"] = p.hess.values.copy()
        out[f"s{s}_energy_only"] = np.array(p.eval_energy_only(x))
        out[f"s{s}_v"] = v
        out[f"s{s}_hvp"] = p.hvp(x, v)
        out[f"s{s}_hvp_psd"] = p.hvp(x, v, psd_floor=FLOOR)
    out["row_offsets"] = p.hess.row_offsets.copy()
    out["col_indices"] = p.hess.col_indices.copy()
    np.savez_compressed(OUT / "vv_grid5.npz", **out)
    print("vv_grid5", {k: np.shape(v) for k, v in out.items() if k in ("row_offsets", "col_indices")})


if __name__ == "__main__":
    main()
