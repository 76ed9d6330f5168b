"""Golden trajectories of the reference apps' drivers (cloth stepping, Tutte +
parameterization, spherical L-BFGS, smoothing), from the UNMODIFIED reference
`meshgrad` (run in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_drivers.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parent.parent))

import meshgrad as mg  # noqa: E402
from meshgrad.apps.cloth import ClothConfig, ClothSim  # noqa: E402
from meshgrad.apps.param import ParamConfig, parameterize, tutte_embedding  # noqa: E402
from meshgrad.apps.smooth import smooth  # noqa: E402
from meshgrad.apps.sphere import SphereConfig, spherical_parameterize  # noqa: E402

from paper_2509_00406_b200.mesh import icosphere_arrays, punctured_icosphere_arrays  # noqa: E402


def main():
    out = {}
    # cloth: 3 implicit-Euler steps of the default 8x8 sheet
    sim = ClothSim(ClothConfig(grid_n=8))
    x, v, reps = sim.simulate(3)
    out["cloth_x"], out["cloth_v"] = x, v
    out["cloth_energies"] = np.array([r.final_energy for r in reps])
    # Tutte + parameterization of a punctured icosphere(2) (a disk)
    pos, faces, _ = punctured_icosphere_arrays(2)
    m = mg.Mesh(pos, faces)
    out["param_pos"], out["param_faces"] = pos, faces
    out["tutte_uv"] = tutte_embedding(m)
    uv, rep = parameterize(m, ParamConfig(outer_iters=8))
    out["param_uv"] = uv
    out["param_energies"] = np.array(rep.energies)
    # sphere: 15 L-BFGS iterations on icosphere(2)
    spos, sfaces = icosphere_arrays(2)
    sm = mg.Mesh(spos, sfaces)
    out["sphere_pos"], out["sphere_faces"] = spos, sfaces
    pts, rep = spherical_parameterize(sm, SphereConfig(iters=15))
    out["sphere_points"] = pts
    out["sphere_energies"] = np.array(rep.energies)
    # smoothing: both kernels on a noisy 6x6 grid
    g = mg.generate_grid(6, 0.2)
    x0 = g.positions + 0.05 * np.random.default_rng(4).normal(size=g.positions.shape)
    out["smooth_x0"] = x0
    for mode in ("ad", "manual"):
        xs, rep = smooth(g, 0.05, 10, mode=mode, x0=x0)
        out[f"smooth_{mode}_x"] = xs
        out[f"smooth_{mode}_energies"] = np.array(rep.energies)
    np.savez_compressed(OUT / "drivers.npz", **out)
    print({k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
