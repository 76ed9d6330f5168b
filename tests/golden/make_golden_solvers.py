"""Golden solver trajectories from the UNMODIFIED reference `meshgrad.solvers`.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_solvers.py

For problems already pinned by tests/golden/<case>.npz (same mesh, terms and
attributes), run the reference's newton_solve / newton_cg_solve from a stored
state and save the SolverReport columns and the final x as
tests/golden/solver_<case>.npz. tests/test_solvers_gpu.py replays them with the
device solvers (paper_2509_00406_b200.solvers).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parent))

import meshgrad as mg  # noqa: E402
from meshgrad.apps.cloth import ClothConfig, ClothSim  # noqa: E402
from meshgrad.apps.param import make_distortion_problem  # noqa: E402
from meshgrad.solvers import SolverConfig, newton_cg_solve, newton_solve  # noqa: E402

from golden_util import load  # noqa: E402


def ref_problem(d):
    """The reference Problem built by the reference apps, with the fixture's
    attributes (same construction as make_golden.py case_cloth / case_dirichlet)."""
    if d["name"] == "cloth8":
        sim = ClothSim(ClothConfig(grid_n=8))
        assert np.array_equal(sim.mesh.positions, d["positions"])
        sim._target[:] = d["a_target"]
        return sim.problem
    mesh = mg.Mesh(d["positions"], d["faces"])
    return make_distortion_problem(mesh, d["a_rest_inv"].reshape(-1, 2, 2), d["a_areas"], with_hessian=True)


def record(name, solver, cfg, x0):
    d = load(name)
    p = ref_problem(d)
    p.x = x0.copy()
    rep = solver(p, cfg)
    out = {
        "case": np.array(name),
        "x0": x0,
        "energies": np.array([r.energy for r in rep.records]),
        "ginf": np.array([r.grad_inf_norm for r in rep.records]),
        "steps": np.array([r.step for r in rep.records]),
        "inner": np.array([r.inner_iters for r in rep.records]),
        "fallback": np.array(rep.fallback_iterations, dtype=np.int64),
        "termination": np.array(rep.termination.value),
        "final_x": p.x.copy(),
        "max_iters": np.array(cfg.max_iters),
        "solver": np.array(solver.__name__),
    }
    np.savez_compressed(OUT / f"solver_{name}_{solver.__name__}.npz", **out)
    print(name, solver.__name__, rep.termination.value, [r.inner_iters for r in rep.records])


if __name__ == "__main__":
    d = load("cloth8")
    record("cloth8", newton_solve, SolverConfig(max_iters=5), d["s0_x"])
    record("cloth8", newton_cg_solve, SolverConfig(max_iters=4), d["s0_x"])
    d = load("dirichlet_ico2")
    record("dirichlet_ico2", newton_cg_solve, SolverConfig(max_iters=4), d["s1_x"])
    record("dirichlet_ico2", newton_solve, SolverConfig(max_iters=4), d["s1_x"])
