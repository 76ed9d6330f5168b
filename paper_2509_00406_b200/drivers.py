"""Device drivers around the hot path: the reference apps'
outer loops with their state kept on the GPU.

  ClothSim                apps/cloth.py:65-156   implicit-Euler steps: the inertial
                          target x_n + h v_n is a CUDA tensor the inertia term
                          reads in place; each step is a device Newton solve
  tutte_embedding         apps/param.py:113-162  boundary on the unit circle,
                          interior by Jacobi-preconditioned CG on the graph
                          Laplacian (cuSPARSE CSR matvec through torch)
  parameterize            apps/param.py:183-209  flip check + matrix-free Newton
  spherical_parameterize  apps/sphere.py:100-134 device L-BFGS with the
                          retraction / tangent-basis rebuild as post_step
  smooth                  apps/smooth.py:62-94   explicit descent, "ad" (engine
                          gradient) or "manual" (closed-form gather)

Same signatures, defaults, error texts and return values as the reference;
positions come back as numpy arrays like the reference's.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass

import numpy as np

from .apps import (ClothConfig, cloth_problem, default_pins, distortion_problem, edge_length_problem,
                   initial_sphere, jacobian_dets, lumped_masses, rest_geometry, rest_lengths2, sphere_problem,
                   tangent_bases)
from .mesh import Mesh, generate_grid
from .solvers import (SolverConfig, SolverReport, Termination, cg_linear_solve, gradient_descent_solve,
                      lbfgs_solve, newton_cg_solve, newton_solve)

__all__ = [
    "ClothSim",
    "ParamConfig",
    "SphereConfig",
    "bench_gradient",
    "boundary_loop",
    "check_genus_zero",
    "face_determinants",
    "manual_energy",
    "manual_gradient",
    "parameterize",
    "planar_project",
    "retract_rows",
    "smooth",
    "spherical_parameterize",
    "tutte_embedding",
]


def _torch():
    import torch

    return torch


# ------------------------------------------------------------------ cloth

class ClothSim:
    """Owns the problem, rest lengths, masses and the device target buffer
    (ref apps/cloth.py:65-156). The same Problem is reused across steps."""

    def __init__(self, cfg: ClothConfig, mesh: Mesh | None = None, solver_cfg: SolverConfig | None = None,
                 masses: np.ndarray | None = None, workers: int = 1, accumulation: str = "deterministic"):
        torch = _torch()
        self.cfg = cfg
        self.mesh = mesh if mesh is not None else generate_grid(cfg.grid_n, cfg.spacing)
        self.solver_cfg = solver_cfg or SolverConfig(grad_tol=1e-8)
        pinned = cfg.pinned if cfg.pinned is not None else (default_pins(cfg.grid_n) if mesh is None else ())
        self.pinned = tuple(pinned)
        self.masses = masses if masses is not None else lumped_masses(self.mesh, cfg.mass_density)
        self.rest_len2 = rest_lengths2(self.mesh)
        self._target = torch.from_numpy(np.ascontiguousarray(self.mesh.positions, dtype=np.float64)).cuda()
        self._pin_idx = torch.tensor(list(self.pinned), dtype=torch.int64, device="cuda")
        self.problem = cloth_problem(cfg, self.mesh, self._target, masses=torch.from_numpy(
                                         np.ascontiguousarray(self.masses, dtype=np.float64)).cuda(),
                                     pinned=self.pinned,
                                     accumulation=accumulation)
        self.problem.precompute_sparsity()

    def step(self, x, v):
        """One implicit-Euler step from (x, v) -> (x_next, v_next, report)."""
        torch = _torch()
        cfg = self.cfg
        xd = torch.as_tensor(np.asarray(x, dtype=np.float64)).reshape(-1, 3).cuda()
        vd = torch.as_tensor(np.asarray(v, dtype=np.float64)).reshape(-1, 3).cuda()
        self._target.copy_(xd).add_(vd, alpha=cfg.h)
        if self.pinned:
            self._target[self._pin_idx] = xd[self._pin_idx]
        self.problem.x_device.copy_(xd.reshape(-1))
        report = newton_solve(self.problem, self.solver_cfg)
        if (report.termination is Termination.LINE_SEARCH_FAILED and report.accepted_steps == 0
                and report.records[0].grad_inf_norm > self.solver_cfg.grad_tol):
            raise RuntimeError(f"cloth step aborted: line search failed at energy {report.final_energy:.6g}")
        x_next = self.problem.x_device.reshape(-1, 3).clone()
        v_next = (x_next - xd) / cfg.h
        return x_next.cpu().numpy(), v_next.cpu().numpy(), report

    def simulate(self, steps: int | None = None, x0=None, v0=None, callback=None):
        """`steps` implicit-Euler steps; returns (x, v, reports)."""
        steps = steps if steps is not None else self.cfg.steps
        x = self.mesh.positions.copy() if x0 is None else np.array(x0, dtype=np.float64)
        v = np.zeros_like(x) if v0 is None else np.array(v0, dtype=np.float64)
        reports: list[SolverReport] = []
        for s in range(steps):
            x, v, rep = self.step(x, v)
            reports.append(rep)
            if callback is not None:
                callback(s, x, v, rep)
        return x, v, reports


# ------------------------------------------------------------------ parameterization

@dataclass
class ParamConfig:
    """Same fields/defaults as the reference (apps/param.py:27-33)."""

    init: str = "tutte"
    outer_iters: int = 30
    cg_tol: float = 1e-4
    cg_max_iters: int = 100
    grad_tol: float = 1e-6


def planar_project(mesh: Mesh) -> np.ndarray:
    return mesh.positions[:, :2].copy()


def _edge_face_counts(mesh: Mesh) -> np.ndarray:
    e = mesh.edges
    nv = mesh.num_vertices
    key = np.minimum(e[:, 0], e[:, 1]).astype(np.int64) * nv + np.maximum(e[:, 0], e[:, 1])
    f = mesh.faces.astype(np.int64)
    fe = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    fk = np.minimum(fe[:, 0], fe[:, 1]) * nv + np.maximum(fe[:, 0], fe[:, 1])
    order = np.argsort(key)
    pos = np.searchsorted(key[order], fk)
    counts = np.zeros(len(key), dtype=np.int64)
    np.add.at(counts, order[pos], 1)
    return counts


def boundary_loop(mesh: Mesh) -> list[int]:
    """Ordered vertex loop of the single boundary (ref apps/param.py:86-110)."""
    bmask = _edge_face_counts(mesh) == 1
    if not bmask.any():
        raise ValueError("mesh has no boundary; expected a topological disk")
    nbr: dict[int, list[int]] = {}
    for i, j in mesh.edges[bmask]:
        nbr.setdefault(int(i), []).append(int(j))
        nbr.setdefault(int(j), []).append(int(i))
    for v, ns in nbr.items():
        if len(ns) != 2:
            raise ValueError(f"boundary vertex {v} has {len(ns)} boundary edges; not a disk")
    start = min(nbr)
    loop = [start]
    prev, cur = start, min(nbr[start])
    while cur != start:
        loop.append(cur)
        a, b = nbr[cur]
        prev, cur = cur, (b if a == prev else a)
    if len(loop) != len(nbr):
        raise ValueError("mesh has more than one boundary loop; not a disk")
    return loop


def tutte_embedding(mesh: Mesh, tol: float = 1e-12, max_iters: int = 20000) -> np.ndarray:
    """Flip-free disk initialization (ref apps/param.py:113-162): boundary on
    the unit circle, interior at the average of its neighbours, solved on the
    device (Jacobi-preconditioned CG on the reduced graph Laplacian)."""
    torch = _torch()
    if mesh.num_vertices - mesh.num_edges + mesh.num_faces != 1:
        raise ValueError("mesh is not a topological disk (Euler characteristic != 1)")
    loop = boundary_loop(mesh)
    nv = mesh.num_vertices
    uv = np.zeros((nv, 2))
    theta = 2.0 * np.pi * np.arange(len(loop)) / len(loop)
    uv[loop, 0] = np.cos(theta)
    uv[loop, 1] = np.sin(theta)
    on_boundary = np.zeros(nv, dtype=bool)
    on_boundary[loop] = True
    interior = np.flatnonzero(~on_boundary)
    if len(interior) == 0:
        return uv
    pos_of = -np.ones(nv, dtype=np.int64)
    pos_of[interior] = np.arange(len(interior))
    e = mesh.edges.astype(np.int64)
    a = np.concatenate([e[:, 0], e[:, 1]])
    b = np.concatenate([e[:, 1], e[:, 0]])
    deg = np.bincount(a, minlength=nv)[interior].astype(np.float64)
    rows = pos_of[a]
    keep = rows >= 0
    a_r, b_v = rows[keep], b[keep]
    inner = pos_of[b_v] >= 0
    rhs = np.zeros((len(interior), 2))
    np.add.at(rhs, a_r[~inner], uv[b_v[~inner]])
    ni = len(interior)
    # interior Laplacian L = D - A as a device CSR operator
    r_all = np.concatenate([np.arange(ni), a_r[inner]])
    c_all = np.concatenate([np.arange(ni), pos_of[b_v[inner]]])
    v_all = np.concatenate([deg, -np.ones(int(inner.sum()))])
    order = np.lexsort((c_all, r_all))
    crow = np.zeros(ni + 1, dtype=np.int64)
    np.cumsum(np.bincount(r_all, minlength=ni), out=crow[1:])
    with warnings.catch_warnings():  # torch flags sparse CSR as beta
        warnings.simplefilter("ignore", UserWarning)
        L = torch.sparse_csr_tensor(torch.from_numpy(crow), torch.from_numpy(c_all[order]),
                                    torch.from_numpy(v_all[order]), size=(ni, ni), dtype=torch.float64).cuda()
    inv_deg = torch.from_numpy(1.0 / deg).cuda()
    apply = lambda y: (L @ y.unsqueeze(1)).squeeze(1)
    for c in range(2):
        sol, info = cg_linear_solve(apply, torch.from_numpy(rhs[:, c].copy()).cuda(), tol, max_iters,
                                    precond=lambda r: inv_deg * r)
        if not info.converged:
            raise RuntimeError("interior solve for the disk embedding did not converge")
        uv[interior, c] = sol.cpu().numpy()
    return uv


def parameterize(mesh: Mesh, cfg: ParamConfig | None = None, workers: int = 1,
                 accumulation: str = "deterministic"):
    """Flatten a disk mesh; returns (uv, report) (ref apps/param.py:183-209)."""
    cfg = cfg or ParamConfig()
    rest_inv, areas = rest_geometry(mesh)
    if cfg.init == "tutte":
        uv0 = tutte_embedding(mesh)
    elif cfg.init == "planar":
        uv0 = planar_project(mesh)
    else:
        raise ValueError(f"unknown initialization {cfg.init!r}")
    dets = jacobian_dets(uv0, mesh, rest_inv)
    if np.any(dets <= 0):
        flipped = np.flatnonzero(dets <= 0)
        raise ValueError(f"initialization contains flipped faces: {flipped[:10].tolist()}")
    problem = distortion_problem(mesh, rest_inv, areas, with_hessian=False, accumulation=accumulation)
    problem.x = uv0.ravel().copy()
    solver_cfg = SolverConfig(max_iters=cfg.outer_iters, grad_tol=cfg.grad_tol, cg_tol=cfg.cg_tol,
                              cg_max_iters=cfg.cg_max_iters)
    report = newton_cg_solve(problem, solver_cfg)
    return problem.x.reshape(-1, 2).copy(), report


# ------------------------------------------------------------------ sphere

@dataclass
class SphereConfig:
    """Same fields/defaults as the reference (apps/sphere.py:24-28)."""

    iters: int = 200
    lbfgs_memory: int = 8
    grad_tol: float = 1e-10


def check_genus_zero(mesh: Mesh) -> None:
    chi = mesh.num_vertices - mesh.num_edges + mesh.num_faces
    if chi != 2:
        raise ValueError(f"mesh is not closed genus 0 (Euler characteristic {chi}, expected 2)")


def face_determinants(points: np.ndarray, faces: np.ndarray) -> np.ndarray:
    a, b, c = points[faces[:, 0]], points[faces[:, 1]], points[faces[:, 2]]
    return np.einsum("ij,ij->i", a, np.cross(b, c))


def retract_rows(s, b1, b2, x2):
    """normalize(s + x1 b1 + x2 b2) row-wise (numpy or torch)."""
    r = s + x2[:, :1] * b1 + x2[:, 1:2] * b2
    if isinstance(r, np.ndarray):
        return r / np.linalg.norm(r, axis=1, keepdims=True)
    return r / r.norm(dim=1, keepdim=True)


def _tangent_bases_device(s):
    torch = _torch()
    axis = torch.zeros_like(s)
    axis.scatter_(1, s.abs().argmin(dim=1, keepdim=True), 1.0)
    b1 = torch.linalg.cross(s, axis, dim=1)
    b1 = b1 / b1.norm(dim=1, keepdim=True)
    return b1, torch.linalg.cross(s, b1, dim=1)


def spherical_parameterize(mesh: Mesh, cfg: SphereConfig | None = None, workers: int = 1,
                           accumulation: str = "deterministic", on_accept=None):
    """Optimize the spherical embedding; returns (points, report) (ref
    apps/sphere.py:100-134). Base points and tangent bases are CUDA tensors
    the sphere term reads in place; the post-step retraction and basis rebuild
    run on the device."""
    torch = _torch()
    cfg = cfg or SphereConfig()
    check_genus_zero(mesh)
    base_h = initial_sphere(mesh)
    dets = face_determinants(base_h, mesh.faces)
    if np.any(dets <= 0):
        flipped = np.flatnonzero(dets <= 0)
        raise ValueError(f"initial sphere projection has flipped faces: {flipped[:10].tolist()}")
    b1_h, b2_h = tangent_bases(base_h)
    base, b1, b2 = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (base_h, b1_h, b2_h))
    problem = sphere_problem(mesh, base, b1, b2, accumulation=accumulation)
    problem.x = np.zeros(2 * mesh.num_vertices)

    def post_step(pb) -> None:
        x2 = pb.x_device.reshape(-1, 2)
        base.copy_(retract_rows(base, b1, b2, x2))
        nb1, nb2 = _tangent_bases_device(base)
        b1.copy_(nb1)
        b2.copy_(nb2)
        pb.x_device.zero_()
        if on_accept is not None:
            on_accept(base.cpu().numpy())

    solver_cfg = SolverConfig(max_iters=cfg.iters, grad_tol=cfg.grad_tol, lbfgs_memory=cfg.lbfgs_memory)
    report = lbfgs_solve(problem, solver_cfg, post_step=post_step)
    return base.cpu().numpy(), report


# ------------------------------------------------------------------ smoothing

def manual_energy(x, mesh: Mesh) -> float:
    d = x[mesh.edges[:, 0]] - x[mesh.edges[:, 1]]
    return float((d * d).sum())


def manual_gradient(x, mesh: Mesh):
    """2 sum_{j in N(i)} (x_i - x_j) by a gather (numpy or torch input)."""
    if isinstance(x, np.ndarray):
        nbr_sum = np.zeros_like(x)
        e = mesh.edges
        np.add.at(nbr_sum, e[:, 0], x[e[:, 1]])
        np.add.at(nbr_sum, e[:, 1], x[e[:, 0]])
        deg = np.bincount(e.ravel(), minlength=mesh.num_vertices).astype(np.float64)
        return 2.0 * (deg[:, None] * x - nbr_sum)
    torch = _torch()
    e = torch.from_numpy(mesh.edges.astype(np.int64)).to(x.device)
    nbr_sum = torch.zeros_like(x)
    nbr_sum.index_add_(0, e[:, 0], x[e[:, 1]])
    nbr_sum.index_add_(0, e[:, 1], x[e[:, 0]])
    deg = torch.bincount(e.reshape(-1), minlength=mesh.num_vertices).to(x.dtype)
    return 2.0 * (deg[:, None] * x - nbr_sum)


def smooth(mesh: Mesh, lam: float, iters: int, mode: str = "ad", x0=None, workers: int = 1,
           accumulation: str = "deterministic"):
    """`iters` explicit updates x <- x - lam grad; returns (positions, report)
    (ref apps/smooth.py:62-94)."""
    torch = _torch()
    if lam < 0:
        raise ValueError("step must be non-negative")
    x0 = mesh.positions.copy() if x0 is None else np.array(x0, dtype=np.float64)
    if mode == "ad":
        problem = edge_length_problem(mesh, accumulation=accumulation)
        problem.x = x0.ravel().copy()
        report = gradient_descent_solve(problem, lam, iters)
        return problem.x.reshape(-1, 3).copy(), report
    if mode != "manual":
        raise ValueError(f"unknown mode {mode!r}")
    x = torch.from_numpy(x0).cuda()
    report = SolverReport()
    g = manual_gradient(x, mesh)
    report.log(0, manual_energy(x, mesh), float(g.abs().max()), 0.0, 0, 0.0)
    for it in range(1, iters + 1):
        t0 = time.perf_counter()
        x = x - lam * g
        g = manual_gradient(x, mesh)
        report.log(it, manual_energy(x, mesh), float(g.abs().max()), lam, 0, (time.perf_counter() - t0) * 1e3)
    report.termination = Termination.MAX_ITERS
    return x.cpu().numpy(), report


def bench_gradient(sizes=(64, 128, 256, 512), repeats: int = 3, workers: int = 1,
                   accumulation: str = "deterministic"):
    """Median per-call time of the smoothing gradient on n x n grids (ref
    apps/smooth.py:97-119): rows of (side, vertices, edges, ms_per_iter, ratio
    to the previous size); mesh construction and layout outside the timing."""
    rows = []
    prev = None
    for n in sizes:
        mesh = generate_grid(n, 1.0 / (n - 1))
        problem = edge_length_problem(mesh, accumulation=accumulation)
        problem.x = mesh.positions.ravel().copy()
        problem.eval_terms()  # layout and pattern outside the timed region
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            problem.eval_terms()
            times.append((time.perf_counter() - t0) * 1e3)
        ms = float(np.median(times))
        rows.append({"side": n, "vertices": mesh.num_vertices, "edges": mesh.num_edges, "ms_per_iter": ms,
                     "ratio": (ms / prev) if prev else float("nan")})
        prev = ms
    return rows
