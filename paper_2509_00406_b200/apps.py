"""Builders for the four benchmark energies (the reference apps' payload).

Only the *energy definitions and their per-element constants* are here — the
pieces the hot path evaluates. Time stepping, Tutte
initialisation and the solvers are callers of the path and out of scope.

Each builder returns a `Problem` with the same terms, in the same
registration order and with the same constants as the reference:
  cloth_problem          apps/cloth.py:77-117   (V inertia, EV spring, V gravity)
  distortion_problem     apps/param.py:165-180
  sphere_problem         apps/sphere.py:62-99
  edge_length_problem    apps/smooth.py:22-31
The constant helpers restate cloth.py:47-62 (lumped masses), param.py:35-64
(rest geometry) and sphere.py:45-68 (tangent bases, initial sphere).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import Element, Mesh, Op
from .problem import Problem
from .terms import EdgeLength, Gravity, Inertia, SphereBarrierStretch, Spring, SymDirichlet

__all__ = [
    "ClothConfig",
    "cloth_problem",
    "default_pins",
    "distortion_problem",
    "edge_length_problem",
    "initial_sphere",
    "jacobian_dets",
    "lumped_masses",
    "rest_geometry",
    "rest_lengths2",
    "sphere_problem",
    "tangent_bases",
]


@dataclass
class ClothConfig:
    """Same fields/defaults as the reference (apps/cloth.py:25-39)."""

    grid_n: int = 10
    spacing: float = 0.1
    h: float = 0.01
    k: float = 1e4
    mass_density: float = 1.0
    gravity: tuple = (0.0, -9.8, 0.0)
    steps: int = 100
    pinned: tuple | None = None

    def __post_init__(self):
        if self.h <= 0:
            raise ValueError("timestep must be positive")
        if self.k <= 0:
            raise ValueError("stiffness must be positive")


def default_pins(n: int) -> tuple:
    return (n * (n - 1), n * n - 1)


def lumped_masses(mesh: Mesh, density: float) -> np.ndarray:
    """1/3 of incident rest area per vertex times density; unit masses for
    face-free meshes."""
    masses = np.zeros(mesh.num_vertices)
    if mesh.num_faces:
        p, f = mesh.positions, mesh.faces
        cr = np.cross(p[f[:, 1]] - p[f[:, 0]], p[f[:, 2]] - p[f[:, 0]])
        areas = 0.5 * np.linalg.norm(cr, axis=1)
        np.add.at(masses, f.ravel(), np.repeat(areas / 3.0, 3))
        masses *= density
    else:
        masses[:] = density
    return masses


def rest_lengths2(mesh: Mesh) -> np.ndarray:
    e = mesh.edges
    d = mesh.positions[e[:, 1]] - mesh.positions[e[:, 0]]
    l2 = np.einsum("ij,ij->i", d, d)
    if np.any(l2 <= 0):
        raise ValueError("degenerate rest edge with zero length")
    return l2


def cloth_problem(cfg: ClothConfig, mesh: Mesh, target, masses=None, pinned=None,
                  accumulation: str = "deterministic", dtype=None, live_host_attrs: bool = True) -> Problem:
    """Inertia + spring + gravity, registered V, EV, V (cloth.py:115-117).
    `target` (V,3) is the inertial target x_n + h v_n: pass a CUDA tensor to
    update it in place between calls, or a numpy array (re-read each call).
    dtype=torch.float32: fp32 storage (Problem)."""
    h2 = cfg.h * cfg.h
    if masses is None:
        masses = lumped_masses(mesh, cfg.mass_density)
    if pinned is None:
        pinned = cfg.pinned if cfg.pinned is not None else ()
    p = Problem(mesh, 3, with_hessian=True, fixed_vertices=tuple(pinned), accumulation=accumulation, dtype=dtype,
                live_host_attrs=live_host_attrs)
    p.add_term(Element.VERTEX, Op.V, Inertia(masses, target))
    import torch  # rest lengths are derived here, not a caller closure: device-resident, never re-uploaded

    p.add_term(Element.EDGE, Op.EV, Spring(torch.from_numpy(rest_lengths2(mesh)).cuda(), 0.5 * cfg.k * h2))
    p.add_term(Element.VERTEX, Op.V, Gravity(masses, np.asarray(cfg.gravity, dtype=np.float64), h2))
    return p


def rest_geometry(mesh: Mesh):
    """(rest_inv (F,2,2), areas (F,)) of the per-face isometric flattening."""
    p, f = mesh.positions, mesh.faces
    e1 = p[f[:, 1]] - p[f[:, 0]]
    e2 = p[f[:, 2]] - p[f[:, 0]]
    len1 = np.linalg.norm(e1, axis=1)
    normal = np.cross(e1, e2)
    areas = 0.5 * np.linalg.norm(normal, axis=1)
    if np.any(len1 <= 0) or np.any(areas <= 0):
        bad = int(np.argmax((len1 <= 0) | (areas <= 0)))
        raise ValueError(f"degenerate face {bad}: zero edge or zero area")
    u = e1 / len1[:, None]
    w = normal / (2.0 * areas)[:, None]
    v = np.cross(w, u)
    r00 = len1
    r01 = np.einsum("ij,ij->i", e2, u)
    r11 = np.einsum("ij,ij->i", e2, v)
    det = r00 * r11
    rest_inv = np.empty((len(f), 2, 2))
    rest_inv[:, 0, 0] = r11 / det
    rest_inv[:, 0, 1] = -r01 / det
    rest_inv[:, 1, 0] = 0.0
    rest_inv[:, 1, 1] = r00 / det
    return rest_inv, areas


def jacobian_dets(uv: np.ndarray, mesh: Mesh, rest_inv: np.ndarray) -> np.ndarray:
    f = mesh.faces
    d = np.stack([uv[f[:, 1]] - uv[f[:, 0]], uv[f[:, 2]] - uv[f[:, 0]]], axis=2)
    j = np.einsum("fij,fjk->fik", d, rest_inv)
    return j[:, 0, 0] * j[:, 1, 1] - j[:, 0, 1] * j[:, 1, 0]


def distortion_problem(mesh: Mesh, rest_inv, areas, with_hessian: bool = False,
                       accumulation: str = "deterministic") -> Problem:
    p = Problem(mesh, 2, with_hessian=with_hessian, accumulation=accumulation)
    if hasattr(rest_inv, "detach"):  # CUDA tensor: read in place by the kernels
        ri = rest_inv.reshape(-1, 4)
    else:  # numpy: a view, so in-place rewrites of the caller's array are seen (live attributes)
        ri = np.ascontiguousarray(rest_inv).reshape(-1, 4)
    p.add_term(Element.FACE, Op.FV, SymDirichlet(ri, areas))
    return p


def tangent_bases(s: np.ndarray):
    axis = np.zeros_like(s)
    axis[np.arange(len(s)), np.argmin(np.abs(s), axis=1)] = 1.0
    b1 = np.cross(s, axis)
    b1 /= np.linalg.norm(b1, axis=1, keepdims=True)
    b2 = np.cross(s, b1)
    return b1, b2


def initial_sphere(mesh: Mesh) -> np.ndarray:
    s = mesh.positions - mesh.positions.mean(axis=0)
    norms = np.linalg.norm(s, axis=1, keepdims=True)
    if np.any(norms == 0):
        raise ValueError("a vertex coincides with the centroid; cannot project to the sphere")
    return s / norms


def sphere_problem(mesh: Mesh, base, b1, b2, with_hessian: bool = False, accumulation: str = "deterministic",
                   include_barrier: bool = True, include_stretch: bool = True) -> Problem:
    p = Problem(mesh, 2, with_hessian=with_hessian, accumulation=accumulation)
    p.add_term(Element.FACE, Op.FV, SphereBarrierStretch(base, b1, b2, include_barrier, include_stretch))
    return p


def edge_length_problem(mesh: Mesh, with_hessian: bool = False, accumulation: str = "deterministic") -> Problem:
    p = Problem(mesh, 3, with_hessian=with_hessian, accumulation=accumulation)
    p.add_term(Element.EDGE, Op.EV, EdgeLength())
    return p
