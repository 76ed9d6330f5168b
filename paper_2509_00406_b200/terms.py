"""Builtin per-element energy terms (the device term registry).

Each class is both
  * a descriptor the engine compiles against (`type_id`, `op`, scalar
    `params`, per-element attribute arrays) — evaluated on the GPU by
    `csrc/terms.cuh`; and
  * a callable with the reference callback signature `fn(handle, nbrs, x)`
    (problem.py:8-14, 440-452) whose body is the reference app's formula in
    the reference's operation order, over the scalar-generic containers of
    `active.py`. The CPU oracle (tests only) runs exactly this callable.

Attribute arrays may be numpy arrays (re-uploaded on every call by default,
`Problem(live_host_attrs=True)`, like the reference re-reading closure arrays
that `ClothSim.step` / the sphere `post_step` rewrite in place) or CUDA torch
tensors (read in place by the kernels, zero copies).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .active import SmallMatrix, log, positive_guard
from .mesh import Element, Op

__all__ = [
    "BuiltinTerm",
    "EdgeLength",
    "Gravity",
    "Inertia",
    "SphereBarrierStretch",
    "Spring",
    "SymDirichlet",
]


def _rows(arr, idx):
    if hasattr(arr, "detach"):  # torch tensor -> host view for callable use
        arr = arr.detach().cpu().numpy()
    return np.asarray(arr)[idx]


class BuiltinTerm:
    type_id: int = 0
    op: Op = Op.V
    kind: Element = Element.VERTEX
    var_dims: tuple = (2, 3)
    attr_names: tuple = ()
    attr_domains: tuple = ()  # per attribute: "V" (per vertex), "E" (per edge) or "F" (per face) rows

    def params(self, n: int) -> list[float]:
        return []

    def attrs(self) -> list:
        return [getattr(self, name) for name in self.attr_names]

    def check_dims(self, n: int) -> None:
        if n not in self.var_dims:
            raise ValueError(f"{type(self).__name__} needs var_dim in {self.var_dims}, got {n}")

    def shard(self, vertex_ids, edge_ids, face_ids) -> "BuiltinTerm":
        """The same term on a submesh: every attribute gathered to the
        submesh's local vertices / edges / faces (global ids given)."""
        import copy

        out = copy.copy(self)
        ids = {"V": vertex_ids, "E": edge_ids, "F": face_ids}
        for name, dom in zip(self.attr_names, self.attr_domains):
            arr = getattr(self, name)
            idx = ids[dom]
            if hasattr(arr, "detach"):
                import torch

                sub = arr[torch.as_tensor(idx, device=arr.device)].contiguous()
            else:
                sub = np.ascontiguousarray(np.asarray(arr)[idx])
            setattr(out, name, sub)
        return out


class Inertia(BuiltinTerm):
    """0.5 * m_v * |x_v - t_v|^2 per vertex (ref apps/cloth.py:102-104)."""

    type_id = _lib.MG_TERM_INERTIA
    op = Op.V
    kind = Element.VERTEX
    attr_names = ("masses", "target")
    attr_domains = ("V", "V")

    def __init__(self, masses, target):
        self.masses = masses
        self.target = target

    def __call__(self, vertex, nbrs, x):
        d = x[vertex] - _rows(self.target, vertex.index)
        return 0.5 * _rows(self.masses, vertex.index) * d.norm2()


class Spring(BuiltinTerm):
    """coef * l2 * (|x_i - x_j|^2 / l2 - 1)^2 per edge; the cloth uses
    coef = 0.5*k*h^2 (ref apps/cloth.py:106-110), the reference tests 0.5*k
    (test_problem.py:21-24)."""

    type_id = _lib.MG_TERM_SPRING
    op = Op.EV
    kind = Element.EDGE
    attr_names = ("rest_len2",)
    attr_domains = ("E",)

    def __init__(self, rest_len2, coef: float):
        self.rest_len2 = rest_len2
        self.coef = float(coef)

    def params(self, n):
        return [self.coef]

    def __call__(self, edge, verts, x):
        d = x[verts[0]] - x[verts[1]]
        l2 = _rows(self.rest_len2, edge.index)
        s = d.norm2() / l2 - 1.0
        return self.coef * l2 * (s * s)


class Gravity(BuiltinTerm):
    """(-h2) * (m_v * x_v . g) per vertex (ref apps/cloth.py:112-113)."""

    type_id = _lib.MG_TERM_GRAVITY
    op = Op.V
    kind = Element.VERTEX
    attr_names = ("masses",)
    attr_domains = ("V",)

    def __init__(self, masses, gravity, h2: float):
        self.masses = masses
        self.gvec = np.asarray(gravity, dtype=np.float64)
        self.h2 = float(h2)

    def params(self, n):
        if len(self.gvec) != n:
            raise ValueError(f"gravity vector has {len(self.gvec)} components, var_dim is {n}")
        return [self.h2] + [float(g) for g in self.gvec]

    def __call__(self, vertex, nbrs, x):
        return (-self.h2) * (_rows(self.masses, vertex.index) * x[vertex].dot(self.gvec))


class EdgeLength(BuiltinTerm):
    """|x_i - x_j|^2 per edge (ref apps/smooth.py:22-31)."""

    type_id = _lib.MG_TERM_EDGE_LENGTH
    op = Op.EV
    kind = Element.EDGE

    def __call__(self, edge, verts, x):
        return (x[verts[0]] - x[verts[1]]).norm2()


class SymDirichlet(BuiltinTerm):
    """area * (|J|_F^2 + |J|_F^2 / det(J)^2), J = [b-a, c-a] @ rest_inv,
    det positive-guarded (ref apps/param.py:170-177). n = 2."""

    type_id = _lib.MG_TERM_SYM_DIRICHLET
    op = Op.FV
    kind = Element.FACE
    var_dims = (2,)
    attr_names = ("rest_inv", "areas")
    attr_domains = ("F", "F")

    def __init__(self, rest_inv, areas):
        self.rest_inv = rest_inv
        self.areas = areas

    def __call__(self, face, verts, x):
        a, b, c = x[verts[0]], x[verts[1]], x[verts[2]]
        d1 = b - a
        d2 = c - a
        rest_inv = _rows(self.rest_inv, face.index).reshape(-1, 2, 2)
        jac = SmallMatrix([[d1[0], d2[0]], [d1[1], d2[1]]]) @ rest_inv
        det = positive_guard(jac.det())
        fro = jac.frobenius2()
        return _rows(self.areas, face.index) * (fro + fro / (det * det))


class SphereBarrierStretch(BuiltinTerm):
    """-log det[p_i, p_j, p_k] + sum |p_a - p_b|^2 with the per-vertex
    retraction p = normalize(x0*b1 + x1*b2 + s) (ref apps/sphere.py:71-99). n = 2."""

    type_id = _lib.MG_TERM_SPHERE
    op = Op.FV
    kind = Element.FACE
    var_dims = (2,)
    attr_names = ("base", "b1", "b2")
    attr_domains = ("V", "V", "V")

    def __init__(self, base, b1, b2, include_barrier: bool = True, include_stretch: bool = True):
        self.base = base
        self.b1 = b1
        self.b2 = b2
        self.include_barrier = bool(include_barrier)
        self.include_stretch = bool(include_stretch)

    def params(self, n):
        return [1.0 if self.include_barrier else 0.0, 1.0 if self.include_stretch else 0.0]

    def __call__(self, face, verts, x):
        from .active import ActiveVec

        ps = []
        for q in range(3):
            vid = verts[q].index
            s, b1, b2 = _rows(self.base, vid), _rows(self.b1, vid), _rows(self.b2, vid)
            x2 = x[verts[q]]
            r = ActiveVec([x2[0] * b1[:, c] + x2[1] * b2[:, c] + s[:, c] for c in range(3)])
            ps.append(r / r.norm())
        total = 0.0
        if self.include_barrier:
            det = SmallMatrix.from_columns(ps[0], ps[1], ps[2]).det()
            total = -log(det) + total
        if self.include_stretch:
            total = total + (ps[0] - ps[1]).norm2() + (ps[1] - ps[2]).norm2() + (ps[2] - ps[0]).norm2()
        return total
