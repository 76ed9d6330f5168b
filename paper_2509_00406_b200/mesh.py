"""Mesh topology for the device engine.

Mirrors the parts of the reference `meshgrad.mesh` the hot path needs
(mesh.py:17-34, 130-249): the element/op vocabulary, input validation with the
reference's error messages, canonical sorted edges, and the deterministic
synthetic generators that define the benchmark meshes.

Edge derivation and patching run on the device (csrc/setup.cu, exposed via
`mg_mesh_create`); the host keeps positions/faces as given. The generators are
exact vectorised restatements of `generate_grid` / `generate_icosphere`
(mesh.py:308-373) so the same arrays feed the device and the
oracle.
"""

from __future__ import annotations

import ctypes
from enum import Enum

import numpy as np

from . import _lib

__all__ = [
    "DEFAULT_PATCH_TARGET",
    "DEFAULT_VALENCE_CAP",
    "Element",
    "Mesh",
    "MeshError",
    "Op",
    "SOURCE_KIND",
    "generate_grid",
    "generate_icosphere",
    "grid_arrays",
    "icosphere_arrays",
    "load_obj",
    "punctured_icosphere_arrays",
    "save_obj",
]

DEFAULT_VALENCE_CAP = 32
DEFAULT_PATCH_TARGET = 512
DEFAULT_PATCH_VERTICES = 128


class MeshError(Exception):
    """Malformed mesh input (ref mesh.py:40-41)."""


class Element(Enum):
    VERTEX = "vertex"
    EDGE = "edge"
    FACE = "face"


class Op(Enum):
    """Neighbourhood access patterns (ref mesh.py:50-66)."""

    FV = "FV"
    EV = "EV"
    VV = "VV"
    VE = "VE"
    VF = "VF"
    V = "V"


SOURCE_KIND = {
    Op.FV: Element.FACE,
    Op.EV: Element.EDGE,
    Op.VV: Element.VERTEX,
    Op.VE: Element.VERTEX,
    Op.VF: Element.VERTEX,
    Op.V: Element.VERTEX,
}


def _host_edges(faces: np.ndarray, explicit, nv: int) -> np.ndarray:
    """Canonical lexicographically sorted edges on the host (no-GPU contexts
    only: multi-process host logic and CPU tests; ref mesh.py:184-202)."""
    if len(faces):
        a = faces[:, [0, 1, 2]].ravel()
        b = faces[:, [1, 2, 0]].ravel()
        key = np.unique(np.minimum(a, b) * nv + np.maximum(a, b))
        return np.stack([key // nv, key % nv], axis=1)
    if explicit is not None and np.size(explicit):
        e = np.sort(np.asarray(explicit, dtype=np.int64).reshape(-1, 2), axis=1)
        key = np.unique(e[:, 0] * nv + e[:, 1])
        return np.stack([key // nv, key % nv], axis=1)
    return np.zeros((0, 2), np.int64)


class Mesh:
    """Indexed triangle mesh (or face-free edge network) bound to the device.

    Construction validates like the reference (mesh.py:139-155). The device
    topology (edges, patches) is built lazily on first use by a Problem, or
    eagerly with `to_device()`.
    """

    def __init__(self, positions, faces, edges=None, patch_target: int = DEFAULT_PATCH_TARGET,
                 patch_vertices: int = DEFAULT_PATCH_VERTICES, owned=None, row_order: str = "auto"):
        if row_order not in _ROW_ORDERS:
            raise MeshError(f"row_order must be one of {sorted(_ROW_ORDERS)}")
        self.row_order = row_order
        if patch_vertices < 32:
            raise MeshError("patch_vertices must be >= 32 (one energy partial per 32-row warp)")
        positions = np.array(positions, dtype=np.float64)
        if positions.ndim != 2 or positions.shape[1] != 3:
            raise MeshError(f"positions must be (V, 3), got {positions.shape}")
        faces = np.array(faces, dtype=np.int64).reshape(-1, 3) if np.size(faces) else np.zeros((0, 3), np.int64)
        nv = len(positions)
        if faces.size:
            out = (faces < 0) | (faces >= nv)
            if out.any():
                bad = int(np.argmax(np.any(out, axis=1)))
                raise MeshError(f"face {bad} references a vertex outside 0..{nv - 1}")
            rep = (faces[:, 0] == faces[:, 1]) | (faces[:, 1] == faces[:, 2]) | (faces[:, 0] == faces[:, 2])
            if rep.any():
                raise MeshError(f"face {int(np.argmax(rep))} has repeated vertices")
            if edges is not None:
                raise MeshError("edges are derived from faces; pass explicit edges only for face-free meshes")
        explicit = None
        if not faces.size and edges is not None and np.size(edges):
            explicit = np.array(edges, dtype=np.int64).reshape(-1, 2)
            if explicit.min() < 0 or explicit.max() >= nv:
                raise MeshError("edge references a vertex out of range")
            if np.any(explicit[:, 0] == explicit[:, 1]):
                raise MeshError("edge with identical endpoints")
        self.positions = positions
        self.faces = faces
        self._explicit_edges = explicit
        self.patch_target = patch_target
        self.patch_vertices = patch_vertices
        # multi-GPU shard: rows of the vertices flagged here are assembled on
        # this device; the others are ribbon (halo) vertices (mg_mesh_set_owned)
        self.owned = None if owned is None else np.asarray(owned, dtype=bool).reshape(nv)
        self._dev = None
        self._edges = None
        self._edges_device = None

    # device ------------------------------------------------------------------

    def to_device(self):
        """Build the device topology (edges, patch layout) once; returns self."""
        if self._dev is not None:
            return self
        import torch

        lib = _lib.require_cuda()
        dev = torch.device("cuda")
        nv = len(self.positions)
        faces_d = torch.from_numpy(self.faces).to(dev) if len(self.faces) else None
        edges_d = torch.from_numpy(self._explicit_edges).to(dev) if self._explicit_edges is not None else None
        pos_d = torch.from_numpy(self.positions).to(dev) if nv else None
        handle = ctypes.c_void_p()
        torch.cuda.synchronize()
        _lib.check(lib.mg_mesh_create(
            faces_d.data_ptr() if faces_d is not None else None, len(self.faces),
            edges_d.data_ptr() if edges_d is not None else None,
            len(self._explicit_edges) if self._explicit_edges is not None else 0,
            nv, pos_d.data_ptr() if pos_d is not None else None, int(self.patch_vertices),
            _lib.stream_ptr(), ctypes.byref(handle)))
        self._dev = handle
        self._lib = lib
        if self.row_order != "auto":
            _lib.check(lib.mg_mesh_set_row_order(handle, _ROW_ORDERS[self.row_order], _lib.stream_ptr()))
        if self.owned is not None:
            own_d = torch.from_numpy(self.owned.astype(np.uint8)).to(dev)
            _lib.check(lib.mg_mesh_set_owned(handle, own_d.data_ptr() if nv else None, _lib.stream_ptr()))
        counts = [ctypes.c_int64() for _ in range(4)]
        _lib.check(lib.mg_mesh_counts(handle, *[ctypes.byref(c) for c in counts]))
        ne = counts[1].value
        e = torch.empty((ne, 2), dtype=torch.int64, device=dev)
        if ne:
            _lib.check(lib.mg_mesh_copy_edges(handle, e.data_ptr(), _lib.stream_ptr()))
        torch.cuda.synchronize()
        self._edges_device = e
        self._edges = e.cpu().numpy()
        return self

    def row_order_used(self):
        """(resolved row order, translation regularity of the numbering):
        the assembly kernels walk rows in the caller's numbering when it is
        regular (structured grids), else in Morton order (mg_mesh_row_order)."""
        self.to_device()
        o, r = ctypes.c_int(), ctypes.c_double()
        _lib.check(self._lib.mg_mesh_row_order(self._dev, ctypes.byref(o), ctypes.byref(r)))
        return {1: "morton", 2: "identity"}[o.value], r.value

    def __del__(self):
        if getattr(self, "_dev", None) is not None:
            try:
                self._lib.mg_mesh_destroy(self._dev)
            except Exception:
                pass
            self._dev = None

    # topology ----------------------------------------------------------------

    @property
    def edges(self) -> np.ndarray:
        if self._edges is None:
            try:
                import torch

                if torch.cuda.is_available() and _lib.LIB_PATH.exists():
                    self.to_device()
                    return self._edges
            except ImportError:
                pass
            self._edges = _host_edges(self.faces, self._explicit_edges, len(self.positions))
        return self._edges

    @property
    def num_vertices(self) -> int:
        return len(self.positions)

    @property
    def num_edges(self) -> int:
        return len(self.edges)

    @property
    def num_faces(self) -> int:
        return len(self.faces)

    def vertex_degrees(self) -> np.ndarray:
        e = self.edges
        return np.bincount(e.ravel(), minlength=self.num_vertices)

    def __repr__(self) -> str:
        return f"Mesh(V={self.num_vertices}, E={self.num_edges}, F={self.num_faces})"


# generators -----------------------------------------------------------------


_ROW_ORDERS = {"auto": 0, "morton": 1, "identity": 2}


def grid_arrays(n: int, spacing: float = 1.0):
    """(positions, faces) of generate_grid(n, spacing) (ref mesh.py:308-332):
    vid = j*n + i, quads split along (i,j)-(i+1,j+1), j-major face order."""
    if n < 2:
        raise ValueError("grid needs at least 2 vertices per side")
    if spacing <= 0:
        raise ValueError("spacing must be positive")
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="xy")
    pos = np.stack([ii.ravel() * spacing, jj.ravel() * spacing, np.zeros(n * n)], axis=1)
    j, i = np.meshgrid(np.arange(n - 1), np.arange(n - 1), indexing="ij")
    v00 = (j * n + i).ravel()
    f = np.empty((2 * (n - 1) ** 2, 3), np.int64)
    f[0::2, 0] = v00
    f[0::2, 1] = v00 + 1
    f[0::2, 2] = v00 + n + 1
    f[1::2, 0] = v00
    f[1::2, 1] = v00 + n + 1
    f[1::2, 2] = v00 + n
    return pos, f


def generate_grid(n: int, spacing: float = 1.0, patch_target: int = DEFAULT_PATCH_TARGET) -> Mesh:
    pos, f = grid_arrays(n, spacing)
    return Mesh(pos, f, patch_target=patch_target)


_PHI = (1.0 + np.sqrt(5.0)) / 2.0
_ICOSAHEDRON_V = [
    (-1, _PHI, 0), (1, _PHI, 0), (-1, -_PHI, 0), (1, -_PHI, 0),
    (0, -1, _PHI), (0, 1, _PHI), (0, -1, -_PHI), (0, 1, -_PHI),
    (_PHI, 0, -1), (_PHI, 0, 1), (-_PHI, 0, -1), (-_PHI, 0, 1),
]
_ICOSAHEDRON_F = [
    (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
    (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
    (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
    (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
]


def icosphere_arrays(subdivisions: int):
    """(positions, faces) of generate_icosphere(s) (ref mesh.py:351-373):
    midpoints numbered in first-request order of (a,b),(b,c),(c,a) per face,
    children (a,ab,ca),(b,bc,ab),(c,ca,bc),(ab,bc,ca)."""
    if subdivisions < 0:
        raise ValueError("subdivisions must be non-negative")
    verts = np.array([np.asarray(v, float) / np.linalg.norm(v) for v in _ICOSAHEDRON_V])
    faces = np.array(_ICOSAHEDRON_F, dtype=np.int64)
    for _ in range(subdivisions):
        nv, nf = len(verts), len(faces)
        a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
        ea = np.stack([a, b, c], 1).ravel()
        eb = np.stack([b, c, a], 1).ravel()
        key = np.minimum(ea, eb) * nv + np.maximum(ea, eb)
        _, first, inv = np.unique(key, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")
        rank = np.empty_like(order)
        rank[order] = np.arange(len(order))
        mid = nv + rank[inv]
        m = verts[ea[first[order]]] + verts[eb[first[order]]]
        # per-row BLAS dot, bitwise equal to the reference's np.linalg.norm(m)
        m = m / np.sqrt((m[:, None, :] @ m[:, :, None])[:, 0, 0])[:, None]
        verts = np.concatenate([verts, m])
        ab, bc, ca = mid.reshape(nf, 3).T
        nfaces = np.empty((4 * nf, 3), np.int64)
        nfaces[0::4] = np.stack([a, ab, ca], 1)
        nfaces[1::4] = np.stack([b, bc, ab], 1)
        nfaces[2::4] = np.stack([c, ca, bc], 1)
        nfaces[3::4] = np.stack([ab, bc, ca], 1)
        faces = nfaces
    return verts, faces


def generate_icosphere(subdivisions: int, patch_target: int = DEFAULT_PATCH_TARGET) -> Mesh:
    pos, f = icosphere_arrays(subdivisions)
    return Mesh(pos, f, patch_target=patch_target)


def punctured_icosphere_arrays(subdivisions: int):
    """Icosphere with the +z pole's fan removed and a flip-free stereographic
    UV (BASELINE config 3). Returns (positions, faces, uv)."""
    p, f = icosphere_arrays(subdivisions)
    pole = int(np.argmax(p[:, 2]))
    f = f[~np.any(f == pole, axis=1)]
    used = np.unique(f)
    remap = -np.ones(len(p), np.int64)
    remap[used] = np.arange(len(used))
    p, f = p[used], remap[f]
    uv = np.stack([p[:, 0] / (1 - p[:, 2]), p[:, 1] / (1 - p[:, 2])], axis=1)
    # det J has the sign of the UV triangle's orientation (the rest frame has
    # positive orientation): make it positive (ref apps/param.py:77-79)
    e1, e2 = uv[f[:, 1]] - uv[f[:, 0]], uv[f[:, 2]] - uv[f[:, 0]]
    if np.max(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]) < 0:
        uv = uv[:, ::-1].copy()
    return p, f, uv


# ---------------------------------------------------------------- OBJ files

def _obj_records(path):
    """(line number, tag, fields) of the v / f records of an OBJ file; every
    other record type (vn, vt, o, g, s, usemtl, ...) and comments are skipped."""
    with open(path, "r") as fh:
        for ln, line in enumerate(fh, start=1):
            fields = line.split()
            if fields and fields[0] in ("v", "f"):
                yield ln, fields[0], fields[1:]


def load_obj(path, patch_target: int = DEFAULT_PATCH_TARGET) -> "Mesh":
    """Wavefront OBJ with `v` and triangular `f` records, 1-indexed, /vt/vn
    suffixes ignored (ref mesh.py:376-418: same accepted input and MeshError
    texts, with the offending line number)."""
    pos, tri = [], []
    for ln, tag, fields in _obj_records(path):
        if tag == "v":
            if len(fields) < 3:
                raise MeshError(f"{path}: line {ln}: vertex record needs 3 coordinates")
            try:
                pos.append((float(fields[0]), float(fields[1]), float(fields[2])))
            except ValueError as exc:
                raise MeshError(f"{path}: line {ln}: bad vertex coordinate: {exc}") from None
            continue
        if len(fields) != 3:
            raise MeshError(f"{path}: line {ln}: non-triangular face with {len(fields)} vertices")
        corner = []
        for ref in fields:
            head = ref.partition("/")[0]
            try:
                k = int(head)
            except ValueError:
                raise MeshError(f"{path}: line {ln}: bad face index {head!r}") from None
            if k < 1:
                raise MeshError(f"{path}: line {ln}: face indices must be positive (1-indexed)")
            corner.append(k - 1)
        tri.append(corner)
    if not tri:
        raise MeshError(f"{path}: no faces")
    try:
        return Mesh(np.asarray(pos, dtype=np.float64).reshape(-1, 3), np.asarray(tri, dtype=np.int64),
                    patch_target=patch_target)
    except MeshError as exc:
        raise MeshError(f"{path}: {exc}") from None


def save_obj(path, positions, faces) -> None:
    """Vertices then faces, 1-indexed, 6 significant digits (ref mesh.py:421-429)."""
    p = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(faces, dtype=np.int64).reshape(-1, 3) + 1
    lines = [f"v {a:.6g} {b:.6g} {c:.6g}" for a, b, c in p]
    lines += [f"f {a} {b} {c}" for a, b, c in f]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + ("\n" if lines else ""))
