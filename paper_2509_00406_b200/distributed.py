"""Multi-GPU patch partition with ribbon (halo) exchange — SURVEY 8(e).

The reference is single-process (problem.py:478-502 threads over chunks); this
is the B200 build's scale-out of the same hot path. One process per GPU, with
`torch.distributed` (NCCL on B200s, gloo for the CPU tests) as the plumbing.

Design: "owner computes".
  * Partition: vertices in Morton order of their positions, cut into `world`
    contiguous ranges balanced by count; rank r owns range r.
  * Shard: every element incident to an owned vertex, on the local vertex set
    (owned + ribbon) numbered in increasing global id, so the shard's sorted
    columns map to sorted global columns and edge orientation (i < j) is
    preserved. The shard mesh restricts assembled rows to owned vertices
    (`mg_mesh_set_owned`): an element's energy counts where its first vertex
    is owned, so the shard energies sum to the global energy.
  * Per call: the ribbon x (and HVP direction v) are refreshed from their
    owners with one `all_to_all_single` (split sizes = ribbon counts per peer),
    the shard kernel runs, and the energy is summed with one `all_reduce`.
    Gradient / Hessian / HVP rows are complete on their owner: nothing else is
    communicated (ribbon elements are recomputed instead).

`ShardPlan` and `HaloExchange` are device-agnostic host logic (numpy / torch)
and are tested with gloo on CPU; `DistributedProblem` runs the CUDA engine.
"""

from __future__ import annotations

import numpy as np

from .mesh import _host_edges

__all__ = ["DistributedProblem", "HaloExchange", "ShardPlan", "morton_owner"]


def _spread3(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def morton_owner(positions: np.ndarray, world: int) -> np.ndarray:
    """Rank owning each vertex: Morton order of the positions cut into
    `world` contiguous, count-balanced ranges (ties broken by vertex id)."""
    nv = len(positions)
    if world <= 1 or nv == 0:
        return np.zeros(nv, dtype=np.int32)
    p = np.asarray(positions, dtype=np.float64)
    lo, hi = p.min(axis=0), p.max(axis=0)
    ext = np.where(hi > lo, hi - lo, 1.0)
    t = np.clip((p - lo) / ext, 0.0, 1.0)
    q = (t * 2097151.0).astype(np.uint64)
    code = (_spread3(q[:, 0]) << np.uint64(2)) | (_spread3(q[:, 1]) << np.uint64(1)) | _spread3(q[:, 2])
    order = np.lexsort((np.arange(nv), code))
    owner = np.empty(nv, dtype=np.int32)
    bounds = (np.arange(world + 1) * nv) // world
    for r in range(world):
        owner[order[bounds[r]:bounds[r + 1]]] = r
    return owner


class ShardPlan:
    """One rank's view of the partition.

    Attributes (local = index into this shard's vertex list `verts`):
      verts        global ids of the shard's vertices (sorted): owned + ribbon
      owned        (len(verts),) bool, True for vertices this rank owns
      faces        global ids of the shard's faces; local_faces their (F,3) local corners
      edges        global ids of the shard's edges (global canonical edge list order);
                   local_edges their (E,2) local endpoints
      send[q]      local ids of owned vertices that rank q holds as ribbon
      recv[q]      local ids of this shard's ribbon vertices owned by rank q
    Both lists are sorted by global id, so sender and receiver agree on order.
    """

    def __init__(self, positions, faces, edges, world: int, rank: int, owner=None):
        positions = np.asarray(positions, dtype=np.float64)
        faces = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
        nv = len(positions)
        self.world, self.rank, self.num_global_vertices = world, rank, nv
        self.global_edges = _host_edges(faces, edges, nv) if (len(faces) or edges is not None) else np.zeros((0, 2), np.int64)
        self.owner = morton_owner(positions, world) if owner is None else np.asarray(owner, dtype=np.int32)
        self.face_free = len(faces) == 0
        elems = faces if not self.face_free else self.global_edges
        own_of = self.owner[elems] if len(elems) else np.zeros((0, elems.shape[1]), np.int32)

        def shard_of(q):
            sel = np.flatnonzero(np.any(own_of == q, axis=1)) if len(elems) else np.zeros(0, np.int64)
            vs = np.unique(np.concatenate([np.flatnonzero(self.owner == q), elems[sel].ravel()]))
            return sel, vs

        sel, verts = shard_of(rank)
        self.verts = verts
        self.owned = self.owner[verts] == rank
        g2l = np.full(nv, -1, dtype=np.int64)
        g2l[verts] = np.arange(len(verts))
        self._g2l = g2l
        if self.face_free:
            self.faces = np.zeros(0, np.int64)
            self.local_faces = np.zeros((0, 3), np.int64)
            self.edges = sel
        else:
            self.faces = sel
            self.local_faces = g2l[faces[sel]]
            le = _host_edges(self.local_faces, None, len(verts))
            ge = verts[le]
            key_g = self.global_edges[:, 0] * nv + self.global_edges[:, 1]
            self.edges = np.searchsorted(key_g, ge[:, 0] * nv + ge[:, 1])
        self.local_edges = g2l[self.global_edges[self.edges]] if len(self.edges) else np.zeros((0, 2), np.int64)
        # halo lists: what every peer's shard holds of mine, and what I hold of theirs
        mine = np.flatnonzero(self.owner == rank)
        self.send, self.recv = {}, {}
        for q in range(world):
            if q == rank:
                continue
            _, vq = shard_of(q)
            need = np.intersect1d(vq, mine, assume_unique=True)       # my owned vertices in q's shard
            have = verts[(~self.owned) & (self.owner[verts] == q)]    # q's vertices in my shard
            self.send[q] = g2l[need]
            self.recv[q] = g2l[have]

    @property
    def num_local(self) -> int:
        return len(self.verts)

    @property
    def owned_global(self) -> np.ndarray:
        return self.verts[self.owned]

    def local_of(self, global_ids) -> np.ndarray:
        return self._g2l[np.asarray(global_ids)]

    def shard_terms(self, terms):
        """[(op, term)] on the shard (attributes gathered to local ids)."""
        return [(op, t.shard(self.verts, self.edges, self.faces)) for op, t in terms]


def _gloo(group) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


class HaloExchange:
    """Refresh ribbon rows of a shard-local (num_local, n) array from their
    owners: one all_to_all_single over `group` (works with NCCL and gloo)."""

    def __init__(self, plan: ShardPlan, n: int, device, group=None):
        import torch

        self.plan, self.n, self.group = plan, n, group
        peers = range(plan.world)
        self.send_counts = [len(plan.send.get(q, ())) * n for q in peers]
        self.recv_counts = [len(plan.recv.get(q, ())) * n for q in peers]
        cat = lambda parts: torch.as_tensor(np.concatenate(parts) if parts else np.zeros(0, np.int64),
                                            dtype=torch.int64, device=device)
        self.send_idx = cat([plan.send[q] for q in peers if q in plan.send])
        self.recv_idx = cat([plan.recv[q] for q in peers if q in plan.recv])
        self.bytes_per_call = 8 * (sum(self.send_counts) + sum(self.recv_counts))

    def exchange(self, local):
        """local: (num_local * n,) or (num_local, n) tensor; ribbon rows overwritten in place."""
        import torch
        import torch.distributed as dist

        if self.plan.world <= 1 or not dist.is_initialized():
            return local
        view = local.view(-1, self.n)
        sendbuf = view.index_select(0, self.send_idx).reshape(-1).contiguous()
        # NCCL moves device buffers directly; gloo (CPU tests, or several ranks
        # sharing one GPU) stages them through host memory
        host = local.is_cuda and _gloo(self.group)
        if host:
            sendbuf = sendbuf.cpu()
        recvbuf = torch.empty(sum(self.recv_counts), dtype=local.dtype, device="cpu" if host else local.device)
        dist.all_to_all_single(recvbuf, sendbuf, self.recv_counts, self.send_counts, group=self.group)
        if host:
            recvbuf = recvbuf.to(local.device)
        view.index_copy_(0, self.recv_idx, recvbuf.view(-1, self.n))
        return local


class DistributedProblem:
    """One rank's shard of a `Problem` (the CUDA engine), SPMD over
    `torch.distributed`. Mirrors the reference calls on the global problem:
    `eval_terms` returns the global energy; `grad_owned`, `hess` rows and
    `hvp` results are this rank's owned rows (global vertex order within the
    rank: `plan.owned_global`)."""

    def __init__(self, positions, faces, var_dim: int, terms, fixed_vertices=(), edges=None,
                 with_hessian: bool = True, accumulation: str = "deterministic", group=None, plan=None,
                 patch_vertices: int = 128):
        import torch
        import torch.distributed as dist

        from .mesh import Element, Mesh, Op
        from .problem import Problem

        if plan is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
            rank = dist.get_rank(group) if dist.is_initialized() else 0
            plan = ShardPlan(positions, faces, edges, world, rank)
        self.plan = plan
        pl = self.plan
        self.n = var_dim
        self.group = group
        positions = np.asarray(positions, dtype=np.float64)
        if pl.face_free:
            mesh = Mesh(positions[pl.verts], np.zeros((0, 3)), edges=pl.local_edges, owned=pl.owned,
                        patch_vertices=patch_vertices)
        else:
            mesh = Mesh(positions[pl.verts], pl.local_faces, owned=pl.owned, patch_vertices=patch_vertices)
        fixed_g = np.zeros(pl.num_global_vertices, dtype=bool)
        fixed_g[list(fixed_vertices)] = True
        self.problem = Problem(mesh, var_dim, with_hessian=with_hessian,
                               fixed_vertices=np.flatnonzero(fixed_g[pl.verts]).tolist(), accumulation=accumulation)
        kinds = {"V": Element.VERTEX, "EV": Element.EDGE, "FV": Element.FACE}
        for op, t in pl.shard_terms(terms):
            self.problem.add_term(kinds[op], getattr(Op, op), t)
        self.halo = HaloExchange(pl, var_dim, torch.device("cuda"), group)
        self._owned_rows = torch.as_tensor(np.flatnonzero(pl.owned), device="cuda")
        self._v_local = None

    # state -------------------------------------------------------------------

    def set_x_global(self, x_global) -> None:
        """Set the shard's x from a full global state (every rank passes the same array)."""
        self.problem.x = np.asarray(x_global, dtype=np.float64).reshape(-1, self.n)[self.plan.verts].ravel()

    def set_x_owned(self, x_owned) -> None:
        """Set this rank's owned rows (device tensor or array, owned-row order); ribbon rows
        arrive from their owners at the next call."""
        import torch

        xl = self.problem.x_device.view(-1, self.n)
        src = torch.as_tensor(x_owned, dtype=torch.float64, device=xl.device).view(-1, self.n)
        xl.index_copy_(0, self._owned_rows, src)

    # calls -------------------------------------------------------------------

    def eval_terms(self, psd_floor=None, sync: bool = True):
        import torch.distributed as dist

        self.halo.exchange(self.problem.x_device)
        self.problem.eval_terms(psd_floor=psd_floor, sync=False)
        e = self.problem.energy_device.clone()
        if dist.is_initialized() and self.plan.world > 1:
            if _gloo(self.group):
                eh = e.cpu()
                dist.all_reduce(eh, group=self.group)
                e = eh.to(e.device)
            else:
                dist.all_reduce(e, group=self.group)
        self.energy_device = e
        return float(e.item()) if sync else float("nan")

    def grad_owned(self):
        """(owned, n) gradient rows of this rank (device tensor)."""
        return self.problem.grad_device.view(-1, self.n).index_select(0, self._owned_rows)

    def hvp_owned(self, v_owned, psd_floor=None):
        """y = H v restricted to owned rows; v given on owned rows (halo-exchanged here)."""
        import torch

        if self._v_local is None:
            self._v_local = torch.zeros_like(self.problem.x_device)
        vl = self._v_local.view(-1, self.n)
        vl.index_copy_(0, self._owned_rows, torch.as_tensor(v_owned, dtype=torch.float64, device=vl.device).view(-1, self.n))
        self.halo.exchange(self._v_local)
        self.halo.exchange(self.problem.x_device)
        y = self.problem.hvp(self.problem.x_device, self._v_local, psd_floor=psd_floor)
        return y.view(-1, self.n).index_select(0, self._owned_rows)

    def hvp_from_global(self, v_global, psd_floor=None):
        """Owned rows of H v for a full global v (every rank passes the same
        array; no exchange needed)."""
        import torch

        vl = torch.as_tensor(np.asarray(v_global, dtype=np.float64).reshape(-1, self.n)[self.plan.verts].ravel(),
                             device="cuda")
        y = self.problem.hvp(self.problem.x_device, vl, psd_floor=psd_floor)
        return y.view(-1, self.n).index_select(0, self._owned_rows)

    def hess_rows_owned(self):
        """(row_offsets, global col_indices, values) of the owned rows, in owned-row order."""
        h = self.problem.hess
        rows = np.flatnonzero(self.plan.owned)
        ro = h.row_offsets
        lens = ro[rows + 1] - ro[rows]
        take = np.concatenate([np.arange(ro[r], ro[r + 1]) for r in rows]) if len(rows) else np.zeros(0, np.int64)
        cols = self.plan.verts[h.col_indices[take]]
        vals = h.values[take]
        offs = np.concatenate([[0], np.cumsum(lens)])
        return offs, cols, vals
