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

`ShardPlan` (torch ops: built on the GPU by DistributedProblem, on the CPU in
the gloo tests; send lists from one exchange of the recv lists) and
`HaloExchange` are tested with gloo on CPU; `DistributedProblem` runs the CUDA
engine. x is exchanged only when its owned rows changed since the last call.
"""

from __future__ import annotations

import numpy as np

__all__ = ["DistributedProblem", "HaloExchange", "ShardPlan", "morton_owner"]


_SPREAD = ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F), (4, 0x10C30C30C30C30C3),
           (2, 0x1249249249249249))


def _spread3(v):
    """Interleave the low 21 bits of v with two zero bits each (torch int64)."""
    v = v & 0x1FFFFF
    for sh, mask in _SPREAD:
        v = (v | (v << sh)) & mask
    return v


def _morton_owner_t(pos, world: int):
    """Owner rank of every vertex (torch, on pos's device): Morton order of the
    positions cut into `world` contiguous count-balanced ranges, ties broken
    by vertex id (a stable sort of the codes)."""
    import torch

    nv = pos.shape[0]
    owner = torch.zeros(nv, dtype=torch.int32, device=pos.device)
    if world <= 1 or nv == 0:
        return owner
    lo, hi = pos.min(dim=0).values, pos.max(dim=0).values
    ext = torch.where(hi > lo, hi - lo, torch.ones_like(hi))
    q = ((pos - lo) / ext).clamp(0.0, 1.0).mul(2097151.0).to(torch.int64)
    code = (_spread3(q[:, 0]) << 2) | (_spread3(q[:, 1]) << 1) | _spread3(q[:, 2])
    order = torch.sort(code, stable=True).indices
    bounds = [(r * nv) // world for r in range(world + 1)]
    for r in range(world):
        owner[order[bounds[r]:bounds[r + 1]]] = r
    return owner


def morton_owner(positions, world: int) -> np.ndarray:
    """Rank owning each vertex (numpy in / out; see _morton_owner_t)."""
    import torch

    return _morton_owner_t(torch.from_numpy(np.asarray(positions, dtype=np.float64)), world).numpy()


def range_owner(nv: int, world: int) -> np.ndarray:
    """Rank owning each vertex when the ranks own balanced contiguous global
    id ranges. For meshes numbered coherently in space (generate_grid's
    row-major grid: horizontal stripes, two ribbon rows per cut) the owned rows
    are then one contiguous slice of every shard-local array (local ids
    increase with global ids), so owned-row inputs and results are views."""
    return (np.arange(nv, dtype=np.int64) * world // max(nv, 1)).astype(np.int32)


def _edge_keys(faces, nv):
    import torch

    if faces.shape[0] == 0:
        return torch.zeros(0, dtype=torch.int64, device=faces.device)
    sides = torch.cat([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]])
    lo, hi = sides.min(dim=1).values, sides.max(dim=1).values
    return torch.unique(lo * nv + hi)  # sorted, canonical (mesh.py:184-202)


class ShardPlan:
    """One rank's view of the partition, built with torch ops on `device`
    (the GPU in production: O(mesh) device work per rank; CPU in the gloo
    tests). Attributes are numpy (local = index into this shard's vertex
    list `verts`):
      verts        global ids of the shard's vertices (sorted): owned + ribbon
      owned        (len(verts),) bool, True for vertices this rank owns
      faces        global ids of the shard's faces; local_faces their (F,3) local corners
      edges        global ids of the shard's edges (global canonical edge list order);
                   local_edges their (E,2) local endpoints
      send[q]      local ids of owned vertices that rank q holds as ribbon
      recv[q]      local ids of this shard's ribbon vertices owned by rank q
    Both lists are sorted by global id, so sender and receiver agree on order.
    With `group` (or the default group) initialised over the same world, the
    send lists come from one exchange of the recv lists (each rank builds only
    its own shard); otherwise every peer's shard is derived locally.
    """

    def __init__(self, positions, faces, edges, world: int, rank: int, owner=None, device=None, group=None):
        import torch

        dev = torch.device(device) if device is not None else torch.device("cpu")
        t = lambda a, dt: torch.as_tensor(np.asarray(a), dtype=dt, device=dev) if not torch.is_tensor(a) else a.to(dev, dt)
        pos = t(positions, torch.float64).reshape(-1, 3)
        faces_t = t(faces, torch.int64).reshape(-1, 3) if faces is not None and np.size(faces) else \
            torch.zeros((0, 3), dtype=torch.int64, device=dev)
        nv = pos.shape[0]
        self.world, self.rank, self.num_global_vertices = world, rank, nv
        self.face_free = faces_t.shape[0] == 0
        if not self.face_free:
            gkeys = _edge_keys(faces_t, nv)
        elif edges is not None and np.size(edges):
            e = t(edges, torch.int64).reshape(-1, 2)
            gkeys = torch.unique(e.min(dim=1).values * nv + e.max(dim=1).values)
        else:
            gkeys = torch.zeros(0, dtype=torch.int64, device=dev)
        gedges = torch.stack([gkeys // nv, gkeys % nv], dim=1) if nv else gkeys.reshape(0, 2)
        self.global_edges = gedges.cpu().numpy()
        own_t = _morton_owner_t(pos, world) if owner is None else t(owner, torch.int32)
        self.owner = own_t.cpu().numpy()
        elems = gedges if self.face_free else faces_t
        own_of = own_t[elems].to(torch.int64)

        def shard_of(q):
            sel = torch.nonzero((own_of == q).any(dim=1)).reshape(-1)
            vs = torch.unique(torch.cat([torch.nonzero(own_t == q).reshape(-1), elems[sel].reshape(-1)]))
            return sel, vs

        sel, verts = shard_of(rank)
        g2l = torch.full((nv,), -1, dtype=torch.int64, device=dev)
        g2l[verts] = torch.arange(verts.numel(), device=dev)
        owned_t = own_t[verts] == rank
        if self.face_free:
            self.faces = np.zeros(0, np.int64)
            self.local_faces = np.zeros((0, 3), np.int64)
            edge_ids = sel
        else:
            self.faces = sel.cpu().numpy()
            lf = g2l[faces_t[sel]]
            self.local_faces = lf.cpu().numpy()
            lkeys = _edge_keys(lf, verts.numel())
            gl = verts[lkeys // max(verts.numel(), 1)] * nv + verts[lkeys % max(verts.numel(), 1)]
            edge_ids = torch.searchsorted(gkeys, gl)
        self.edges = edge_ids.cpu().numpy()
        self.local_edges = g2l[gedges[edge_ids]].cpu().numpy() if edge_ids.numel() else np.zeros((0, 2), np.int64)
        self.verts = verts.cpu().numpy()
        self.owned = owned_t.cpu().numpy()
        self._g2l = g2l.cpu().numpy()
        # halo lists: recv from my ribbon; send by exchanging recv lists (or deriving peers' shards)
        ribbon = verts[~owned_t]
        rib_owner = own_t[ribbon]
        self.send, self.recv = {}, {}
        for q in range(world):
            if q != rank:
                self.recv[q] = g2l[ribbon[rib_owner == q]].cpu().numpy()
        import torch.distributed as dist

        if world > 1 and dist.is_initialized() and dist.get_world_size(group) == world:
            self.send = self._exchange_send(ribbon, rib_owner, g2l, group)
        else:
            mine = torch.nonzero(own_t == rank).reshape(-1)
            for q in range(world):
                if q == rank:
                    continue
                _, vq = shard_of(q)
                need = vq[torch.isin(vq, mine)]  # my owned vertices in q's shard, sorted
                self.send[q] = g2l[need].cpu().numpy()

    def _exchange_send(self, ribbon, rib_owner, g2l, group):
        """Each rank tells every owner which of its vertices it holds as ribbon
        (global ids, sorted); what arrives from q is my send list to q."""
        import torch
        import torch.distributed as dist

        world = self.world
        cpu = dist.get_backend(group) == "gloo"
        dev = torch.device("cpu") if cpu else ribbon.device
        order = torch.argsort(rib_owner.to(torch.int64) * self.num_global_vertices + ribbon)
        ids = ribbon[order].to(dev)
        counts = torch.bincount(rib_owner.to(torch.int64), minlength=world).to(dev)
        rcounts = torch.empty_like(counts)
        dist.all_to_all_single(rcounts, counts, group=group)
        got = torch.empty(int(rcounts.sum()), dtype=torch.int64, device=dev)
        dist.all_to_all_single(got, ids, rcounts.tolist(), counts.tolist(), group=group)
        send, off = {}, 0
        g2l_d = g2l.to(dev)
        for q, c in enumerate(rcounts.tolist()):
            if q != self.rank:
                send[q] = g2l_d[got[off:off + c]].cpu().numpy()
            off += c
        return send

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

    def start(self, local):
        """Post the exchange of `local`'s ribbon rows; returns a handle for
        finish(). With NCCL the transfer runs on the communicator's stream
        while the caller keeps launching work on the current stream."""
        import torch
        import torch.distributed as dist

        if self.plan.world <= 1 or not dist.is_initialized():
            return None
        view = local.view(-1, self.n)
        sendbuf = view.index_select(0, self.send_idx).reshape(-1).contiguous()
        # NCCL moves device buffers directly; gloo (CPU tests, or several ranks
        # sharing one GPU) stages them through host memory
        host = local.is_cuda and _gloo(self.group)
        if host:
            sendbuf = sendbuf.cpu()
        recvbuf = torch.empty(sum(self.recv_counts), dtype=local.dtype, device="cpu" if host else local.device)
        work = dist.all_to_all_single(recvbuf, sendbuf, self.recv_counts, self.send_counts, group=self.group,
                                      async_op=True)
        return (view, recvbuf, work, host, sendbuf)

    def finish(self, handle):
        """Wait for a posted exchange (the current stream waits on the
        communicator's) and write the ribbon rows."""
        if handle is None:
            return
        view, recvbuf, work, host, _ = handle
        work.wait()
        if host:
            recvbuf = recvbuf.to(view.device)
        view.index_copy_(0, self.recv_idx, recvbuf.view(-1, self.n))

    def exchange(self, local):
        """local: (num_local * n,) or (num_local, n) tensor; ribbon rows overwritten in place."""
        self.finish(self.start(local))
        return local


class DistributedProblem:
    """One rank's shard of a `Problem` (the CUDA engine), SPMD over
    `torch.distributed`. Mirrors the reference calls on the global problem:
    `eval_terms` returns the global energy; `grad_owned`, `hess` rows and
    `hvp` results are this rank's owned rows (global vertex order within the
    rank: `plan.owned_global`)."""

    def __init__(self, positions, faces, var_dim: int, terms, fixed_vertices=(), edges=None,
                 with_hessian: bool = True, accumulation: str = "deterministic", group=None, plan=None,
                 patch_vertices: int = 128, overlap: bool = False, partition: str = "morton"):
        """overlap (gradient-mode problems, deterministic accumulation): the
        owned rows are split into interior rows (no ribbon vertex in any
        incident element) and boundary rows, assembled by two engine problems
        on the same shard and sharing x / gradient / HVP buffers; the interior
        kernel runs while the ribbon exchange is in flight, the boundary
        kernel after it lands.

        partition: "morton" (default; balanced Morton ranges of the
        positions, any numbering) or "range" (balanced global id ranges,
        `range_owner`; owned rows become contiguous views). Ignored when
        `plan` is given."""
        import torch
        import torch.distributed as dist

        from .mesh import Element, Mesh, Op
        from .problem import Problem

        if partition not in ("morton", "range"):
            raise ValueError(f"partition must be 'morton' or 'range', got {partition!r}")
        if plan is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
            rank = dist.get_rank(group) if dist.is_initialized() else 0
            owner = range_owner(len(positions), world) if partition == "range" else None
            plan = ShardPlan(positions, faces, edges, world, rank, owner=owner, device="cuda", group=group)
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
        fixed_l = np.flatnonzero(fixed_g[pl.verts]).tolist()
        kinds = {"V": Element.VERTEX, "EV": Element.EDGE, "FV": Element.FACE}
        sterms = pl.shard_terms(terms)
        self.overlap = bool(overlap) and pl.world > 1
        if self.overlap and (with_hessian or accumulation != "deterministic"):
            raise ValueError("overlap needs a gradient-mode problem with deterministic accumulation")
        if self.overlap:
            elems = pl.local_edges if pl.face_free else pl.local_faces
            touch = (~pl.owned)[elems].any(axis=1)  # elements with a ribbon vertex
            boundary = np.zeros(pl.num_local, dtype=bool)
            boundary[elems[touch].ravel()] = True
            boundary &= pl.owned
            interior = pl.owned & ~boundary
            sub = []
            for own in (interior, boundary):
                if pl.face_free:
                    m = Mesh(positions[pl.verts], np.zeros((0, 3)), edges=pl.local_edges, owned=own,
                             patch_vertices=patch_vertices)
                else:
                    m = Mesh(positions[pl.verts], pl.local_faces, owned=own, patch_vertices=patch_vertices)
                q = Problem(m, var_dim, with_hessian=False, fixed_vertices=fixed_l, accumulation=accumulation)
                for op, t in sterms:
                    q.add_term(kinds[op], getattr(Op, op), t)
                sub.append(q)
            self.problem, self._boundary = sub
            self._boundary.x_device = self.problem.x_device  # one x / gradient for both row sets
            self._boundary.grad_device = self.problem.grad_device
            self.interior_rows, self.boundary_rows = int(interior.sum()), int(boundary.sum())
        else:
            self.problem = Problem(mesh, var_dim, with_hessian=with_hessian, fixed_vertices=fixed_l,
                                   accumulation=accumulation)
            self.interior_rows, self.boundary_rows = int(pl.owned.sum()), 0
            for op, t in sterms:
                self.problem.add_term(kinds[op], getattr(Op, op), t)
            self._boundary = None
        self.halo = HaloExchange(pl, var_dim, torch.device("cuda"), group)
        self._owned_rows = torch.as_tensor(np.flatnonzero(pl.owned), device="cuda")
        self.num_owned = int(pl.owned.sum())
        # owned rows contiguous in the local numbering (id-range partitions:
        # local ids increase with global ids): views instead of gathers
        o0 = int(np.argmax(pl.owned)) if self.num_owned else 0
        self._slice = slice(o0, o0 + self.num_owned) if pl.owned[o0:o0 + self.num_owned].all() else None
        self._v_local = None
        self._x_fresh = False  # ribbon rows of x hold their owners' current values

    # state -------------------------------------------------------------------

    def set_x_global(self, x_global) -> None:
        """Set the shard's x from a full global state (every rank passes the same array)."""
        self.problem.x = np.asarray(x_global, dtype=np.float64).reshape(-1, self.n)[self.plan.verts].ravel()
        self._x_fresh = True

    def set_x_owned(self, x_owned) -> None:
        """Set this rank's owned rows (device tensor or array, owned-row order); ribbon rows
        arrive from their owners at the next call."""
        import torch

        xl = self.problem.x_device.view(-1, self.n)
        src = torch.as_tensor(x_owned, dtype=torch.float64, device=xl.device).view(-1, self.n)
        if self._slice is not None:
            xl[self._slice].copy_(src)
        else:
            xl.index_copy_(0, self._owned_rows, src)
        self._x_fresh = False

    def _sync_x(self):
        if not self._x_fresh:
            self.halo.exchange(self.problem.x_device)
            self._x_fresh = True

    # calls -------------------------------------------------------------------

    def eval_terms(self, psd_floor=None, sync: bool = True):
        import torch.distributed as dist

        if self._boundary is not None:  # interior rows under the in-flight ribbon exchange
            h = None if self._x_fresh else self.halo.start(self.problem.x_device)
            self.problem.eval_terms(psd_floor=psd_floor, sync=False)
            self.halo.finish(h)
            self._x_fresh = True
            self._boundary.eval_terms(psd_floor=psd_floor, sync=False)
            e = self.problem.energy_device + self._boundary.energy_device
        else:
            self._sync_x()
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
        return self.owned_view(self.problem.grad_device)

    def owned_view(self, local):
        """(owned, n) rows of a shard-local array: a view when the owned rows
        are contiguous (id-range partitions), else a gather."""
        t = local.view(-1, self.n)
        return t[self._slice] if self._slice is not None else t.index_select(0, self._owned_rows)

    def hvp_owned(self, v_owned, psd_floor=None, out=None):
        """y = H v restricted to owned rows; v given on owned rows (halo-exchanged here).
        Without `out` the rows are a view of the shard's result buffer when the
        owned rows are contiguous (overwritten by the next call)."""
        import torch

        if self._v_local is None:
            self._v_local = torch.zeros_like(self.problem.x_device)
            self._y_local = torch.empty_like(self.problem.x_device)
        vl = self._v_local.view(-1, self.n)
        src = torch.as_tensor(v_owned, dtype=torch.float64, device=vl.device).view(-1, self.n)
        if self._slice is None:
            vl.index_copy_(0, self._owned_rows, src)
        elif src.data_ptr() != vl[self._slice].data_ptr():  # v_owned_buffer(): written in place
            vl[self._slice].copy_(src)
        if self._boundary is not None:
            hv = self.halo.start(self._v_local)
            hx = None if self._x_fresh else self.halo.start(self.problem.x_device)
            self.problem.hvp(self.problem.x_device, self._v_local, psd_floor=psd_floor, out=self._y_local)
            self.halo.finish(hv)
            self.halo.finish(hx)
            self._x_fresh = True
            self._boundary.hvp(self.problem.x_device, self._v_local, psd_floor=psd_floor, out=self._y_local)
            y = self._y_local
        else:
            self.halo.exchange(self._v_local)
            self._sync_x()  # x only when its owned rows changed since the last exchange
            y = self.problem.hvp(self.problem.x_device, self._v_local, psd_floor=psd_floor, out=self._y_local)
        rows = self.owned_view(y)
        if out is not None:
            out.view(-1, self.n).copy_(rows)
            return out
        return rows

    def v_owned_buffer(self):
        """The (owned, n) direction rows hvp_owned reads, as a writable view of
        the shard-local direction (id-range partitions): a caller that writes
        its direction here and passes this view skips the copy-in."""
        import torch

        if self._v_local is None:
            self._v_local = torch.zeros_like(self.problem.x_device)
            self._y_local = torch.empty_like(self.problem.x_device)
        if self._slice is None:
            raise ValueError("owned rows are not contiguous in the shard numbering (use partition='range')")
        return self._v_local.view(-1, self.n)[self._slice]

    def hvp_from_global(self, v_global, psd_floor=None):
        """Owned rows of H v for a full global v (every rank passes the same
        array; no exchange needed)."""
        import torch

        vl = torch.as_tensor(np.asarray(v_global, dtype=np.float64).reshape(-1, self.n)[self.plan.verts].ravel(),
                             device="cuda")
        y = self.problem.hvp(self.problem.x_device, vl, psd_floor=psd_floor)
        return self.owned_view(y)

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
