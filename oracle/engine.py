"""Oracle restatement of the reference Problem pipeline (problem.py:243-617).

Given the same mesh arrays, terms (callables with the reference callback
signature) and states, `OracleProblem` computes energy, gradient, the block
CSR Hessian (pattern + values), energy-only probes and HVPs exactly the way
the reference does: lift with unit seeds (free-masked), call the term on a
batch, extract (broadcast, symmetrise, optional PSD via eigh), scatter with
np.add.at into padded buffers with dump slots for pinned rows.

Differences that only move rounding: elements are processed in element-id
order (the reference sorts by BFS patch first, problem.py:366) and chunks are
plain 4096-element ranges.
"""

from __future__ import annotations

import itertools
import os
from collections import deque
from concurrent.futures import ThreadPoolExecutor, as_completed

import numpy as np

from .dual import Dual, project_psd

_P_OF_OP = {"FV": 3, "EV": 2, "V": 1}


class _Handle:
    """Batch handle passed to callbacks (problem.py:170-183): `index` holds
    element ids; vertex handles carry their local slot."""

    __slots__ = ("kind", "index", "slot")

    def __init__(self, kind, index, slot=None):
        self.kind = kind
        self.index = index
        self.slot = slot


class _Slots:
    __slots__ = ("vecs",)

    def __init__(self, vecs):
        self.vecs = vecs

    def __getitem__(self, h):
        if h.slot is None:
            raise KeyError("non-vertex handle carries no variables")
        return self.vecs[h.slot]


class _Group:
    __slots__ = ("ids", "sel", "free", "gidx", "bids")

    def __init__(self, ids, sel, free, gidx):
        self.ids = ids
        self.sel = sel
        self.free = free
        self.gidx = gidx
        self.bids = None


def derive_edges(faces: np.ndarray, nv: int, explicit=None) -> np.ndarray:
    """Canonical sorted edges (mesh.py:184-202)."""
    faces = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
    if len(faces):
        sides = np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]])
        return np.unique(np.sort(sides, axis=1), axis=0)
    if explicit is not None and np.size(explicit):
        return np.unique(np.sort(np.asarray(explicit, dtype=np.int64).reshape(-1, 2), axis=1), axis=0)
    return np.zeros((0, 2), np.int64)


def pattern_keys(nv, sels, fixed=None):
    """Sorted unique pair keys row*nv + col of every ordered (a, b) vertex
    pair of every element, both free (problem.py:389-398)."""
    keyset = []
    for sel in sels:
        sel = np.asarray(sel, dtype=np.int64)
        k = sel[:, :, None] * nv + sel[:, None, :]
        if fixed is not None:
            fm = ~fixed[sel]
            k = k[fm[:, :, None] & fm[:, None, :]]
        keyset.append(k.ravel())
    return np.unique(np.concatenate(keyset)) if keyset else np.zeros(0, np.int64)


def pattern_from_keys(keys, nv):
    """int64 row_offsets (nv+1) and col_indices from sorted keys
    (problem.py:399-402)."""
    rows, cols = keys // nv, keys % nv
    ro = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=nv), out=ro[1:])
    return ro, cols


def sparsity_pattern(nv, sels, fixed=None):
    """(row_offsets, col_indices) of the block Hessian (problem.py:383-402)."""
    return pattern_from_keys(pattern_keys(nv, sels, fixed), nv)


def _pairwise_total(parts) -> float:
    vals = [float(p) for p in parts]
    if not vals:
        return 0.0
    while len(vals) > 1:
        nxt = [vals[i] + vals[i + 1] for i in range(0, len(vals) - 1, 2)]
        if len(vals) % 2:
            nxt.append(vals[-1])
        vals = nxt
    return vals[0]


class OracleProblem:
    """CPU restatement of `meshgrad.Problem` for FV / EV / V terms.

    terms: list of (op_name, callable) with op_name in {"FV","EV","V"}.
    """

    def __init__(self, num_vertices, faces, edges, n, terms, with_hessian=True, fixed_vertices=(),
                 workers=1, accumulation="deterministic", chunk=4096, element_ids=None):
        """`element_ids` (optional, one entry per term, None = all): evaluate
        only these global element ids of each term. Callbacks still see
        global ids in `handle.index`, so closure arrays index correctly. A
        vertex row whose incident elements are all included is complete
        (gradient, Hessian row, HVP row: problem.py:535-544 scatter only
        inside an element's own vertices), which is what the at-scale
        sampled-row parity tests rely on."""
        self.nv = int(num_vertices)
        self.faces = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
        self.edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        self.n = int(n)
        self.with_hessian = with_hessian
        self.fixed = np.zeros(self.nv, dtype=bool)
        self.fixed[list(fixed_vertices)] = True
        self.workers = max(1, int(workers))
        self.accumulation = accumulation
        self.chunk = int(chunk)
        self.task_slice = None
        self.ndofs = self.n * self.nv
        self.terms = [(op, fn) for op, fn in terms]
        ids = list(element_ids) if element_ids is not None else [None] * len(self.terms)
        self.groups = [self._layout(op, i) for (op, _), i in zip(self.terms, ids)]
        self.row_offsets = self.col_indices = None
        self.nnzb = None
        if with_hessian:
            self.precompute_sparsity()

    # layout (problem.py:327-379) ----------------------------------------------
    def _layout(self, op, subset=None):
        if op == "FV":
            sel = self.faces
        elif op == "EV":
            sel = self.edges
        elif op == "V":
            sel = np.arange(self.nv, dtype=np.int64)[:, None]
        else:
            raise ValueError(f"oracle supports FV, EV, V terms, not {op}")
        ids = np.arange(len(sel), dtype=np.int64)
        if subset is not None:
            ids = np.asarray(subset, dtype=np.int64)
            sel = sel[ids]
        free = (~self.fixed[sel]).astype(np.float64) if self.fixed.any() else None
        gidx = (sel[:, :, None] * self.n + np.arange(self.n)).reshape(len(ids), -1)
        if free is not None:
            gidx = np.where(np.repeat(free.astype(bool), self.n, axis=1), gidx, self.ndofs)
        return _Group(ids, np.ascontiguousarray(sel), free, gidx)

    # sparsity (problem.py:383-416) --------------------------------------------
    def precompute_sparsity(self):
        nv = self.nv
        keys = pattern_keys(nv, [g.sel for g in self.groups], self.fixed if self.fixed.any() else None)
        ro, cols = pattern_from_keys(keys, nv)
        self.row_offsets, self.col_indices, self.nnzb = ro, cols, len(keys)
        for g in self.groups:
            b = np.searchsorted(keys, g.sel[:, :, None] * nv + g.sel[:, None, :])
            if g.free is not None:
                fm = g.free.astype(bool)
                b = np.where(fm[:, :, None] & fm[:, None, :], b, self.nnzb)
            g.bids = b
        return ro, cols

    # per-chunk work (problem.py:420-476) ---------------------------------------
    def _lift(self, g, sl, x2d, mode):
        sel = g.sel[sl]
        m, p = sel.shape
        vals = x2d[sel]
        from paper_2509_00406_b200.active import ActiveVec

        if mode == "passive":
            return [ActiveVec([Dual(vals[:, q, c]) for c in range(self.n)]) for q in range(p)]
        k = p * self.n
        second = mode != "gradient"
        free = g.free[sl] if g.free is not None else None
        out = []
        for q in range(p):
            comps = []
            for c in range(self.n):
                seed = np.zeros((m, k))
                seed[:, q * self.n + c] = 1.0 if free is None else free[:, q]
                comps.append(Dual(vals[:, q, c], seed, 0.0 if second else None))
            out.append(ActiveVec(comps))
        return out

    def _call(self, op, fn, g, sl, slots):
        sel = g.sel[sl]
        ids = g.ids[sl]
        if op == "V":
            h = _Handle("vertex", ids, 0)
            return fn(h, (h,), _Slots(slots))
        h = _Handle("edge" if op == "EV" else "face", ids, None)
        nb = tuple(_Handle("vertex", sel[:, q], q) for q in range(sel.shape[1]))
        return fn(h, nb, _Slots(slots))

    @staticmethod
    def _extract(res, m, k, want_h, floor):
        f = np.broadcast_to(np.asarray(res.val, dtype=np.float64), (m,))
        g = None if res.jac is None else np.broadcast_to(np.asarray(res.jac, dtype=np.float64), (m, k))
        h = None
        if want_h:
            if res.jac is not None and isinstance(res.hes, np.ndarray):
                h = np.broadcast_to(res.hes, (m, k, k))
            elif floor is not None:
                h = np.zeros((m, k, k))
            if h is not None:
                h = 0.5 * (h + np.swapaxes(h, -1, -2))
                if floor is not None:
                    ok = np.isfinite(h).all(axis=(-2, -1))
                    if ok.all():
                        h = project_psd(h, floor)
                    else:
                        h = np.array(h)
                        h[ok] = project_psd(h[ok], floor)
        return f, g, h

    def _tasks(self):
        out = []
        for t, (op, fn) in enumerate(self.terms):
            g = self.groups[t]
            for s in range(0, len(g.ids), self.chunk):
                out.append((op, fn, g, slice(s, min(s + self.chunk, len(g.ids)))))
        return out

    def _run(self, fn):
        tasks = self._tasks()
        if self.task_slice is not None:  # a bounded sample of the call's chunks (bench CPU baseline)
            tasks = tasks[self.task_slice]
        if self.workers <= 1 or len(tasks) <= 1:
            for t in tasks:
                yield fn(t)
            return
        with ThreadPoolExecutor(max_workers=self.workers) as ex:
            if self.accumulation == "atomic":
                for fut in as_completed([ex.submit(fn, t) for t in tasks]):
                    yield fut.result()
            else:
                it = iter(tasks)
                pend = deque(ex.submit(fn, t) for t in itertools.islice(it, 4 * self.workers))
                while pend:
                    r = pend.popleft().result()
                    nxt = next(it, None)
                    if nxt is not None:
                        pend.append(ex.submit(fn, nxt))
                    yield r

    def _reduce(self, parts):
        return _pairwise_total(parts) if self.accumulation == "deterministic" else float(np.sum(parts))

    # public (problem.py:504-617) -------------------------------------------------
    def eval_terms(self, x, psd_floor=None):
        """Returns (energy, grad (n*V), hess values (nnzb,n,n) or None)."""
        if psd_floor is not None and not self.with_hessian:
            raise ValueError("psd_floor requires a Hessian-mode problem")
        n = self.n
        x2d = np.asarray(x, dtype=np.float64).reshape(self.nv, n)
        gpad = np.zeros(self.ndofs + 1)
        hpad = np.zeros((self.nnzb + 1, n, n)) if self.with_hessian else None
        mode = "hessian" if self.with_hessian else "gradient"

        def work(task):
            op, fn, g, sl = task
            m = sl.stop - sl.start
            p = g.sel.shape[1]
            res = self._call(op, fn, g, sl, self._lift(g, sl, x2d, mode))
            f, gr, h = self._extract(res, m, p * n, self.with_hessian, psd_floor)
            blocks = None
            if h is not None:
                blocks = h.reshape(m, p, n, p, n).transpose(0, 1, 3, 2, 4).reshape(-1, n, n)
            return float(np.sum(f)), gr, g.gidx[sl], (g.bids[sl].ravel() if blocks is not None else None), blocks

        parts = []
        for fs, gr, gidx, bids, blocks in self._run(work):
            parts.append(fs)
            if gr is not None:
                np.add.at(gpad, gidx.ravel(), gr.ravel())
            if blocks is not None:
                np.add.at(hpad, bids, blocks)
        if self.task_slice is not None:  # a timed sample: views (the reference returns its buffers, no copy)
            return self._reduce(parts), gpad[: self.ndofs], (hpad[: self.nnzb] if hpad is not None else None)
        return self._reduce(parts), gpad[: self.ndofs].copy(), (hpad[: self.nnzb].copy() if hpad is not None else None)

    def eval_energy_only(self, x):
        x2d = np.asarray(x, dtype=np.float64).reshape(self.nv, self.n)

        def work(task):
            op, fn, g, sl = task
            res = self._call(op, fn, g, sl, self._lift(g, sl, x2d, "passive"))
            return float(np.sum(np.broadcast_to(np.asarray(res.val, dtype=np.float64), (sl.stop - sl.start,))))

        return self._reduce(list(self._run(work)))

    def hvp(self, x, v, psd_floor=None):
        n = self.n
        x2d = np.asarray(x, dtype=np.float64).reshape(self.nv, n)
        v2d = np.asarray(v, dtype=np.float64).reshape(self.nv, n)
        ypad = np.zeros(self.ndofs + 1)

        def work(task):
            op, fn, g, sl = task
            m = sl.stop - sl.start
            k = g.sel.shape[1] * n
            res = self._call(op, fn, g, sl, self._lift(g, sl, x2d, "hessian"))
            _, _, h = self._extract(res, m, k, True, psd_floor)
            if h is None:
                return None, None
            vloc = v2d[g.sel[sl]].reshape(m, k)
            if g.free is not None:
                vloc = vloc * np.repeat(g.free[sl], n, axis=1)
            return g.gidx[sl], np.einsum("mij,mj->mi", h, vloc)

        for gidx, y in self._run(work):
            if y is not None:
                np.add.at(ypad, gidx.ravel(), y.ravel())
        return ypad[: self.ndofs] if self.task_slice is not None else ypad[: self.ndofs].copy()


def default_workers():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
