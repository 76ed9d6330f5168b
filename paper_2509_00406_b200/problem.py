"""`Problem` — the reference's hot-path API over the CUDA engine.

Same constructor, methods, attributes and error behaviour as
`meshgrad.problem.Problem` (problem.py:243-629); the work happens in
`libmeshgrad_b200.so` (include/meshgrad_b200.h):

  eval_terms        -> mg_eval   (grad + block-CSR Hessian, optional PSD clamp)
  eval_energy_only  -> mg_energy
  hvp               -> mg_hvp    (matrix free; forward-over-forward duals)
  precompute_sparsity -> mg_precompute_sparsity (device-built pattern)

State lives on the GPU (`x_device`, `grad_device`, `hess.values_device`);
the numpy views the reference exposes (`x`, `grad`, `hess.values`) are copied
to the host lazily on access. There is no CPU fallback: without the library or
a CUDA device the constructor raises.
"""

from __future__ import annotations

import ctypes
import os
import time
import weakref

import numpy as np

from . import _lib
from .mesh import DEFAULT_VALENCE_CAP, Element, Mesh, Op, SOURCE_KIND
from .terms import BuiltinTerm

__all__ = ["BlockSparseMatrix", "Problem", "read_matrix_market"]

_TERM_OPS = (Op.FV, Op.EV, Op.VV, Op.V)


def _torch():
    import torch

    return torch


def _as_device(a, torch, dev):
    if isinstance(a, torch.Tensor):
        if a.device.type != "cuda" or a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("attribute tensors must be contiguous float64 CUDA tensors")
        return a
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(dev)


class BlockSparseMatrix:
    """Symmetric block-CSR Hessian (ref problem.py:57-146). Pattern arrays are
    int64 host numpy (bit-exact with the reference); `values` is pulled from
    the device on access; `values_device` is the live (nnzb, n, n) tensor."""

    def __init__(self, block_dim, num_block_rows, row_offsets, col_indices, values_device, problem=None):
        self.block_dim = block_dim
        self.num_block_rows = num_block_rows
        self.row_offsets = row_offsets
        self.col_indices = col_indices
        self.values_device = values_device
        self._problem_ref = weakref.ref(problem) if problem is not None else None
        self._block_rows = np.repeat(np.arange(num_block_rows, dtype=np.int64), np.diff(row_offsets))

    @property
    def values(self) -> np.ndarray:
        return self.values_device.cpu().numpy()

    @property
    def nnz_blocks(self) -> int:
        return len(self.col_indices)

    @property
    def nnz_scalar(self) -> int:
        return self.nnz_blocks * self.block_dim * self.block_dim

    @property
    def shape(self):
        n = self.num_block_rows * self.block_dim
        return (n, n)

    def block_index(self, i: int, j: int):
        lo, hi = self.row_offsets[i], self.row_offsets[i + 1]
        k = lo + np.searchsorted(self.col_indices[lo:hi], j)
        if k < hi and self.col_indices[k] == j:
            return int(k)
        return None

    def block(self, i: int, j: int):
        k = self.block_index(i, j)
        return None if k is None else self.values_device[k].cpu().numpy()

    def block_pairs(self):
        return np.stack([self._block_rows, self.col_indices], axis=1)

    @property
    def _problem(self):
        return self._problem_ref() if self._problem_ref is not None else None

    def matvec(self, v):
        """H v with the device block-CSR SpMV (problem.py:100-106)."""
        torch = _torch()
        p = self._problem
        host = not isinstance(v, torch.Tensor)
        n = self.num_block_rows * self.block_dim
        if (v.numel() if not host else np.size(v)) != n:
            raise ValueError(f"cannot reshape array of size {np.size(v) if host else v.numel()} into shape ({n},)")
        vd = _as_device(v if not host else np.asarray(v, dtype=np.float64).reshape(-1), torch,
                        torch.device("cuda")).reshape(-1)
        y = torch.empty_like(vd)
        _lib.check(p._lib.mg_bsr_matvec(p._h, self.values_device.data_ptr(), vd.data_ptr(), y.data_ptr(),
                                        _lib.stream_ptr()))
        return y.cpu().numpy() if host else y

    def to_dense(self) -> np.ndarray:
        n = self.block_dim
        size = self.num_block_rows * n
        dense = np.zeros((size, size))
        vals = self.values
        for k in range(self.nnz_blocks):
            i = self._block_rows[k]
            j = self.col_indices[k]
            dense[i * n:(i + 1) * n, j * n:(j + 1) * n] = vals[k]
        return dense

    def diagonal_block_inverses(self) -> np.ndarray:
        n = self.block_dim
        inv = np.tile(np.eye(n), (self.num_block_rows, 1, 1))
        vals = self.values
        diag = self.col_indices == self._block_rows
        rows = self._block_rows[diag]
        blocks = vals[diag]
        for r, b in zip(rows, blocks):
            try:
                inv[r] = np.linalg.inv(b)
            except np.linalg.LinAlgError:
                pass
        return inv

    def write_matrix_market(self, path) -> None:
        """Coordinate format, 1-indexed, every stored entry, 17 significant
        digits (ref problem.py:133-146)."""
        n = self.block_dim
        vals = self.values
        rows = (self._block_rows[:, None, None] * n + np.arange(n)[None, :, None] + 1)
        cols = (self.col_indices[:, None, None] * n + np.arange(n)[None, None, :] + 1)
        rows = np.broadcast_to(rows, vals.shape).ravel()
        cols = np.broadcast_to(cols, vals.shape).ravel()
        flat = vals.ravel()
        with open(path, "w") as fh:
            fh.write("%%MatrixMarket matrix coordinate real general\n")
            size = self.num_block_rows * n
            fh.write(f"{size} {size} {self.nnz_scalar}\n")
            fh.writelines(f"{r} {c} {v:.17g}\n" for r, c, v in zip(rows.tolist(), cols.tolist(), flat.tolist()))


def read_matrix_market(path):
    """Inverse of write_matrix_market (ref problem.py:149-167)."""
    with open(path) as fh:
        header = fh.readline()
        if not header.startswith("%%MatrixMarket matrix coordinate real"):
            raise ValueError(f"{path}: unsupported MatrixMarket header: {header.strip()}")
        line = fh.readline()
        while line.startswith("%"):
            line = fh.readline()
        rows, cols, nnz = (int(t) for t in line.split())
        entries = []
        for _ in range(nnz):
            i, j, v = fh.readline().split()
            entries.append((int(i) - 1, int(j) - 1, float(v)))
    return rows, cols, entries


class _TermRecord:
    __slots__ = ("term", "kind", "op", "host_attrs", "dev_attrs", "tid", "traced", "groups", "sel", "index", "error")

    def __init__(self, term, kind, op):
        self.term = term
        self.kind = kind
        self.op = op
        self.host_attrs = []
        self.dev_attrs = []
        self.tid = -1
        self.traced = None
        self.groups = None  # VV: one engine term per valence group (sub-records)
        self.sel = None     # VV group: (M, P) neighbourhoods (host) and their device copy in dev_attrs' keep-alive
        self.index = None   # VV group: center vertex ids
        self.error = None   # deferred layout error (valence cap), raised like the reference at layout time


class Problem:
    """Registered builtin energy terms plus the device evaluation state
    (ref problem.py:243-297). `workers` and `chunk_elements` are accepted for
    signature compatibility; the device decomposes work by patches."""

    def __init__(self, mesh: Mesh, var_dim: int, with_hessian: bool = True,
                 fixed_vertices=(), accumulation: str = "deterministic",
                 workers: int = 1, valence_cap: int = DEFAULT_VALENCE_CAP,
                 chunk_elements: int = 4096, live_host_attrs: bool = True, dtype=None):
        if var_dim < 1:
            raise ValueError("var_dim must be at least 1")
        if accumulation not in ("deterministic", "atomic"):
            raise ValueError(f"unknown accumulation mode {accumulation!r}")
        if os.environ.get("MESHGRAD_DETERMINISTIC") == "1":
            accumulation = "deterministic"
        torch = _torch()
        self._lib = _lib.require_cuda()
        # storage precision (the reference computes in float64, active.py:333):
        # float32 halves every stream's bytes; the kernels still compute in fp64
        # (mg_problem_set_storage). Edge row kernels only: builtin vertex and
        # radial edge terms, deterministic accumulation; eval_terms / hvp /
        # eval_energy_only (the solvers' BSR kernels stay fp64).
        self.dtype = torch.float64 if dtype is None else dtype
        if self.dtype not in (torch.float64, torch.float32):
            raise ValueError("dtype must be torch.float64 or torch.float32")
        if self.dtype == torch.float32 and accumulation != "deterministic":
            raise ValueError("float32 storage needs deterministic accumulation")
        self.mesh = mesh
        self.n = var_dim
        self.with_hessian = with_hessian
        self.accumulation = accumulation
        self.workers = max(1, int(workers))
        self.valence_cap = valence_cap
        self._chunk_elements = chunk_elements
        self.live_host_attrs = live_host_attrs
        nv = mesh.num_vertices
        self._fixed = np.zeros(nv, dtype=bool)
        for v in fixed_vertices:
            self._fixed[v] = True
        self._num_dofs = var_dim * nv
        self._dev = torch.device("cuda")
        mesh.to_device()
        self._fixed_device = torch.from_numpy(self._fixed.astype(np.uint8)).to(self._dev)
        h = ctypes.c_void_p()
        _lib.check(self._lib.mg_problem_create(mesh._dev, var_dim, int(bool(with_hessian)),
                                               self._fixed_device.data_ptr() if nv else None,
                                               int(accumulation == "deterministic"), ctypes.byref(h)))
        self._h = h
        if self.dtype == torch.float32:
            _lib.check(self._lib.mg_problem_set_storage(h, 32))
        self.x_device = torch.zeros(self._num_dofs, dtype=self.dtype, device=self._dev)
        self.grad_device = torch.zeros(self._num_dofs, dtype=self.dtype, device=self._dev)
        self._energy_device = torch.full((1,), float("nan"), dtype=torch.float64, device=self._dev)
        self.hess: BlockSparseMatrix | None = None
        self.energy: float = float("nan")
        self._terms: list[_TermRecord] = []
        self._pattern_ready = False
        self._patch_checked = False
        self.patch_module = False  # traced terms run through a generated patch module
        self.row_module = False  # ... and, radial edge terms, through a generated row module
        self.stats = {
            "eval_terms_calls": 0, "eval_terms_ms": 0.0,
            "energy_only_calls": 0, "energy_only_ms": 0.0,
            "hvp_calls": 0, "hvp_ms": 0.0,
        }

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            try:
                self._lib.mg_problem_destroy(self._h)
            except Exception:
                pass
            self._h = None

    # registration ----------------------------------------------------------

    def add_term(self, kind: Element, op: Op, fn) -> int:
        """Register a per-element energy (ref problem.py:301-310). `fn` must be
        a builtin term from `paper_2509_00406_b200.terms`."""
        if SOURCE_KIND[op] is not kind:
            raise ValueError(f"{op.name} iterates over {SOURCE_KIND[op].value} elements, not {kind.value}")
        self._patch_checked = self.patch_module = self.row_module = False  # the library drops a generated patch module on add
        if op not in _TERM_OPS:
            raise ValueError(f"{op.name} does not resolve to vertex variables; terms support FV, EV, VV, V")
        if not isinstance(fn, BuiltinTerm):
            return self._add_traced_term(kind, op, fn)
        if op is not fn.op:
            raise ValueError(f"{type(fn).__name__} is an {fn.op.name} term, registered with {op.name}")
        fn.check_dims(self.n)
        torch = _torch()
        rec = _TermRecord(fn, kind, op)
        for a in fn.attrs():
            if self.dtype == torch.float32:  # fp32 copies (a CUDA tensor is snapshotted: refresh_attrs updates)
                rec.host_attrs.append(a)
                rec.dev_attrs.append(_as_device(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a,
                                                torch, self._dev).to(torch.float32))
                continue
            rec.host_attrs.append(None if isinstance(a, torch.Tensor) else a)
            rec.dev_attrs.append(_as_device(a, torch, self._dev))
        params = fn.params(self.n)
        cparams = (ctypes.c_double * max(1, len(params)))(*params)
        cattrs = (ctypes.c_void_p * max(1, len(rec.dev_attrs)))(*[t.data_ptr() for t in rec.dev_attrs])
        tid = ctypes.c_int()
        _lib.check(self._lib.mg_problem_add_term(self._h, fn.type_id, _lib.MG_OP[op.name], cparams, len(params),
                                                 cattrs, len(rec.dev_attrs), ctypes.byref(tid)))
        rec.tid = tid.value
        self._terms.append(rec)
        self._pattern_ready = False
        self._patch_checked = self.patch_module = self.row_module = False
        return len(self._terms) - 1

    def _num_elements(self, op: Op) -> int:
        return {Op.V: self.mesh.num_vertices, Op.EV: self.mesh.num_edges, Op.FV: self.mesh.num_faces}[op]

    def _element_vertices(self, op: Op):
        return {Op.V: None, Op.EV: self.mesh.edges, Op.FV: self.mesh.faces}[op]

    def _add_traced_term(self, kind: Element, op: Op, fn) -> int:
        if self.dtype != _torch().float64:
            raise NotImplementedError("float32 storage supports the builtin terms only")
        return self._add_traced_term64(kind, op, fn)

    def _add_traced_term64(self, kind: Element, op: Op, fn) -> int:
        """A general callback (ref problem.py:8-14, 301-310): traced once on
        symbolic inputs, compiled to an sm_100a module, launched by the engine
        (jit.py). Closure arrays indexed by `handle.index` become per-element
        attribute streams (refresh_attrs() re-gathers them)."""
        if op is Op.VV:
            return self._add_vv_term(kind, fn)
        from . import jit

        torch = _torch()
        tt = jit.trace_callback(fn, op.name, self.n, self._num_elements(op), self._element_vertices(op))
        image = jit.compile_term(tt)
        rec = _TermRecord(fn, kind, op)
        rec.traced = tt
        rec.dev_attrs = [torch.from_numpy(a).to(self._dev) for a in tt.attrs]
        rec.host_attrs = [None] * len(rec.dev_attrs)
        buf = ctypes.create_string_buffer(image, len(image))
        cattrs = (ctypes.c_void_p * max(1, len(rec.dev_attrs)))(*[t.data_ptr() for t in rec.dev_attrs])
        tid = ctypes.c_int()
        _lib.check(self._lib.mg_problem_add_jit_term(self._h, _lib.MG_OP[op.name], self.n, buf, cattrs,
                                                     len(rec.dev_attrs), ctypes.byref(tid)))
        rec.tid = tid.value
        self._terms.append(rec)
        self._pattern_ready = False
        self._patch_checked = self.patch_module = self.row_module = False
        return len(self._terms) - 1

    def _one_rings(self):
        """Vertex -> one-ring, ascending (ref mesh.py vertex_to_vertex): CSR over the edges."""
        e = np.asarray(self.mesh.edges, dtype=np.int64).reshape(-1, 2)
        nv = self.mesh.num_vertices
        a = np.concatenate([e[:, 0], e[:, 1]])
        b = np.concatenate([e[:, 1], e[:, 0]])
        order = np.lexsort((b, a))
        a, b = a[order], b[order]
        off = np.zeros(nv + 1, dtype=np.int64)
        np.cumsum(np.bincount(a, minlength=nv), out=off[1:])
        return off, b

    def _add_vv_term(self, kind: Element, fn) -> int:
        """A traced VV term (ref problem.py:340-353): the neighbourhood (center,
        one-ring ascending) has one arity per valence, so each valence group is
        traced and registered as its own engine term over an explicit
        selection; a valence above the cap fails at layout time, as in the
        reference."""
        from . import jit

        torch = _torch()
        rec = _TermRecord(fn, kind, Op.VV)
        rec.groups = []
        off, ring = self._one_rings()
        degs = np.diff(off)
        if degs.size and degs.max() > self.valence_cap:
            worst = int(np.argmax(degs))
            rec.error = ValueError(
                f"vertex {worst} has valence {int(degs[worst])}, exceeding the cap {self.valence_cap}")
            self._terms.append(rec)
            self._pattern_ready = False
            return len(self._terms) - 1
        for d in np.unique(degs):
            ids = np.flatnonzero(degs == d).astype(np.int64)
            sel = np.empty((len(ids), 1 + int(d)), dtype=np.int64)
            sel[:, 0] = ids
            if d:
                sel[:, 1:] = ring[off[ids][:, None] + np.arange(int(d))]
            tt = jit.trace_callback(fn, "VV", self.n, len(ids), sel, index=ids)
            image = jit.compile_term(tt)
            sub = _TermRecord(fn, kind, Op.VV)
            sub.traced = tt
            sub.sel, sub.index = sel, ids
            sub.dev_attrs = [torch.from_numpy(a).to(self._dev) for a in tt.attrs]
            sub.host_attrs = [torch.from_numpy(sel.astype(np.int32)).to(self._dev)]  # keeps the selection alive
            buf = ctypes.create_string_buffer(image, len(image))
            cattrs = (ctypes.c_void_p * max(1, len(sub.dev_attrs)))(*[t.data_ptr() for t in sub.dev_attrs])
            tid = ctypes.c_int()
            _lib.check(self._lib.mg_problem_add_jit_term_sel(
                self._h, _lib.MG_OP["VV"], self.n, sel.shape[1], sub.host_attrs[0].data_ptr(), len(ids), buf, cattrs,
                len(sub.dev_attrs), ctypes.byref(tid)))
            sub.tid = tid.value
            rec.groups.append(sub)
        self._terms.append(rec)
        self._pattern_ready = False
        return len(self._terms) - 1

    def _check_terms(self):
        if not self._terms:
            raise ValueError("no energy terms registered")
        for rec in self._terms:
            if rec.error is not None:
                raise rec.error
        if not self._patch_checked:
            self._patch_checked = True
            self._use_patch_module()

    def _use_patch_module(self):
        """Traced terms on the patch-owner path: when every term is a traced
        V / EV / FV callback, deterministic accumulation, and the problem has
        at least MG_JIT_PATCH_MIN elements (default 65536; smaller problems
        keep the element-parallel kernels, compiled once per term), generate
        and compile one module with all the problem's functors and hand it to
        the library (mg_problem_set_patch_module)."""
        from . import jit

        recs = self._terms
        if self.accumulation != "deterministic" or not all(r.traced is not None and r.groups is None for r in recs):
            return
        if len(recs) > 8 or self.mesh.num_vertices == 0:
            return
        total = sum(self._num_elements(r.op) for r in recs)
        if total < int(os.environ.get("MG_JIT_PATCH_MIN", "65536")):
            return
        image = jit.compile_patch([r.traced for r in recs], self.n)
        buf = ctypes.create_string_buffer(image, len(image))
        _lib.check(self._lib.mg_problem_set_patch_module(self._h, buf))
        self.patch_module = True
        # every EV callback radial (proved on the trace), the rest V terms: the
        # edge row kernel, with the patch module as its exact re-run
        if os.environ.get("MG_JIT_ROWS", "1") != "0":
            rimage = jit.compile_rows([r.traced for r in recs], self.n)
            if rimage is not None:
                rbuf = ctypes.create_string_buffer(rimage, len(rimage))
                _lib.check(self._lib.mg_problem_set_row_module(self._h, rbuf))
                self.row_module = True

    def _sync_attrs(self):
        if self.live_host_attrs:
            self.refresh_attrs(only_host=True)

    def refresh_attrs(self, only_host: bool = False):
        """Re-upload the host (numpy) attribute arrays of every term.

        The reference's callbacks read their closure arrays live on every call
        (ClothSim.step rewrites `target` in place, apps/cloth.py:128; the
        sphere app rewrites its bases, apps/sphere.py:123-126). By default
        (`live_host_attrs=True`) every call does the same: numpy attributes of
        builtin terms are copied to the device again and traced callbacks with
        closure arrays are re-gathered. CUDA tensor attributes are read in
        place by the kernels (zero copies) — the fast way to mutate state.
        With `live_host_attrs=False` numpy attributes are snapshots taken at
        `add_term`, refreshed only by calling this method."""
        from . import jit

        for rec in self._terms:
            if only_host:
                if rec.groups is not None:
                    live = any(sub.dev_attrs for sub in rec.groups)
                elif rec.traced is not None:
                    live = bool(rec.dev_attrs)  # without closure arrays a traced callback is constants only
                else:
                    live = any(h is not None for h in rec.host_attrs)
                if not live:
                    continue
            if rec.groups is not None:  # VV: every valence group
                for sub in rec.groups:
                    tt = jit.trace_callback(rec.term, "VV", self.n, len(sub.index), sub.sel, index=sub.index)
                    if tt.source() != sub.traced.source():
                        raise ValueError("a traced callback changed its expression; register it again")
                    for dev, host in zip(sub.dev_attrs, tt.attrs):
                        dev.copy_(_torch().from_numpy(host))
                continue
            if rec.traced is not None:  # re-gather the closure arrays of a traced callback
                tt = jit.trace_callback(rec.term, rec.op.name, self.n, self._num_elements(rec.op),
                                        self._element_vertices(rec.op))
                if tt.source() != rec.traced.source():
                    raise ValueError("a traced callback changed its expression; register it again")
                for dev, host in zip(rec.dev_attrs, tt.attrs):
                    dev.copy_(_torch().from_numpy(host))
                continue
            for slot, host in enumerate(rec.host_attrs):
                if host is not None:
                    if isinstance(host, _torch().Tensor):  # float32 storage: a snapshotted CUDA tensor
                        rec.dev_attrs[slot].view(-1).copy_(host.reshape(-1))
                        continue
                    src = np.ascontiguousarray(np.asarray(host, dtype=np.float64)).reshape(-1)
                    rec.dev_attrs[slot].view(-1).copy_(_torch().from_numpy(src), non_blocking=False)

    def set_term_attr(self, term_id: int, name: str, value) -> None:
        """Rebind a term attribute (device tensor by reference or host array)."""
        rec = self._terms[term_id]
        slot = rec.term.attr_names.index(name)
        torch = _torch()
        setattr(rec.term, name, value)
        rec.host_attrs[slot] = None if isinstance(value, torch.Tensor) else value
        rec.dev_attrs[slot] = _as_device(value, torch, self._dev)
        _lib.check(self._lib.mg_problem_set_attr(self._h, rec.tid, slot, rec.dev_attrs[slot].data_ptr()))

    # properties --------------------------------------------------------------

    @property
    def num_dofs(self) -> int:
        return self._num_dofs

    @property
    def fixed_mask(self) -> np.ndarray:
        return self._fixed

    @property
    def free_dof_indices(self) -> np.ndarray:
        free_v = np.flatnonzero(~self._fixed)
        return (free_v[:, None] * self.n + np.arange(self.n)).ravel()

    @property
    def x(self) -> np.ndarray:
        return self.x_device.cpu().numpy()

    @x.setter
    def x(self, value) -> None:
        torch = _torch()
        if isinstance(value, torch.Tensor):
            src = value.detach().to(device=self._dev, dtype=self.dtype).reshape(-1)
        else:
            src = torch.from_numpy(np.ascontiguousarray(np.asarray(value, dtype=np.float64)).reshape(-1))
        if src.numel() != self._num_dofs:
            raise ValueError(f"x must have shape ({self._num_dofs},)")
        self.x_device.copy_(src)

    @property
    def grad(self) -> np.ndarray:
        return self.grad_device.cpu().numpy()

    # sparsity ------------------------------------------------------------------

    def precompute_sparsity(self) -> BlockSparseMatrix:
        """Device-built block pattern (ref problem.py:383-416)."""
        self._check_terms()
        torch = _torch()
        nnzb = ctypes.c_int64()
        _lib.check(self._lib.mg_precompute_sparsity(self._h, ctypes.byref(nnzb), _lib.stream_ptr()))
        nv = self.mesh.num_vertices
        ro = torch.empty(nv + 1, dtype=torch.int64, device=self._dev)
        ci = torch.empty(max(1, nnzb.value), dtype=torch.int64, device=self._dev)
        _lib.check(self._lib.mg_copy_pattern(self._h, ro.data_ptr(), ci.data_ptr(), _lib.stream_ptr()))
        n = self.n
        values = torch.zeros((nnzb.value, n, n), dtype=self.dtype, device=self._dev)
        self.hess = BlockSparseMatrix(n, nv, ro.cpu().numpy(), ci[: nnzb.value].cpu().numpy(), values, self)
        self.hess.row_offsets_device = ro
        self.hess.col_indices_device = ci[: nnzb.value]
        self._pattern_ready = True
        return self.hess

    # evaluation --------------------------------------------------------------

    def eval_terms(self, psd_floor: float | None = None, sync: bool = True) -> float:
        """Energy, gradient and (Hessian mode) the assembled Hessian at `x`
        (ref problem.py:504-549). With `sync=False` the call stays
        stream-ordered and returns NaN; read `energy_device` later."""
        t0 = time.perf_counter()
        self._check_terms()
        if psd_floor is not None and not self.with_hessian:
            raise ValueError("psd_floor requires a Hessian-mode problem")
        if psd_floor is not None and psd_floor <= 0:
            raise ValueError("floor must be positive")
        if self.with_hessian and not self._pattern_ready:
            self.precompute_sparsity()
        self._sync_attrs()
        hptr = self.hess.values_device.data_ptr() if (self.with_hessian and self.hess.nnz_blocks) else None
        _lib.check(self._lib.mg_eval(self._h, self.x_device.data_ptr(), int(psd_floor is not None),
                                     float(psd_floor or 0.0), self._energy_device.data_ptr(),
                                     self.grad_device.data_ptr(), hptr, _lib.stream_ptr()))
        total = float(self._energy_device.item()) if sync else float("nan")
        self.energy = total
        self.stats["eval_terms_calls"] += 1
        self.stats["eval_terms_ms"] += (time.perf_counter() - t0) * 1e3
        return total

    @property
    def energy_device(self):
        return self._energy_device

    def eval_energy_only(self, x_trial) -> float:
        """Total energy at a trial state; leaves the problem untouched
        (ref problem.py:551-576)."""
        t0 = time.perf_counter()
        self._check_terms()
        xd = self._vec_in(x_trial, "trial state must have shape ({},)")
        self._sync_attrs()
        out = _torch().empty(1, dtype=_torch().float64, device=self._dev)
        _lib.check(self._lib.mg_energy(self._h, xd.data_ptr(), out.data_ptr(), _lib.stream_ptr()))
        total = float(out.item())
        self.stats["energy_only_calls"] += 1
        self.stats["energy_only_ms"] += (time.perf_counter() - t0) * 1e3
        return total

    def _vec_in(self, v, msg):
        torch = _torch()
        if isinstance(v, torch.Tensor):
            if v.numel() != self._num_dofs:
                raise ValueError(msg.format(self._num_dofs))
            return v.detach().to(device=self._dev, dtype=self.dtype).contiguous().reshape(-1)
        a = np.asarray(v, dtype=np.float64)
        if a.shape != (self._num_dofs,):
            raise ValueError(msg.format(self._num_dofs))
        return torch.from_numpy(np.ascontiguousarray(a)).to(self._dev).to(self.dtype)

    def hvp(self, x, v, psd_floor: float | None = None, out=None):
        """Matrix-free Hessian-vector product (ref problem.py:578-617).
        numpy in -> numpy out; CUDA tensors in -> CUDA tensor out."""
        t0 = time.perf_counter()
        torch = _torch()
        self._check_terms()
        if psd_floor is not None and psd_floor <= 0:
            raise ValueError("floor must be positive")
        host = not isinstance(v, torch.Tensor)
        msg = "x and v must have shape ({},)"
        xd = self._vec_in(x, msg)
        vd = self._vec_in(v, msg)
        self._sync_attrs()
        if out is not None and not (isinstance(out, torch.Tensor) and out.dtype == self.dtype
                                    and out.device == vd.device and out.is_contiguous()
                                    and out.numel() == self._num_dofs):
            raise ValueError(f"out must be a contiguous {self.dtype} CUDA tensor of {self._num_dofs} entries")
        y = out if out is not None else torch.empty(self._num_dofs, dtype=self.dtype, device=self._dev)
        _lib.check(self._lib.mg_hvp(self._h, xd.data_ptr(), vd.data_ptr(), int(psd_floor is not None),
                                    float(psd_floor or 0.0), y.data_ptr(), _lib.stream_ptr()))
        res = y.cpu().numpy() if host else y
        self.stats["hvp_calls"] += 1
        self.stats["hvp_ms"] += (time.perf_counter() - t0) * 1e3
        return res

    def launch_count(self) -> int:
        c = ctypes.c_int()
        _lib.check(self._lib.mg_last_launch_count(self._h, ctypes.byref(c)))
        return c.value

    def set_kernel_timing(self, enable: bool = True) -> None:
        """Record device time of the main kernel of every call (benchmarks)."""
        _lib.check(self._lib.mg_problem_set_timing(self._h, int(bool(enable))))

    def kernel_time(self):
        """(total ms, launches) of the main kernel since the last query; synchronizes."""
        t, c = ctypes.c_double(), ctypes.c_int()
        _lib.check(self._lib.mg_problem_kernel_time(self._h, ctypes.byref(t), ctypes.byref(c)))
        return t.value, c.value

    def exact_runs(self) -> int:
        """Calls whose exact re-run executed (fast row kernels fall back on
        non-finite lanes); synchronizes."""
        n = ctypes.c_int64()
        _lib.check(self._lib.mg_problem_exact_runs(self._h, ctypes.byref(n)))
        return n.value

    def patch_stats(self) -> dict:
        arr = (ctypes.c_int64 * 4)()
        _lib.check(self._lib.mg_problem_patch_stats(self._h, arr))
        return {"patches": arr[0], "rows": arr[1], "ribbon_vertices": arr[2], "recomputed_elements": arr[3]}

    # export ------------------------------------------------------------------

    def export_hessian(self, path) -> None:
        if self.hess is None or not self._pattern_ready:
            raise ValueError("no Hessian assembled")
        self.hess.write_matrix_market(path)

    def export_gradient(self, path) -> None:
        with open(path, "w") as fh:
            fh.writelines(f"{g:.17g}\n" for g in self.grad.tolist())
