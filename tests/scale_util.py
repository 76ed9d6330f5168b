"""Sampled-row parity at the BASELINE sizes.

The CPU oracle cannot evaluate a 2048^2 cloth or a 21M-face icosphere in
seconds per call, but it does not need to: every gradient entry, Hessian
row and HVP row of vertex r is a sum over the elements incident to r only
(the reference scatters an element's blocks inside its own vertices,
problem.py:535-544, 606-614). So the oracle evaluates exactly the elements
incident to a sample of rows (global element ids, so closure arrays index
the same way) and those rows are complete and exactly comparable; the
energy is compared against a full-mesh oracle energy probe, and the block
pattern against a full-mesh restatement of problem.py:383-402.
"""

from __future__ import annotations

import numpy as np

from oracle.engine import OracleProblem, default_workers, sparsity_pattern


def op_selection(op, nv, faces, edges):
    if op == "FV":
        return np.asarray(faces, dtype=np.int64)
    if op == "EV":
        return np.asarray(edges, dtype=np.int64)
    return np.arange(nv, dtype=np.int64)[:, None]


def sample_rows(nv, rng, k, extra=()):
    """k random rows plus the given ones (pins, their neighbours, corners)."""
    rows = rng.choice(nv, size=min(k, nv), replace=False)
    return np.unique(np.concatenate([rows, np.asarray(extra, dtype=np.int64)]))


def block_index(row_offsets, rows):
    """Positions of the blocks of `rows` (in order) in a CSR values array."""
    lo, hi = row_offsets[rows], row_offsets[rows + 1]
    lens = hi - lo
    start = np.repeat(lo - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    return start + np.arange(int(lens.sum()))


def dof_index(rows, n):
    return (np.asarray(rows)[:, None] * n + np.arange(n)).ravel()


class SampledOracle:
    """OracleProblem restricted to the elements incident to `rows`."""

    def __init__(self, nv, faces, edges, n, terms, rows, fixed=(), with_hessian=True):
        self.nv, self.n, self.rows = nv, n, np.asarray(rows, dtype=np.int64)
        mask = np.zeros(nv, dtype=bool)
        mask[self.rows] = True
        ids = [np.flatnonzero(mask[op_selection(op, nv, faces, edges)].any(axis=1)) for op, _ in terms]
        self.elements = sum(len(i) for i in ids)
        self.o = OracleProblem(nv, faces, edges, n, terms, with_hessian=with_hessian, fixed_vertices=fixed,
                               workers=default_workers(), accumulation="atomic", element_ids=ids)
        self.dofs = dof_index(self.rows, n)
        if with_hessian:
            self.bidx = block_index(self.o.row_offsets, self.rows)

    def eval_rows(self, x, psd_floor=None):
        """(grad rows, Hessian blocks of the rows, their column ids)."""
        _, g, h = self.o.eval_terms(x, psd_floor=psd_floor)
        if h is None:
            return g[self.dofs], None, None
        return g[self.dofs], h[self.bidx], self.o.col_indices[self.bidx]

    def hvp_rows(self, x, v, psd_floor=None):
        return self.o.hvp(x, v, psd_floor=psd_floor)[self.dofs]


def full_energy(nv, faces, edges, n, terms, x, fixed=()):
    """Whole-mesh energy probe (problem.py:551-576), all host threads."""
    o = OracleProblem(nv, faces, edges, n, terms, with_hessian=False, fixed_vertices=fixed,
                      workers=default_workers(), accumulation="atomic")
    return o.eval_energy_only(x)


def full_pattern(nv, faces, edges, terms, fixed=()):
    fx = None
    if len(fixed):
        fx = np.zeros(nv, dtype=bool)
        fx[list(fixed)] = True
    return sparsity_pattern(nv, [op_selection(op, nv, faces, edges) for op, _ in terms], fx)


def device_rows(p, rows, hidx=None):
    """Gradient rows, and (Hessian mode) the rows' blocks + columns, read
    from the engine's device buffers without copying the whole Hessian."""
    import torch

    dofs = torch.from_numpy(dof_index(rows, p.n)).to(p.grad_device.device)
    g = p.grad_device[dofs].cpu().numpy()
    if hidx is None:
        return g, None, None
    vals = p.hess.values_device[torch.from_numpy(hidx).to(p.grad_device.device)].cpu().numpy()
    return g, vals, p.hess.col_indices[hidx]
