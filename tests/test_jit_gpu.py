"""Traced user callbacks (paper_2509_00406_b200.jit): the reference callback
protocol, run through tracer -> CUDA codegen -> nvcc -> driver-API launch,
against the golden vectors of the unmodified reference (<= 1e-10, patterns
bit-exact). Each builtin term is registered as a plain Python function (its
body is the reference app's formula), so nothing takes the builtin path."""

import numpy as np
import pytest

from engine_util import engine_mesh
from golden_util import FLOOR, build_terms, cases, load, rel, rel_scalar, states

pytestmark = pytest.mark.gpu

_KIND = {"V": "VERTEX", "EV": "EDGE", "FV": "FACE"}
CASES = [c for c in cases() if c not in ("cloth16_asis",)]


def traced_problem(d):
    import paper_2509_00406_b200 as mg

    p = mg.Problem(engine_mesh(d), int(d["n"]), with_hessian=bool(d["with_hessian"]),
                   fixed_vertices=d["fixed"].tolist())
    for op, term in build_terms(d):
        p.add_term(getattr(mg.Element, _KIND[op]), getattr(mg.Op, op),
                   lambda h, nb, x, _t=term: _t(h, nb, x))  # a plain callback, not a builtin
    return p


@pytest.mark.parametrize("name", CASES)
def test_traced_callbacks_match_reference(name):
    d = load(name)
    p = traced_problem(d)
    assert all(r.traced is not None for r in p._terms)
    if p.with_hessian:
        h = p.precompute_sparsity()
        assert np.array_equal(h.row_offsets, d["row_offsets"])
        assert np.array_equal(h.col_indices, d["col_indices"])
    for s in states(d):
        x = d[f"s{s}_x"]
        p.x = x
        e = p.eval_terms()
        assert rel_scalar(e, d[f"s{s}_energy"]) <= 1e-10
        assert rel(p.grad, d[f"s{s}_grad"]) <= 1e-10
        if f"s{s}_hess" in d:
            assert rel(p.hess.values, d[f"s{s}_hess"]) <= 1e-10
        if f"s{s}_psd_hess" in d:
            e = p.eval_terms(psd_floor=FLOOR)
            assert rel_scalar(e, d[f"s{s}_psd_energy"]) <= 1e-10
            assert rel(p.hess.values, d[f"s{s}_psd_hess"]) <= 1e-10
        assert rel_scalar(p.eval_energy_only(x), d[f"s{s}_energy_only"]) <= 1e-10
        if f"s{s}_v0" in d:
            ref = d[f"s{s}_hvp0"]
            got = p.hvp(x, d[f"s{s}_v0"])
            if np.isfinite(ref).all():
                assert rel(got, ref) <= 1e-10
            if f"s{s}_hvp_psd0" in d and np.isfinite(d[f"s{s}_hvp_psd0"]).all():
                assert rel(p.hvp(x, d[f"s{s}_v0"], psd_floor=FLOOR), d[f"s{s}_hvp_psd0"]) <= 1e-10


def test_traced_closure_refresh():
    """A closure array mutated in place (ClothSim.step's target rewrite,
    apps/cloth.py:128) is re-read after refresh_attrs()."""
    import paper_2509_00406_b200 as mg

    d = load("cloth8")
    target = d["a_target"].copy()
    masses = d["a_masses"]

    def inertia(v, nbrs, x):
        dd = x[v] - target[v.index]
        return 0.5 * masses[v.index] * dd.norm2()

    p = mg.Problem(engine_mesh(d), 3)
    p.add_term(mg.Element.VERTEX, mg.Op.V, inertia)
    x = d["s0_x"]
    p.x = x
    e0 = p.eval_terms()
    target += 0.5
    p.refresh_attrs()
    e1 = p.eval_terms()
    dx = x.reshape(-1, 3) - target
    assert abs(e1 - 0.5 * np.sum(masses[:, None] * dx * dx)) <= 1e-12 * abs(e1)
    assert e1 != e0


@pytest.mark.parametrize("name", CASES)
def test_traced_deterministic_gather(name):
    """Deterministic mode (the default) assembles traced terms through
    per-element scratch + a fixed-order gather: repeat calls are bitwise equal
    and agree with the atomic assembly."""
    d = load(name)
    p = traced_problem(d)
    assert p.accumulation == "deterministic"
    s = states(d)[-1]
    x = d[f"s{s}_x"]
    v = np.sin(np.arange(p.num_dofs))

    def run(q):
        q.x = x
        e = q.eval_terms()
        return e, q.grad.copy(), (q.hess.values.copy() if q.with_hessian else None), q.hvp(x, v)

    a, b = run(p), run(p)
    for u, w in zip(a, b):
        assert u is None or np.array_equal(u, w, equal_nan=True)
    import paper_2509_00406_b200 as mg

    pa = mg.Problem(engine_mesh(d), int(d["n"]), with_hessian=bool(d["with_hessian"]),
                    fixed_vertices=d["fixed"].tolist(), accumulation="atomic")
    for op, term in build_terms(d):
        pa.add_term(getattr(mg.Element, _KIND[op]), getattr(mg.Op, op), lambda h, nb, xx, _t=term: _t(h, nb, xx))
    c = run(pa)
    if np.isfinite(a[0]):
        assert rel_scalar(c[0], a[0]) <= 1e-12
    for u, w in zip(a[1:], c[1:]):
        if u is not None and np.isfinite(u).all():
            assert rel(w, u) <= 1e-12
