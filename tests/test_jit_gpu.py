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


@pytest.mark.parametrize("path", ["element", "patch", "rows"])
@pytest.mark.parametrize("name", CASES)
def test_traced_callbacks_match_reference(name, path, monkeypatch):
    """The three engine paths for traced terms: element-parallel kernels (one
    module per term, fixed-order gather), the problem's generated patch
    module (jit_patch.cuh) and, when the tracer proves every edge callback
    radial, the generated edge row module (jit_rows.cuh, the patch module as
    its exact re-run); the last two forced here at golden sizes by
    MG_JIT_PATCH_MIN=0."""
    monkeypatch.setenv("MG_JIT_PATCH_MIN", "0" if path != "element" else str(1 << 62))
    monkeypatch.setenv("MG_JIT_ROWS", "1" if path == "rows" else "0")
    d = load(name)
    if path == "rows" and not {op for op, _ in build_terms(d)} <= {"V", "EV"}:
        pytest.skip("face terms: no edge row module")
    p = traced_problem(d)
    assert all(r.traced is not None for r in p._terms)
    if p.with_hessian:
        h = p.precompute_sparsity()
        assert np.array_equal(h.row_offsets, d["row_offsets"])
        assert np.array_equal(h.col_indices, d["col_indices"])
    else:
        p.eval_terms()
    assert p.patch_module == (path != "element")
    if path == "rows":
        assert p.row_module, "the tracer should prove these edge callbacks radial"
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


@pytest.mark.parametrize("traced", [True, False])
def test_numpy_closure_mutated_in_place(traced):
    """A numpy closure array mutated in place between calls (ClothSim.step's
    target rewrite, apps/cloth.py:128) is seen by the next eval_terms, as in
    the reference, for traced callbacks and builtin terms alike. With
    live_host_attrs=False the arrays are snapshots until refresh_attrs()."""
    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200 import terms as T

    d = load("cloth8")
    masses = d["a_masses"]

    def expect(x, target):
        dx = x.reshape(-1, 3) - target
        return 0.5 * np.sum(masses[:, None] * dx * dx)

    for live in (True, False):
        target = d["a_target"].copy()

        def inertia(v, nbrs, x):
            dd = x[v] - target[v.index]
            return 0.5 * masses[v.index] * dd.norm2()

        p = mg.Problem(engine_mesh(d), 3, live_host_attrs=live)
        p.add_term(mg.Element.VERTEX, mg.Op.V, inertia if traced else T.Inertia(masses, target))
        x = d["s0_x"]
        p.x = x
        e0 = p.eval_terms()
        assert abs(e0 - expect(x, target)) <= 1e-12 * abs(e0)
        target += 0.5  # in place, like target[:] = ... in the reference app
        e1 = p.eval_terms()
        if live:
            assert abs(e1 - expect(x, target)) <= 1e-12 * abs(e1) and e1 != e0
            assert abs(p.eval_energy_only(x) - e1) <= 1e-12 * abs(e1)
        else:
            assert e1 == e0  # snapshot semantics
            p.refresh_attrs()
            assert abs(p.eval_terms() - expect(x, target)) <= 1e-12 * abs(e1)


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
