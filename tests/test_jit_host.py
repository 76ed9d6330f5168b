"""Tracer / code generation of arbitrary callbacks (CPU side): the recorded
SSA follows the callback's operation order, closure gathers become attribute
streams, constants are exact, unsupported constructs fail loudly, and the
generated functor compiles for sm_100a with nvcc."""

import numpy as np
import pytest

from paper_2509_00406_b200 import jit
from paper_2509_00406_b200.active import SmallMatrix, log, positive_guard, sqrt


def spring(l2, coef):
    def fn(edge, verts, x):
        d = x[verts[0]] - x[verts[1]]
        s = d.norm2() / l2[edge.index] - 1.0
        return coef * l2[edge.index] * (s * s)
    return fn


def test_trace_records_operations_in_order():
    l2 = np.linspace(1.0, 2.0, 7)
    tt = jit.trace_callback(spring(l2, 0.5), "EV", 3, 7, sel=np.zeros((7, 2), np.int64))
    body = "\n".join(tt.body)
    assert body.index("X[0][0] - X[1][0]") < body.index(" / A[0][e]") < body.index("A[1][e] * ")
    # coef * l2[edge.index] is numpy arithmetic in the callback: one precomputed stream, as in the reference
    assert len(tt.attrs) == 2 and np.array_equal(tt.attrs[0], l2) and np.array_equal(tt.attrs[1], 0.5 * l2)
    assert "0x1.0000000000000p+0" in body  # the exact literal 1.0


def test_vertex_batches_index_slot_vertices():
    base = np.arange(30.0).reshape(10, 3)
    sel = np.array([[1, 2, 3], [4, 5, 6]])

    def fn(face, verts, x):
        return x[verts[0]][0] * base[verts[2].index][:, 1]

    tt = jit.trace_callback(fn, "FV", 2, 2, sel=sel)
    assert np.array_equal(tt.attrs[0], base[sel[:, 2], 1])


def test_branching_and_float_conversion_fail():
    with pytest.raises(TypeError):
        jit.trace_callback(lambda v, n, x: x[v][0] if x[v][0] > 0 else x[v][1], "V", 2, 3)
    with pytest.raises(TypeError):
        jit.trace_callback(lambda v, n, x: float(x[v][0]), "V", 2, 3)
    with pytest.raises(TypeError):
        jit.trace_callback(lambda v, n, x: x[v][0] ** 0.5, "V", 2, 3)


def test_generated_functor_compiles():
    rest_inv = np.random.default_rng(0).random((5, 2, 2))
    areas = np.ones(5)

    def dirichlet(face, verts, x):
        a, b, c = x[verts[0]], x[verts[1]], x[verts[2]]
        d1, d2 = b - a, c - a
        j = SmallMatrix([[d1[0], d2[0]], [d1[1], d2[1]]]) @ rest_inv[face.index]
        det = positive_guard(j.det())
        fro = j.frobenius2()
        return areas[face.index] * (fro + fro / (det * det)) + log(sqrt(det)) * 0.0 + abs(a[0]) ** 2

    tt = jit.trace_callback(dirichlet, "FV", 2, 5, sel=np.zeros((5, 3), np.int64))
    assert len(tt.attrs) == 5  # four rest_inv entries + areas (views of one array dedupe)
    image = jit.compile_term(tt)
    assert image[:4] == b"\x7fELF"


def test_vv_trace_uses_center_and_ring_slots():
    """VV (ref problem.py:340-353, 443-448): the handle is the center (slot 0)
    and carries the centers' ids; nbrs are the ring slots 1..d."""
    w = np.arange(10.0)
    sel = np.array([[3, 1, 4, 5], [7, 2, 6, 8]])
    ids = sel[:, 0]

    def ring(vertex, nbrs, x):
        c = x[vertex]
        total = 0.0
        for nb in nbrs:
            total = total + (c - x[nb]).norm2() * w[vertex.index]
        return total

    tt = jit.trace_callback(ring, "VV", 3, 2, sel, index=ids)
    assert tt.P == 4
    body = "\n".join(tt.body)
    assert "X[0][0] - X[3][0]" in body and "X[4]" not in body
    # each closure gather is one per-element stream of the group's centers
    assert tt.attrs and all(np.array_equal(a, w[ids]) for a in tt.attrs)
    with pytest.raises(ValueError, match="neighbourhoods"):
        jit.trace_callback(ring, "VV", 3, 2, None)


def _ev(fn, n=3, M=4):
    return jit.trace_callback(fn, "EV", n, M, sel=np.zeros((M, 2), np.int64))


def test_radial_form_proves_spring_and_edge_length():
    """radial_form finds r = |x_0 - x_1|^2 in the trace and returns the
    operations after it (the row module's phi(r))."""
    rf = jit.radial_form(_ev(spring(np.linspace(1.0, 2.0, 4), 0.5)))
    assert rf is not None
    r, lines = rf
    assert lines[0] == f"auto {r} = R;" and not any("X[" in ln for ln in lines)
    rf = jit.radial_form(_ev(lambda e, v, x: (x[v[1]] - x[v[0]]).norm2(), n=2))  # the energy is r itself
    assert rf is not None and len(rf[1]) == 1
    rf = jit.radial_form(_ev(lambda e, v, x: sqrt((x[v[0]] - x[v[1]]).dot(x[v[0]] - x[v[1]])) * 2.0))
    assert rf is not None  # dot(d, d) of two equal differences, then sqrt


@pytest.mark.parametrize("fn", [
    lambda e, v, x: (x[v[0]] - x[v[1]])[0] * (x[v[0]] - x[v[1]])[0],        # one component only
    lambda e, v, x: (x[v[0]] - x[v[1]]).norm2() + x[v[0]][0],                # a direct use of x
    lambda e, v, x: (x[v[0]] - x[v[1]]).dot(x[v[1]] - x[v[0]]),              # -|d|^2: mixed signs
    lambda e, v, x: (x[v[0]] - x[v[1]]).norm2() * (x[v[0]] - x[v[1]])[1],    # d beyond the norm
    lambda e, v, x: (x[v[0]] - x[v[1]]).norm2() + (x[v[0]] - x[v[1]]).norm2(),  # two r symbols
    lambda e, v, x: (x[v[0]] + x[v[1]]).norm2(),                              # not a difference
])
def test_radial_form_rejects_non_radial(fn):
    assert jit.radial_form(_ev(fn)) is None


def test_rows_source_needs_every_edge_term_radial():
    rad = _ev(spring(np.linspace(1.0, 2.0, 4), 0.5))
    lin = _ev(lambda e, v, x: (x[v[0]] - x[v[1]])[0] * 1.0)
    vt = jit.trace_callback(lambda h, nb, x: 0.5 * x[h].norm2(), "V", 3, 5)
    src = jit.rows_source([vt, rad], 3)
    assert src is not None and "MG_ROWS_JIT_INSTANTIATE(Pol, 3)" in src and "A[" not in src
    assert jit.rows_source([vt, rad, lin], 3) is None
    assert jit.rows_source([vt], 3) is None  # no edge term: nothing for the edge row kernel


def test_generated_row_module_compiles():
    import shutil
    if shutil.which("nvcc") is None:
        pytest.skip("nvcc not available")
    rad = _ev(spring(np.linspace(1.0, 2.0, 4), 0.5))
    vt = jit.trace_callback(lambda h, nb, x: 0.5 * x[h].norm2(), "V", 3, 5)
    assert len(jit.compile_rows([vt, rad], 3)) > 1000
