"""VV (vertex one-ring) callback terms against the unmodified reference
(tests/golden/make_golden_vv.py): the callback is traced per valence group and
assembled element-parallel (deterministic scratch + gather). Pattern bit-exact
(distance-2 couplings through the center), values <= 1e-10."""

import numpy as np
import pytest

from golden_util import GOLDEN, rel, rel_scalar

pytestmark = pytest.mark.gpu

FLOOR = 1e-9


def make_ring_energy(w):
    from paper_2509_00406_b200.active import sqrt

    def ring_energy(vertex, nbrs, x):  # verbatim from make_golden_vv.py
        c = x[vertex]
        total = 0.0
        for nb in nbrs:
            d = c - x[nb]
            r = sqrt(d.norm2() + 0.01)
            total = total + (r - 0.3) * (r - 0.3) * w[vertex.index]
        return total

    return ring_energy


def vv_problem(d, **kw):
    import paper_2509_00406_b200 as mg

    mesh = mg.Mesh(d["positions"], d["faces"])
    p = mg.Problem(mesh, int(d["n"]), fixed_vertices=d["fixed"].tolist(), **kw)
    p.add_term(mg.Element.VERTEX, mg.Op.VV, make_ring_energy(d["w"]))
    return p


def test_vv_matches_reference():
    d = np.load(GOLDEN / "vv_grid5.npz")
    p = vv_problem(d)
    h = p.precompute_sparsity()
    assert np.array_equal(h.row_offsets, d["row_offsets"])
    assert np.array_equal(h.col_indices, d["col_indices"])
    for s in range(2):
        x = d[f"s{s}_x"]
        p.x = x
        assert rel_scalar(p.eval_terms(), d[f"s{s}_energy"]) <= 1e-10
        assert rel(p.grad, d[f"s{s}_grad"]) <= 1e-10
        assert rel(p.hess.values, d[f"s{s}_hess"]) <= 1e-10
        assert rel_scalar(p.eval_terms(psd_floor=FLOOR), d[f"s{s}_psd_energy"]) <= 1e-10
        assert rel(p.hess.values, d[f"s{s}_psd_hess"]) <= 1e-10
        assert rel_scalar(p.eval_energy_only(x), d[f"s{s}_energy_only"]) <= 1e-10
        assert rel(p.hvp(x, d[f"s{s}_v"]), d[f"s{s}_hvp"]) <= 1e-10
        assert rel(p.hvp(x, d[f"s{s}_v"], psd_floor=FLOOR), d[f"s{s}_hvp_psd"]) <= 1e-10


def test_vv_deterministic_and_atomic_agree():
    d = np.load(GOLDEN / "vv_grid5.npz")
    x = d["s1_x"]
    runs = []
    for acc in ("deterministic", "deterministic", "atomic"):
        p = vv_problem(d, accumulation=acc)
        p.x = x
        e = p.eval_terms()
        runs.append((e, p.grad.copy(), p.hess.values.copy()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1]) and np.array_equal(runs[0][2], runs[1][2])
    assert runs[2][0] == pytest.approx(runs[0][0], rel=1e-12)
    assert rel(runs[2][2], runs[0][2]) <= 1e-12
