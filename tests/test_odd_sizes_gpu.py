"""Row counts that are not multiples of the 64-row blocks, fewer row blocks
than resident CTAs, and rectangular / Morton-ordered meshes: the staged
(TMA-ring, persistent) edge row kernels, the CTA face-list kernels and the
energy probe against the CPU oracle (pinned to the reference's golden
vectors, tests/test_oracle_golden.py) on the same inputs — energy, gradient,
Hessian (plain and clamped), HVP (plain and clamped), energy probe, pattern
bit-exact."""

import numpy as np
import pytest

from golden_util import FLOOR, rel, rel_scalar

pytestmark = pytest.mark.gpu


def _check(p, op, x, v, with_h):
    p.x = x
    e = p.eval_terms()
    oe, og, oh = op.eval_terms(x)
    assert rel_scalar(e, oe) <= 1e-10
    assert rel(p.grad, og) <= 1e-10
    if with_h:
        assert rel(p.hess.values, oh) <= 1e-10
        e = p.eval_terms(psd_floor=FLOOR)
        oe, og, oh = op.eval_terms(x, psd_floor=FLOOR)
        assert rel_scalar(e, oe) <= 1e-10 and rel(p.hess.values, oh) <= 1e-10
    assert rel(p.hvp(x, v), op.hvp(x, v)) <= 1e-10
    assert rel(p.hvp(x, v, psd_floor=FLOOR), op.hvp(x, v, psd_floor=FLOOR)) <= 1e-10
    assert rel_scalar(p.eval_energy_only(x), op.eval_energy_only(x)) <= 1e-10
    assert p.exact_runs() == 0


@pytest.mark.parametrize("nx,ny", [(7, 5), (33, 17), (97, 61)])
def test_cloth_rectangles(nx, ny):
    """Cloth on nx x ny grids (V = 35 .. 5917 rows, none a multiple of 64)."""
    from oracle import OracleProblem

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.mesh import _host_edges
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    ii, jj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    pos = np.stack([ii.ravel() / (nx - 1), jj.ravel() / (nx - 1), np.zeros(nx * ny)], axis=1)
    j, i = np.meshgrid(np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    v00 = (j * nx + i).ravel()
    faces = np.empty((2 * (nx - 1) * (ny - 1), 3), np.int64)
    faces[0::2] = np.stack([v00, v00 + 1, v00 + nx + 1], 1)
    faces[1::2] = np.stack([v00, v00 + nx + 1, v00 + nx], 1)
    rng = np.random.default_rng(nx * ny)
    nv = len(pos)
    edges = _host_edges(faces, None, nv)
    d = pos[edges[:, 1]] - pos[edges[:, 0]]
    masses = rng.uniform(0.5, 1.5, nv) / nv
    target = pos + 0.01 / nx * rng.normal(size=pos.shape)
    terms = [("V", Inertia(masses, target)), ("EV", Spring(np.einsum("ij,ij->i", d, d), 0.5)),
             ("V", Gravity(masses, np.array([0.0, -9.8, 0.0]), 1e-4))]
    pins = [0, nx - 1]
    mesh = mg.Mesh(pos, faces)
    p = mg.Problem(mesh, 3, fixed_vertices=pins)
    for op, t in terms:
        p.add_term(getattr(mg.Element, "VERTEX" if op == "V" else "EDGE"), getattr(mg.Op, op), t)
    h = p.precompute_sparsity()
    o = OracleProblem(nv, faces, edges, 3, terms, with_hessian=True, fixed_vertices=pins, workers=1,
                      accumulation="deterministic")
    o.precompute_sparsity()
    assert np.array_equal(h.row_offsets, o.row_offsets) and np.array_equal(h.col_indices, o.col_indices)
    x = (pos + 0.01 / nx * rng.normal(size=pos.shape)).ravel()
    _check(p, o, x, rng.normal(size=x.size), True)


@pytest.mark.parametrize("sub", [1, 3])
def test_icosphere_edges_and_faces(sub):
    """Morton-ordered rows (icosphere: V = 42, 642): smoothing on the edge row
    kernel, symmetric Dirichlet on the face kernels (punctured sphere)."""
    from oracle import OracleProblem

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import rest_geometry
    from paper_2509_00406_b200.mesh import _host_edges
    from paper_2509_00406_b200.terms import EdgeLength, SymDirichlet

    rng = np.random.default_rng(sub)
    pos, faces = mg.icosphere_arrays(sub)
    nv = len(pos)
    edges = _host_edges(faces, None, nv)
    p = mg.Problem(mg.Mesh(pos, faces), 3, fixed_vertices=[1])
    p.add_term(mg.Element.EDGE, mg.Op.EV, EdgeLength())
    p.precompute_sparsity()
    o = OracleProblem(nv, faces, edges, 3, [("EV", EdgeLength())], with_hessian=True, fixed_vertices=[1],
                      workers=1, accumulation="deterministic")
    x = (pos + 0.01 * rng.normal(size=pos.shape)).ravel()
    _check(p, o, x, rng.normal(size=x.size), True)

    pos, faces, uv = mg.punctured_icosphere_arrays(sub + 1)
    mesh = mg.Mesh(pos, faces)
    ri, ar = rest_geometry(mesh)
    term = SymDirichlet(np.ascontiguousarray(ri).reshape(-1, 4), ar)
    p = mg.Problem(mesh, 2)
    p.add_term(mg.Element.FACE, mg.Op.FV, term)
    p.precompute_sparsity()
    o = OracleProblem(len(pos), faces, _host_edges(faces, None, len(pos)), 2, [("FV", term)], with_hessian=True,
                      workers=1, accumulation="deterministic")
    x = uv.ravel() * (1.0 + 0.01 * rng.normal(size=uv.size))
    _check(p, o, x, rng.normal(size=x.size), True)
