"""Parity against the pinned CPU oracle AT the BASELINE sizes.

North-star acceptance: on a >= 10M-face mesh, gradient + sparse Hessian
assembly and HVP each within tolerance of the CPU reference, with the block
pattern bit-exact. Every config is run at its BASELINE size:

  config 2   cloth 2048^2 (8.4M faces), default pins     E, g, H, H(psd), HVP, HVP(psd)
  config 2'  cloth 2240^2 (10.0M faces), default pins    same
  config 3   symmetric Dirichlet, punctured icosphere(10) (21.0M faces)   same
  config 4b  sphere barrier+stretch, icosphere(10) (21.0M faces)          E, g, HVP, HVP(psd)
  config 4a  smoothing edge term, icosphere(10) (31.5M edges)             E, g, HVP

Method (tests/scale_util.py): the block pattern is compared bit-for-bit
against the oracle's pair-key restatement of problem.py:383-402 on the whole
mesh; the energy (eval_terms and eval_energy_only) against the oracle's
whole-mesh energy probe; gradient entries, Hessian rows (their column ids
bit-exact, values <= 1e-10) and HVP rows against the oracle evaluated on
exactly the elements incident to ~20k sampled rows (random rows plus the
pinned vertices' neighbourhoods and the mesh corners). A row's values depend
only on its incident elements, so the sampled comparison is exact, not an
approximation. Tolerance: max|diff| / max|ref| over the compared entries
<= 1e-10 (fp64, BASELINE north_star).
"""

import gc

import numpy as np
import pytest

from golden_util import FLOOR, rel, rel_scalar
from scale_util import SampledOracle, block_index, device_rows, dof_index, full_energy, full_pattern, sample_rows

pytestmark = pytest.mark.gpu

TOL = 1e-10
SAMPLE = 20000


def _free():
    import torch

    gc.collect()
    torch.cuda.empty_cache()


def _check_pattern(p, nv, faces, edges, terms, fixed=()):
    ro, ci = full_pattern(nv, faces, edges, terms, fixed)
    assert np.array_equal(p.hess.row_offsets, ro)
    assert np.array_equal(p.hess.col_indices, ci)


def _check_eval(p, so, x, floors):
    hidx = block_index(p.hess.row_offsets, so.rows) if p.with_hessian else None
    for floor in floors:
        p.eval_terms(psd_floor=floor)
        g, h, cols = device_rows(p, so.rows, hidx)
        og, oh, ocols = so.eval_rows(x, psd_floor=floor)
        assert rel(g, og) <= TOL, (floor, rel(g, og))
        if oh is not None:
            assert np.array_equal(cols, ocols)
            assert rel(h, oh) <= TOL, (floor, rel(h, oh))


def _check_hvp(p, so, x, v, floors):
    import torch

    xd = torch.from_numpy(x).cuda()
    vd = torch.from_numpy(v).cuda()
    dofs = torch.from_numpy(dof_index(so.rows, p.n)).cuda()
    for floor in floors:
        y = p.hvp(xd, vd, psd_floor=floor)[dofs].cpu().numpy()
        ref = so.hvp_rows(x, v, psd_floor=floor)
        assert rel(y, ref) <= TOL, (floor, rel(y, ref))


def _check_energy(p, e_ref, x):
    e = p.eval_terms()
    assert rel_scalar(e, e_ref) <= TOL, (e, e_ref)
    assert rel_scalar(p.eval_energy_only(x), e_ref) <= TOL


@pytest.mark.parametrize("n", [2048, 2240])
def test_cloth_matches_oracle_at_baseline_size(n):
    """Configs 2 and 2': the cloth Newton-step energy on the full grid."""
    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import ClothConfig, default_pins, lumped_masses, rest_lengths2
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    pos, faces = mg.grid_arrays(n, 1.0 / (n - 1))
    mesh = mg.Mesh(pos, faces)
    edges = mesh.edges
    nv = len(pos)
    rng = np.random.default_rng(0)
    sig = 0.01 / (n - 1)
    target = pos + sig * rng.normal(size=pos.shape)
    x = (pos + sig * rng.normal(size=pos.shape)).ravel()
    v = np.random.default_rng(1).normal(size=x.size)
    cfg = ClothConfig(grid_n=n, spacing=1.0 / (n - 1))
    h2 = cfg.h * cfg.h
    masses = lumped_masses(mesh, cfg.mass_density)
    terms = [("V", Inertia(masses, target)), ("EV", Spring(rest_lengths2(mesh), 0.5 * cfg.k * h2)),
             ("V", Gravity(masses, np.asarray(cfg.gravity, dtype=np.float64), h2))]
    pins = default_pins(n)
    p = mg.Problem(mesh, 3, fixed_vertices=pins)
    for op, t in terms:
        p.add_term(getattr(mg.Element, {"V": "VERTEX", "EV": "EDGE"}[op]), getattr(mg.Op, op), t)
    p.precompute_sparsity()
    _check_pattern(p, nv, faces, edges, terms, pins)
    p.x = x
    _check_energy(p, full_energy(nv, faces, edges, 3, terms, x, pins), x)
    # rows around both pins, the four corners and the first/last grid lines
    ring = lambda c: [c + dj * n + di for dj in (-1, 0, 1) for di in (-1, 0, 1) if 0 <= c + dj * n + di < nv]
    extra = sum((ring(c) for c in (0, n - 1, nv - n, nv - 1) + tuple(pins)), [])
    so = SampledOracle(nv, faces, edges, 3, terms, sample_rows(nv, rng, SAMPLE, extra), fixed=pins)
    _check_eval(p, so, x, (None, FLOOR))
    _check_hvp(p, so, x, v, (None, FLOOR))
    assert p.exact_runs() == 0  # the fast row / tile kernels carried every call
    del p
    _free()


@pytest.fixture(scope="module")
def ico10():
    import paper_2509_00406_b200 as mg

    return mg.icosphere_arrays(10)


def test_dirichlet_matches_oracle_at_baseline_size():
    """Config 3: symmetric Dirichlet on the punctured icosphere(10), x = the
    stereographic UV (all det J > 0)."""
    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import rest_geometry
    from paper_2509_00406_b200.terms import SymDirichlet

    pos, faces, uv = mg.punctured_icosphere_arrays(10)
    mesh = mg.Mesh(pos, faces)
    nv = len(pos)
    rest_inv, areas = rest_geometry(mesh)
    terms = [("FV", SymDirichlet(np.ascontiguousarray(rest_inv).reshape(-1, 4), areas))]
    p = mg.Problem(mesh, 2, with_hessian=True)
    p.add_term(mg.Element.FACE, mg.Op.FV, terms[0][1])
    p.precompute_sparsity()
    _check_pattern(p, nv, faces, mesh.edges, terms)
    x = uv.ravel().copy()
    v = np.random.default_rng(1).normal(size=x.size)
    p.x = x
    _check_energy(p, full_energy(nv, faces, mesh.edges, 2, terms, x), x)
    rng = np.random.default_rng(0)
    # the puncture's boundary ring (valence 4-5 rows) and the 12 valence-5 vertices' images
    deg = np.bincount(faces.ravel(), minlength=nv)
    extra = np.concatenate([np.flatnonzero(deg < 6)[:2000], [0, nv - 1]])
    so = SampledOracle(nv, faces, mesh.edges, 2, terms, sample_rows(nv, rng, SAMPLE, extra))
    _check_eval(p, so, x, (None, FLOOR))
    _check_hvp(p, so, x, v, (None, FLOOR))
    assert p.exact_runs() == 0
    del p
    _free()


def test_sphere_matches_oracle_at_baseline_size(ico10):
    """Config 4b: sphere barrier + stretch on icosphere(10) (gradient-mode
    problem as apps/sphere.py builds it), x = 1e-5 N(0,1) tangent coordinates
    (below the 1.1e-3 edge length: no flipped faces), v = N(0,1)."""
    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import initial_sphere, tangent_bases
    from paper_2509_00406_b200.terms import SphereBarrierStretch

    pos, faces = ico10
    mesh = mg.Mesh(pos, faces)
    nv = len(pos)
    base = initial_sphere(mesh)
    b1, b2 = tangent_bases(base)
    terms = [("FV", SphereBarrierStretch(base, b1, b2, True, True))]
    p = mg.Problem(mesh, 2, with_hessian=False)
    p.add_term(mg.Element.FACE, mg.Op.FV, terms[0][1])
    x = 1e-5 * np.random.default_rng(0).normal(size=2 * nv)
    v = np.random.default_rng(1).normal(size=x.size)
    p.x = x
    _check_energy(p, full_energy(nv, faces, mesh.edges, 2, terms, x), x)
    rng = np.random.default_rng(2)
    extra = np.arange(12)  # the icosahedron's valence-5 vertices
    so = SampledOracle(nv, faces, mesh.edges, 2, terms, sample_rows(nv, rng, SAMPLE, extra), with_hessian=False)
    _check_eval(p, so, x, (None,))
    _check_hvp(p, so, x, v, (None, FLOOR))
    del p
    _free()


def test_smoothing_matches_oracle_at_baseline_size(ico10):
    """Config 4a: the smoothing edge term on icosphere(10), x = positions."""
    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.terms import EdgeLength

    pos, faces = ico10
    mesh = mg.Mesh(pos, faces)
    nv = len(pos)
    terms = [("EV", EdgeLength())]
    p = mg.Problem(mesh, 3, with_hessian=False)
    p.add_term(mg.Element.EDGE, mg.Op.EV, terms[0][1])
    x = pos.ravel().copy()
    v = np.random.default_rng(1).normal(size=x.size)
    p.x = x
    _check_energy(p, full_energy(nv, faces, mesh.edges, 3, terms, x), x)
    so = SampledOracle(nv, faces, mesh.edges, 3, terms, sample_rows(nv, np.random.default_rng(3), SAMPLE, np.arange(12)),
                       with_hessian=False)
    _check_eval(p, so, x, (None,))
    _check_hvp(p, so, x, v, (None,))
    del p
    _free()
