"""Host-side pieces of the device drivers (paper_2509_00406_b200/drivers.py):
topology checks, boundary loop, planar start, retraction and the closed-form
smoothing gradient, against direct restatements. CPU only."""

import numpy as np
import pytest


def _mg():
    import paper_2509_00406_b200 as mg

    return mg


def test_boundary_loop_of_a_grid_is_its_perimeter():
    from paper_2509_00406_b200.drivers import boundary_loop

    mg = _mg()
    n = 5
    m = mg.generate_grid(n)
    loop = boundary_loop(m)
    assert len(loop) == 4 * (n - 1) and loop[0] == 0
    per = {0, n - 1, n * (n - 1), n * n - 1}
    assert per <= set(loop)
    e = {tuple(sorted(p)) for p in m.edges.tolist()}
    for a, b in zip(loop, loop[1:] + loop[:1]):
        assert (min(a, b), max(a, b)) in e


def test_topology_errors():
    from paper_2509_00406_b200.drivers import boundary_loop, check_genus_zero

    mg = _mg()
    with pytest.raises(ValueError, match="no boundary"):
        boundary_loop(mg.generate_icosphere(1))
    with pytest.raises(ValueError, match="not closed genus 0"):
        check_genus_zero(mg.generate_grid(3))
    check_genus_zero(mg.generate_icosphere(1))


def test_numpy_helpers():
    from paper_2509_00406_b200.drivers import face_determinants, manual_energy, manual_gradient, retract_rows

    mg = _mg()
    rng = np.random.default_rng(2)
    m = mg.generate_grid(4)
    x = m.positions + 0.1 * rng.normal(size=m.positions.shape)
    g = manual_gradient(x, m)
    ref = np.zeros_like(x)
    for i, j in m.edges:
        ref[i] += 2 * (x[i] - x[j])
        ref[j] += 2 * (x[j] - x[i])
    assert np.allclose(g, ref, atol=1e-13)
    d = x[m.edges[:, 0]] - x[m.edges[:, 1]]
    assert manual_energy(x, m) == pytest.approx(float((d * d).sum()), rel=1e-14)
    s = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
    b1 = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    b2 = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    r = retract_rows(s, b1, b2, np.array([[0.5, 0.0], [0.0, 0.0]]))
    assert np.allclose(np.linalg.norm(r, axis=1), 1.0) and np.allclose(r[1], s[1])
    pts = mg.generate_icosphere(1).positions
    assert np.all(face_determinants(pts / np.linalg.norm(pts, axis=1, keepdims=True),
                                    mg.generate_icosphere(1).faces) > 0)
