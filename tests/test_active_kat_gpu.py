"""The reference's dual-number known-answer tests (pkg/tests/test_active.py)
replayed on the DEVICE duals: every expression is a reference-style callback
traced by jit.py, compiled for sm_100a and evaluated by the engine as a V
term on a face-free mesh whose vertices are the test's lanes (var_dim = the
expression's variable count). Value = the energy (one lane), gradient = the
lane's gradient row, Hessian = the lane's diagonal block (a V term's whole
local Hessian), so each assertion reads like the reference's.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FD_STEP = 1e-5


# pkg/tests/oracles.py:9-38 (independent central differences and the error metric)
def fd_gradient(f, x, h=FD_STEP):
    x = np.asarray(x, dtype=np.float64)
    g = np.zeros_like(x)
    for i in range(x.size):
        e = np.zeros_like(x)
        e[i] = h
        g[i] = (f(x + e) - f(x - e)) / (2.0 * h)
    return g


def fd_jacobian(g, x, h=FD_STEP):
    x = np.asarray(x, dtype=np.float64)
    g0 = np.asarray(g(x))
    out = np.zeros((g0.size, x.size))
    for j in range(x.size):
        e = np.zeros_like(x)
        e[j] = h
        out[:, j] = (np.asarray(g(x + e)) - np.asarray(g(x - e))) / (2.0 * h)
    return out


def rel_err(candidate, reference):
    candidate = np.asarray(candidate, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    scale = max(1.0, float(np.max(np.abs(reference))) if reference.size else 0.0)
    return float(np.max(np.abs(candidate - reference))) / scale if candidate.size else 0.0


class Lanes:
    """`expr` over M lanes of k variables on the device: a V term per vertex."""

    def __init__(self, expr, vals, with_hessian=True):
        import paper_2509_00406_b200 as mg

        vals = np.atleast_2d(np.asarray(vals, dtype=np.float64))
        self.m, self.k = vals.shape
        mesh = mg.Mesh(np.zeros((self.m, 3)), np.zeros((0, 3)))
        self.p = mg.Problem(mesh, self.k, with_hessian=with_hessian)
        k = self.k
        self.p.add_term(mg.Element.VERTEX, mg.Op.V, lambda h, nb, x: expr(*[x[h][c] for c in range(k)]))
        self.p.x = vals.ravel()

    def run(self, psd_floor=None):
        e = self.p.eval_terms(psd_floor=psd_floor)
        g = self.p.grad.reshape(self.m, self.k)
        h = None
        if self.p.with_hessian:
            hs = self.p.hess
            assert np.array_equal(hs.col_indices, np.arange(self.m))  # one diagonal block per lane
            h = hs.values
        return e, g, h


def one(expr, vals, **kw):
    e, g, h = Lanes(expr, [vals], **kw).run()
    return e, g[0], (h[0] if h is not None else None)


def test_mul_frozen():  # test_active.py:40-46
    e, g, h = one(lambda x, y: x * y, [2.0, 3.0])
    assert e == 6.0
    assert np.allclose(g, [3.0, 2.0])
    assert np.allclose(h, [[0.0, 1.0], [1.0, 0.0]])


def test_div_frozen():  # :54-59 (division by a passive 2)
    e, g, h = one(lambda x: x / 2.0, [1.0])
    assert e == 0.5 and np.allclose(g, [0.5]) and np.allclose(h, [[0.0]])


def test_div_full_quotient_rule():  # :61-67
    f = lambda v: v[0] / v[1]
    x0 = np.array([1.7, -2.3])
    _, g, h = one(lambda x, y: x / y, x0)
    assert rel_err(g, fd_gradient(f, x0)) < 1e-9
    assert rel_err(h, fd_jacobian(lambda v: fd_gradient(f, v, 1e-4), x0, 1e-4)) < 1e-5


def test_reflected_ops():  # :75-82
    e, g, _ = one(lambda a: 3.0 - a, [2.0])
    assert e == 1.0 and np.allclose(g, [-1.0])
    e, g, _ = one(lambda a: 3.0 / a, [2.0])
    assert e == 1.5 and np.allclose(g, [-0.75])
    e, _, _ = one(lambda a: np.float64(2.0) * a, [2.0])
    assert e == 4.0


def test_pow_int():  # :84-94
    e, g, h = one(lambda a: a ** 3, [3.0])
    assert e == 27.0 and np.allclose(g, [27.0]) and np.allclose(h, [[18.0]])
    e, g, _ = one(lambda a: a ** 0 + 0.0 * a, [3.0])
    assert e == 1.0 and np.allclose(g, [0.0])


def test_division_by_zero_propagates():  # :96-99
    e, _, _ = one(lambda a, b: a / b, [1.0, 0.0])
    assert not np.isfinite(e)


def test_log_frozen():  # :103-107
    from paper_2509_00406_b200.active import log

    e, g, h = one(lambda x: log(x), [1.0])
    assert e == 0.0 and np.allclose(g, [1.0]) and np.allclose(h, [[-1.0]])


def test_sqrt_frozen():  # :109-113
    from paper_2509_00406_b200.active import sqrt

    e, g, h = one(lambda x: sqrt(x), [4.0])
    assert e == 2.0 and np.allclose(g, [0.25]) and np.allclose(h, [[-0.03125]])


def test_abs_at_zero():  # :120-124
    e, g, _ = one(lambda a: abs(a), [0.0])
    assert e == 0.0 and np.allclose(g, [0.0])


def test_out_of_domain_propagates():  # :126-128
    from paper_2509_00406_b200.active import log, sqrt

    assert not np.isfinite(one(lambda a: log(a), [-1.0])[0])
    assert not np.isfinite(one(lambda a: sqrt(a), [-1.0])[0])


@pytest.mark.parametrize("name,domain", [("sqrt", (0.1, 10.0)), ("log", (0.1, 10.0)), ("exp", (-3.0, 3.0)),
                                         ("sin", (-3.0, 3.0)), ("cos", (-3.0, 3.0))])
def test_unary_vs_fd(name, domain):  # :130-146, the 20 draws as 20 lanes of one problem
    import paper_2509_00406_b200.active as A

    fn, np_fn = getattr(A, name), getattr(np, name)
    x0 = np.random.default_rng(0).uniform(*domain, size=20)
    _, g, h = Lanes(lambda a: fn(a), x0[:, None]).run()
    for lane in range(20):
        gf = fd_gradient(lambda v: np_fn(v[0]), [x0[lane]])
        hf = fd_jacobian(lambda v: fd_gradient(lambda w: np_fn(w[0]), v), [x0[lane]])
        assert rel_err(g[lane], gf) < 1e-6
        assert rel_err(h[lane], hf) < 1e-5


def _composite(x, y, z):  # :149-153
    from paper_2509_00406_b200.active import cos, exp, log, sin, sqrt

    t = exp(sin(x) * 0.3) + sqrt(z) / (y * y + 1.0)
    u = log(z + 4.0) * cos(x - y) - abs(y) / z
    return t * u + (x - 2.0 * y + z) ** 2 + t / u


def _composite_plain(v):  # :156-160
    x, y, z = v
    t = np.exp(np.sin(x) * 0.3) + np.sqrt(z) / (y * y + 1.0)
    u = np.log(z + 4.0) * np.cos(x - y) - abs(y) / z
    return t * u + (x - 2.0 * y + z) ** 2 + t / u


def _draws(seed, n):
    rng = np.random.default_rng(seed)
    return np.array([[rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.5, 4)] for _ in range(n)])


def test_composite_gradient_100_random_inputs():  # :164-169
    v = _draws(42, 100)
    _, g, _ = Lanes(_composite, v).run()
    for lane in range(100):
        assert rel_err(g[lane], fd_gradient(_composite_plain, v[lane])) < 1e-6


def test_composite_hessian_vs_fd_of_ad_gradient_and_symmetric():  # :171-187
    v = _draws(43, 25)
    _, _, h = Lanes(_composite, v).run()
    g1 = Lanes(_composite, v[:1], with_hessian=False)

    def ad_grad(w):
        g1.p.x = np.asarray(w, dtype=np.float64)
        return g1.run()[1][0]

    for lane in range(25):
        assert rel_err(h[lane], fd_jacobian(ad_grad, v[lane])) < 1e-5
    assert np.array_equal(h, np.swapaxes(h, 1, 2))  # bitwise symmetric


def test_composite_first_and_second_order_agree():  # :189-197
    v = _draws(45, 20)
    e2, g2, _ = Lanes(_composite, v, with_hessian=True).run()
    e1, g1, h1 = Lanes(_composite, v, with_hessian=False).run()
    assert h1 is None
    assert e1 == e2
    assert np.array_equal(g1, g2)


def test_batch_lanes_match_scalar():  # :209-228
    from paper_2509_00406_b200.active import log, sqrt

    expr = lambda x, y: sqrt(x * x + y * y) * log(y) + x / y
    vals = np.random.default_rng(46).uniform(0.5, 3.0, size=(8, 2))
    _, g, h = Lanes(expr, vals).run()
    for lane in range(8):
        e1, g1, h1 = one(expr, vals[lane])
        assert np.allclose(g[lane], g1, rtol=1e-15) and np.allclose(h[lane], h1, rtol=1e-15)


def test_vec_dot_cross_norm_values():  # :239-251
    from paper_2509_00406_b200.active import ActiveVec

    rng = np.random.default_rng(47)
    a, b = rng.normal(size=3), rng.normal(size=3)
    cases = [(lambda *v: ActiveVec(v[:3]).dot(ActiveVec(v[3:])), a @ b),
             (lambda *v: ActiveVec(v[:3]).norm2(), a @ a),
             (lambda *v: ActiveVec(v[:3]).norm(), np.linalg.norm(a))]
    cr = np.cross(a, b)
    cases += [(lambda *v, c=c: ActiveVec(v[:3]).cross(ActiveVec(v[3:]))[c], cr[c]) for c in range(3)]
    for expr, want in cases:
        e, _, _ = one(expr, np.concatenate([a, b]))
        assert e == pytest.approx(want)


def test_cross_gradient_vs_fd():  # :253-263
    from paper_2509_00406_b200.active import ActiveVec

    v0 = np.random.default_rng(48).normal(size=6)
    f = lambda v: float(np.cross(v[:3], v[3:]) @ np.array([1.0, 2.0, 3.0]))
    _, g, _ = one(lambda *v: ActiveVec(v[:3]).cross(ActiveVec(v[3:])).dot(np.array([1.0, 2.0, 3.0])), v0)
    assert rel_err(g, fd_gradient(f, v0)) < 1e-7


def test_normalized_unit():  # :271-274
    from paper_2509_00406_b200.active import ActiveVec

    e, _, _ = one(lambda *v: ActiveVec(v).normalized().norm(), [3.0, 4.0, 0.0])
    assert e == pytest.approx(1.0)


def test_det_gradient():  # :285-293
    from paper_2509_00406_b200.active import SmallMatrix

    e, g, _ = one(lambda x: SmallMatrix([[x, 0.0], [0.0, 1.0]]).det(), [2.0])
    assert e == 2.0 and np.allclose(g, [1.0])


def test_inverse_times_matrix_is_identity():  # :295-304
    from paper_2509_00406_b200.active import SmallMatrix

    for seed in range(5):
        m = np.random.default_rng(seed).uniform(-2, 2, size=(2, 2)) + 3.0 * np.eye(2)
        for i in range(2):
            for j in range(2):
                def expr(a, b, c, d, i=i, j=j):
                    sm = SmallMatrix([[a, b], [c, d]])
                    return (sm.inverse() @ sm)[i, j]
                e, _, _ = one(expr, m.ravel())
                assert e == pytest.approx(1.0 if i == j else 0.0, abs=1e-12)


def test_matmul_and_frobenius():  # :306-315
    from paper_2509_00406_b200.active import SmallMatrix

    other = np.array([[1.0, 1.0], [0.0, 1.0]])
    assert one(lambda a, b, c, d: (SmallMatrix([[a, b], [c, d]]) @ other)[0, 1], [1.0, 2.0, 3.0, 4.0])[0] == 3.0
    assert one(lambda a, b, c, d: (SmallMatrix([[a, b], [c, d]]) @ other)[1, 1], [1.0, 2.0, 3.0, 4.0])[0] == 7.0
    assert one(lambda a, b, c, d: SmallMatrix([[a, b], [c, d]]).frobenius2(), [1.0, 2.0, 3.0, 4.0])[0] == 30.0


# project_psd (:318-349) through eval_terms(psd_floor): a quadratic 0.5 x^T H x
# has local Hessian H, so the assembled block is the reference's project_psd(H)

def _quadratic(h):
    k = len(h)

    def expr(*v):
        total = 0.0
        for i in range(k):
            for j in range(k):
                if h[i][j] != 0.0:
                    total = total + (0.5 * h[i][j]) * (v[i] * v[j])
        return total
    return expr


def _psd_block(h, floor=1e-9):
    lanes = Lanes(_quadratic(h), [np.full(len(h), 0.3)])
    return lanes.run(psd_floor=floor)[2][0]


def test_psd_already_psd_unchanged():  # :318-320
    assert np.allclose(_psd_block(np.diag([2.0, 3.0])), np.diag([2.0, 3.0]), atol=1e-12)


def test_psd_indefinite_frozen():  # :322-325
    assert np.allclose(_psd_block(np.array([[0.0, 2.0], [2.0, 0.0]])), [[1.0, 1.0], [1.0, 1.0]], atol=1e-8)


def test_psd_scalar_clamp():  # :327-328
    assert np.allclose(_psd_block(np.array([[-5.0]])), [[1e-9]])


def test_psd_floor_must_be_positive():  # :330-332
    lanes = Lanes(_quadratic(np.eye(2)), [[0.3, 0.3]])
    with pytest.raises(ValueError):
        lanes.run(psd_floor=0.0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_psd_min_eigenvalue_at_least_floor(seed):  # :333-340 (random symmetric 6x6)
    a = np.random.default_rng(seed).normal(size=(6, 6))
    out = _psd_block(0.5 * (a + a.T))
    assert np.array_equal(out, out.T)
    assert np.linalg.eigvalsh(out).min() >= 1e-9 - 1e-12


def test_positive_guard_poisons_nonpositive_lanes():  # :351-356 (values; derivatives pass through, active.py:326-327)
    from paper_2509_00406_b200.active import positive_guard

    assert one(lambda a: positive_guard(a), [1.0], with_hessian=False)[0] == 1.0
    for bad in (-2.0, 0.0):
        e, g, _ = one(lambda a: positive_guard(a), [bad], with_hessian=False)
        assert np.isnan(e) and np.array_equal(g, [1.0])
