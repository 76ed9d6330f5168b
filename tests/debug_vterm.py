import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, paper_2509_00406_b200 as mg
pos, f = mg.grid_arrays(4, 0.1)
rng = np.random.default_rng(0)
x = (pos + 0.01 * rng.normal(size=pos.shape)).ravel()
for acc in ("deterministic", "atomic"):
    m = mg.Mesh(pos, f)
    p = mg.Problem(m, 3, accumulation=acc)
    p.add_term(mg.Element.VERTEX, mg.Op.V, mg.Inertia(np.ones(16), np.zeros((16, 3))))
    p.x = x
    e = p.eval_terms()
    print(acc, e, p.grad[:6], p.hess.values[:2].ravel()[:6])
    p2 = mg.Problem(m, 3, accumulation=acc, with_hessian=False)
    p2.add_term(mg.Element.VERTEX, mg.Op.V, mg.Inertia(np.ones(16), np.zeros((16, 3))))
    p2.x = x
    print(' grad-only', p2.eval_terms(), p2.grad[:6])
    print(' hvp', p.hvp(x, np.ones_like(x))[:6])
print('x', x[:6])
