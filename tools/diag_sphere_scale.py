"""Diagnose sphere-gradient parity at icosphere(s): GPU vs oracle vs a
40-digit mpmath evaluation on the worst rows."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import mpmath as mp
import torch
import paper_2509_00406_b200 as mg
from paper_2509_00406_b200.apps import initial_sphere, tangent_bases
from paper_2509_00406_b200.terms import SphereBarrierStretch
from scale_util import SampledOracle, device_rows, sample_rows

sub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
mp.mp.dps = 40
pos, faces = mg.icosphere_arrays(sub)
mesh = mg.Mesh(pos, faces)
nv = len(pos)
base = initial_sphere(mesh)
b1, b2 = tangent_bases(base)
terms = [("FV", SphereBarrierStretch(base, b1, b2, True, True))]
p = mg.Problem(mesh, 2, with_hessian=False)
p.add_term(mg.Element.FACE, mg.Op.FV, terms[0][1])
x = 1e-5 * np.random.default_rng(0).normal(size=2 * nv)
p.x = x
p.eval_terms()
rows = sample_rows(nv, np.random.default_rng(2), 20000, np.arange(12))
so = SampledOracle(nv, faces, mesh.edges, 2, terms, rows, with_hessian=False)
g, _, _ = device_rows(p, rows)
og, _, _ = so.eval_rows(x)
scale = np.abs(og).max()
err = np.abs(g - og).reshape(-1, 2).max(axis=1)
worst = np.argsort(err)[::-1][:4]
X = x.reshape(-1, 2)


def face_energy_mp(f, v, k, t):
    ps = []
    for q in range(3):
        u = f[q]
        xx = [mp.mpf(X[u, 0]), mp.mpf(X[u, 1])]
        if u == v:
            xx[k] += t
        r = [xx[0] * mp.mpf(b1[u, c]) + xx[1] * mp.mpf(b2[u, c]) + mp.mpf(base[u, c]) for c in range(3)]
        n = mp.sqrt(sum(c * c for c in r))
        ps.append([c / n for c in r])
    m = mp.matrix([[ps[j][i] for j in range(3)] for i in range(3)])
    e = -mp.log(mp.det(m))
    for a, b in ((0, 1), (1, 2), (2, 0)):
        e += sum((ps[a][c] - ps[b][c]) ** 2 for c in range(3))
    return e


inc = {}
for i in worst.tolist() + [0, 1]:
    inc[int(rows[i])] = np.flatnonzero((faces == rows[i]).any(axis=1))
print("scale", scale, "max rel", err.max() / scale)
for i in worst.tolist() + [0, 1]:
    v = int(rows[i])
    tru = []
    for k in range(2):
        d = mp.diff(lambda t: sum(face_energy_mp(faces[f], v, k, t) for f in inc[v]), 0)
        tru.append(float(d))
    tru = np.array(tru)
    print(v, "gpu", g[2 * i:2 * i + 2], "orc", og[2 * i:2 * i + 2], "true", tru,
          "gpu err/scale", np.abs(g[2 * i:2 * i + 2] - tru).max() / scale,
          "orc err/scale", np.abs(og[2 * i:2 * i + 2] - tru).max() / scale)
