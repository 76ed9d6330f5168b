"""Generate golden vectors by running the UNMODIFIED reference `meshgrad`.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each case builds the reference Problem with the reference's own builders /
callbacks (apps/cloth.py, apps/param.py, apps/sphere.py, apps/smooth.py and
the test-suite spring of test_problem.py:12-25), evaluates it on seeded
states and stores inputs + outputs in tests/golden/<case>.npz together with a
`spec` describing the equivalent builtin terms. Nothing at test time imports
the reference; the GPU box never sees /root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import meshgrad as mg  # noqa: E402
from meshgrad.apps.cloth import ClothConfig, ClothSim  # noqa: E402
from meshgrad.apps.param import make_distortion_problem, rest_geometry  # noqa: E402
from meshgrad.apps.smooth import edge_length_energy  # noqa: E402
from meshgrad.apps.sphere import initial_sphere, make_sphere_problem, tangent_bases  # noqa: E402
from meshgrad.mesh import Element, Op  # noqa: E402

sys.path.insert(0, str(OUT.parent.parent))
from paper_2509_00406_b200.mesh import icosphere_arrays, punctured_icosphere_arrays  # noqa: E402

FLOOR = 1e-9


def battery(p, states, vs, tag_hess=True, psd=True):
    """Evaluate the reference on every state: eval (+psd), energy-only, hvp (+psd)."""
    out = {}
    for s, x in enumerate(states):
        p.x = x.copy()
        out[f"s{s}_x"] = x
        out[f"s{s}_energy"] = np.array(p.eval_terms())
        out[f"s{s}_grad"] = p.grad.copy()
        if p.with_hessian and tag_hess:
            out[f"s{s}_hess"] = p.hess.values.copy()
            if psd:
                out[f"s{s}_psd_energy"] = np.array(p.eval_terms(psd_floor=FLOOR))
                out[f"s{s}_psd_grad"] = p.grad.copy()
                out[f"s{s}_psd_hess"] = p.hess.values.copy()
        out[f"s{s}_energy_only"] = np.array(p.eval_energy_only(x))
        for k, v in enumerate(vs):
            out[f"s{s}_v{k}"] = v
            out[f"s{s}_hvp{k}"] = p.hvp(x, v)
            if psd:
                out[f"s{s}_hvp_psd{k}"] = p.hvp(x, v, psd_floor=FLOOR)
    if p.hess is not None:
        out["row_offsets"] = p.hess.row_offsets.copy()
        out["col_indices"] = p.hess.col_indices.copy()
    return out


def save(name, mesh, n, spec, outs, fixed=(), with_hessian=True, extra=None):
    data = {
        "positions": mesh.positions,
        "faces": mesh.faces,
        "edges": mesh.edges,
        "n": np.array(n),
        "fixed": np.array(list(fixed), dtype=np.int64),
        "with_hessian": np.array(with_hessian),
        "spec": np.array(json.dumps(spec)),
    }
    data.update(outs)
    if extra:
        data.update(extra)
    path = OUT / f"{name}.npz"
    np.savez_compressed(path, **data)
    print(f"{name}: {path.stat().st_size / 1024:.1f} KiB, states={sum(1 for k in outs if k.endswith('_x'))}")


def ref_spring_problem(mesh, l2, k=1.0, **kw):
    p = mg.Problem(mesh, 3, **kw)

    def spring(edge, verts, x):
        d = x[verts[0]] - x[verts[1]]
        s = d.norm2() / l2[edge.index] - 1.0
        return (0.5 * k) * l2[edge.index] * (s * s)

    p.add_term(Element.EDGE, Op.EV, spring)
    return p


def case_springs():
    mesh = mg.Mesh(np.array([[0.0, 0, 0], [2.0, 0, 0]]), np.zeros((0, 3)), edges=[[0, 1]])
    l2 = np.ones(1)
    spec = [{"type": "Spring", "op": "EV", "coef": 0.5, "attrs": {"rest_len2": "a_l2"}}]
    rng = np.random.default_rng(5)
    states = [mesh.positions.ravel().copy(), mesh.positions.ravel() + 0.3 * rng.normal(size=6)]
    vs = [rng.normal(size=6), np.eye(6)[2]]
    p = ref_spring_problem(mesh, l2)
    save("spring_single", mesh, 3, spec, battery(p, states, vs), extra={"a_l2": l2})
    p = ref_spring_problem(mesh, l2, fixed_vertices=[0])
    save("spring_pinned", mesh, 3, spec, battery(p, states, vs), fixed=[0], extra={"a_l2": l2})
    # non-finite state: NaN surfaces, no exception (test_problem.py:157-161)
    p = ref_spring_problem(mesh, l2)
    save("spring_nan", mesh, 3, spec, battery(p, [np.full(6, np.nan)], [np.ones(6)]), extra={"a_l2": l2})
    # grid 16 springs, pinned corners (accumulation test shape, test_problem.py:352-358)
    g = mg.generate_grid(16, 1.0 / 15)
    l2 = np.full(g.num_edges, 0.05 ** 2)
    x = g.positions.ravel() + 0.01 * np.sin(np.arange(3 * g.num_vertices))
    p = ref_spring_problem(g, l2, fixed_vertices=[0, 255])
    save("spring_grid16", g, 3, spec, battery(p, [x], [rng.normal(size=3 * g.num_vertices)]),
         fixed=[0, 255], extra={"a_l2": l2})


def case_cloth(grid_n, name, seed=0):
    sim = ClothSim(ClothConfig(grid_n=grid_n))
    rng = np.random.default_rng(seed)
    pos = sim.mesh.positions
    sim._target[:] = pos + 0.01 * rng.normal(size=pos.shape)
    x = (pos + 0.01 * rng.normal(size=pos.shape)).ravel()
    v = np.random.default_rng(1).normal(size=x.size)
    cfg = sim.cfg
    spec = [
        {"type": "Inertia", "op": "V", "attrs": {"masses": "a_masses", "target": "a_target"}},
        {"type": "Spring", "op": "EV", "coef": 0.5 * cfg.k * (cfg.h * cfg.h), "attrs": {"rest_len2": "a_l2"}},
        {"type": "Gravity", "op": "V", "h2": cfg.h * cfg.h, "gravity": list(cfg.gravity),
         "attrs": {"masses": "a_masses"}},
    ]
    outs = battery(sim.problem, [x], [v])
    save(name, sim.mesh, 3, spec, outs, fixed=sim.pinned,
         extra={"a_masses": sim.masses, "a_target": sim._target.copy(), "a_l2": sim.rest_len2})


def case_cloth_asis():
    """Every Newton iterate the unmodified ClothSim visits in 2 steps (config 1
    'as-is', at 16x16 to keep the fixture small)."""
    sim = ClothSim(ClothConfig(grid_n=16))
    rec = {}
    orig = sim.problem.eval_terms
    count = [0]

    def spy(psd_floor=None):
        e = orig(psd_floor=psd_floor)
        i = count[0]
        rec[f"s{i}_x"] = sim.problem.x.copy()
        rec[f"s{i}_target"] = sim._target.copy()
        rec[f"s{i}_floor"] = np.array(np.nan if psd_floor is None else psd_floor)
        rec[f"s{i}_energy"] = np.array(e)
        rec[f"s{i}_grad"] = sim.problem.grad.copy()
        rec[f"s{i}_hess"] = sim.problem.hess.values.copy()
        count[0] += 1
        return e

    sim.problem.eval_terms = spy
    sim.simulate(steps=2)
    cfg = sim.cfg
    spec = [
        {"type": "Inertia", "op": "V", "attrs": {"masses": "a_masses", "target": "a_target"}},
        {"type": "Spring", "op": "EV", "coef": 0.5 * cfg.k * (cfg.h * cfg.h), "attrs": {"rest_len2": "a_l2"}},
        {"type": "Gravity", "op": "V", "h2": cfg.h * cfg.h, "gravity": list(cfg.gravity),
         "attrs": {"masses": "a_masses"}},
    ]
    rec["row_offsets"] = sim.problem.hess.row_offsets.copy()
    rec["col_indices"] = sim.problem.hess.col_indices.copy()
    save("cloth16_asis", sim.mesh, 3, spec, rec, fixed=sim.pinned,
         extra={"a_masses": sim.masses, "a_target": sim._target.copy(), "a_l2": sim.rest_len2,
                "iterates": np.array(count[0])})


def case_cloth64_asis():
    """Config 1 as-is at its own size: every Newton iterate the unmodified
    64x64 ClothSim visits in 2 steps. The Hessians are stored as H r for one
    seeded r (full values would be ~2 MB per iterate); the step states after
    simulate() check the device driver end to end."""
    sim = ClothSim(ClothConfig(grid_n=64))
    rec = {}
    orig = sim.problem.eval_terms
    count = [0]
    r = np.random.default_rng(7).normal(size=sim.problem.num_dofs)

    def spy(psd_floor=None):
        e = orig(psd_floor=psd_floor)
        i = count[0]
        rec[f"s{i}_x"] = sim.problem.x.copy()
        rec[f"s{i}_target"] = sim._target.copy()
        rec[f"s{i}_floor"] = np.array(np.nan if psd_floor is None else psd_floor)
        rec[f"s{i}_energy"] = np.array(e)
        rec[f"s{i}_grad"] = sim.problem.grad.copy()
        rec[f"s{i}_hr"] = sim.problem.hess.matvec(r)
        count[0] += 1
        return e

    sim.problem.eval_terms = spy
    x, v, reps = sim.simulate(steps=2)
    cfg = sim.cfg
    spec = [
        {"type": "Inertia", "op": "V", "attrs": {"masses": "a_masses", "target": "a_target"}},
        {"type": "Spring", "op": "EV", "coef": 0.5 * cfg.k * (cfg.h * cfg.h), "attrs": {"rest_len2": "a_l2"}},
        {"type": "Gravity", "op": "V", "h2": cfg.h * cfg.h, "gravity": list(cfg.gravity),
         "attrs": {"masses": "a_masses"}},
    ]
    rec["r"] = r
    rec["final_x"], rec["final_v"] = x, v
    rec["step_energies"] = np.array([rp.final_energy for rp in reps])
    save("traj_cloth64_asis", sim.mesh, 3, spec, rec, fixed=sim.pinned,
         extra={"a_masses": sim.masses, "a_target": sim._target.copy(), "a_l2": sim.rest_len2,
                "iterates": np.array(count[0])})


def case_dirichlet():
    p3, f, uv = punctured_icosphere_arrays(2)
    mesh = mg.Mesh(p3, f)
    rest_inv, areas = rest_geometry(mesh)
    from meshgrad.apps.param import jacobian_dets

    if jacobian_dets(uv, mesh, rest_inv).max() < 0:
        uv = uv[:, ::-1].copy()
    rng = np.random.default_rng(0)
    states = [uv.ravel().copy(), (uv + 0.002 * rng.normal(size=uv.shape)).ravel()]
    vs = [np.random.default_rng(1).normal(size=uv.size)]
    spec = [{"type": "SymDirichlet", "op": "FV", "attrs": {"rest_inv": "a_rest_inv", "areas": "a_areas"}}]
    extra = {"a_rest_inv": rest_inv.reshape(-1, 4), "a_areas": areas}
    p = make_distortion_problem(mesh, rest_inv, areas, with_hessian=True)
    save("dirichlet_ico2", mesh, 2, spec, battery(p, states, vs), extra=extra)
    p = make_distortion_problem(mesh, rest_inv, areas, with_hessian=False)
    save("dirichlet_ico2_grad", mesh, 2, spec, battery(p, states, vs), with_hessian=False, extra=extra)
    # pinned corners: the reference's masked lift (the app's own callback on a pinned Problem)
    fn = make_distortion_problem(mesh, rest_inv, areas)._terms[0].fn
    pins = [0, 7, 31, 60]
    p = mg.Problem(mesh, 2, with_hessian=True, fixed_vertices=pins)
    p.add_term(Element.FACE, Op.FV, fn)
    save("dirichlet_ico2_pinned", mesh, 2, spec, battery(p, states, vs), fixed=pins, extra=extra)
    # one flipped face on a flat 4x4 grid: NaN spreads per field
    g = mg.generate_grid(4, 1.0 / 3)
    ri, ar = rest_geometry(g)
    uvg = g.positions[:, :2].copy()
    uvg[5] = uvg[10] + 0.05  # drag an interior vertex across its neighbour
    p = make_distortion_problem(g, ri, ar, with_hessian=True)
    save("dirichlet_flip", g, 2, spec, battery(p, [uvg.ravel()], [np.ones(uvg.size)], psd=True),
         extra={"a_rest_inv": ri.reshape(-1, 4), "a_areas": ar})


def case_sphere():
    pos, f = icosphere_arrays(2)
    mesh = mg.Mesh(pos * np.array([1.3, 1.0, 0.8]), f)
    base = initial_sphere(mesh)
    b1, b2 = tangent_bases(base)
    rng = np.random.default_rng(0)
    x = 1e-3 * rng.normal(size=2 * mesh.num_vertices)
    vs = [np.random.default_rng(1).normal(size=x.size)]
    extra = {"a_base": base, "a_b1": b1, "a_b2": b2}
    for tag, bar, st in (("", True, True), ("_barrier", True, False), ("_stretch", False, True)):
        spec = [{"type": "SphereBarrierStretch", "op": "FV", "include_barrier": bar, "include_stretch": st,
                 "attrs": {"base": "a_base", "b1": "a_b1", "b2": "a_b2"}}]
        p = make_sphere_problem(mesh, base, b1, b2, with_hessian=True, include_barrier=bar, include_stretch=st)
        save(f"sphere_ico2{tag}", mesh, 2, spec, battery(p, [x], vs), extra=extra)
    spec = [{"type": "SphereBarrierStretch", "op": "FV", "include_barrier": True, "include_stretch": True,
             "attrs": {"base": "a_base", "b1": "a_b1", "b2": "a_b2"}}]
    p = make_sphere_problem(mesh, base, b1, b2, with_hessian=False)
    save("sphere_ico2_grad", mesh, 2, spec, battery(p, [x], vs), with_hessian=False, extra=extra)
    fn = make_sphere_problem(mesh, base, b1, b2)._terms[0].fn
    pins = [1, 12, 40, 99]
    p = mg.Problem(mesh, 2, with_hessian=True, fixed_vertices=pins)
    p.add_term(Element.FACE, Op.FV, fn)
    save("sphere_ico2_pinned", mesh, 2, spec, battery(p, [x], vs), fixed=pins, extra=extra)
    # a large tangent step that flips faces: -log(det<0) -> NaN energy, finite grad
    xf = x.copy()
    xf[0:2] = [2.5, -1.5]
    p = make_sphere_problem(mesh, base, b1, b2, with_hessian=True)
    save("sphere_flip", mesh, 2, spec, battery(p, [xf], vs), extra=extra)


def case_smooth():
    pos, f = icosphere_arrays(2)
    mesh = mg.Mesh(pos, f)
    rng = np.random.default_rng(3)
    x = (pos + 0.05 * rng.normal(size=pos.shape)).ravel()
    vs = [rng.normal(size=x.size)]
    spec = [{"type": "EdgeLength", "op": "EV", "attrs": {}}]
    save("smooth_ico2", mesh, 3, spec, battery(edge_length_energy(mesh, with_hessian=True), [x], vs))
    save("smooth_ico2_grad", mesh, 3, spec, battery(edge_length_energy(mesh, with_hessian=False), [x], vs),
         with_hessian=False)


def case_additivity():
    """EV + V terms in one problem (test_problem.py:177-206)."""
    mesh = mg.generate_grid(4)
    rng = np.random.default_rng(8)
    x = mesh.positions.ravel() + 0.2 * rng.normal(size=3 * mesh.num_vertices)
    p = mg.Problem(mesh, 3)
    p.add_term(Element.EDGE, Op.EV, lambda e, vs, xx: (xx[vs[0]] - xx[vs[1]]).norm2())
    p.add_term(Element.VERTEX, Op.V, lambda v, nb, xx: 0.5 * xx[v].norm2())
    spec = [{"type": "EdgeLength", "op": "EV", "attrs": {}},
            {"type": "Inertia", "op": "V", "attrs": {"masses": "a_ones", "target": "a_zeros"}}]
    save("additivity_grid4", mesh, 3, spec, battery(p, [x], [rng.normal(size=x.size)]),
         extra={"a_ones": np.ones(mesh.num_vertices), "a_zeros": np.zeros((mesh.num_vertices, 3))})


def case_mixed():
    """FV + EV + V terms on one UV problem (n = 2), pinned vertices: the
    generic patch-owner path (no single-term fast kernel applies)."""
    p3, f, uv = punctured_icosphere_arrays(1)
    mesh = mg.Mesh(p3, f)
    rest_inv, areas = rest_geometry(mesh)
    from meshgrad.apps.param import jacobian_dets

    if jacobian_dets(uv, mesh, rest_inv).max() < 0:
        uv = uv[:, ::-1].copy()
    rng = np.random.default_rng(21)
    e = mesh.edges
    l2 = np.einsum("ij,ij->i", uv[e[:, 1]] - uv[e[:, 0]], uv[e[:, 1]] - uv[e[:, 0]]) * 1.1
    masses = 1.0 + rng.random(mesh.num_vertices)
    target = uv + 0.01 * rng.normal(size=uv.shape)
    pins = [2, 9]
    fn_d = make_distortion_problem(mesh, rest_inv, areas)._terms[0].fn

    def spring(edge, verts, x):
        d = x[verts[0]] - x[verts[1]]
        s_ = d.norm2() / l2[edge.index] - 1.0
        return 0.7 * l2[edge.index] * (s_ * s_)

    def inertia(vertex, nbrs, x):
        d = x[vertex] - target[vertex.index]
        return 0.5 * masses[vertex.index] * d.norm2()

    p = mg.Problem(mesh, 2, with_hessian=True, fixed_vertices=pins)
    p.add_term(Element.FACE, Op.FV, fn_d)
    p.add_term(Element.EDGE, Op.EV, spring)
    p.add_term(Element.VERTEX, Op.V, inertia)
    spec = [{"type": "SymDirichlet", "op": "FV", "attrs": {"rest_inv": "a_rest_inv", "areas": "a_areas"}},
            {"type": "Spring", "op": "EV", "coef": 0.7, "attrs": {"rest_len2": "a_l2"}},
            {"type": "Inertia", "op": "V", "attrs": {"masses": "a_masses", "target": "a_target"}}]
    states = [(uv + 0.003 * rng.normal(size=uv.shape)).ravel()]
    vs = [rng.normal(size=uv.size)]
    save("mixed_fv_ev_v", mesh, 2, spec, battery(p, states, vs), fixed=pins,
         extra={"a_rest_inv": rest_inv.reshape(-1, 4), "a_areas": areas, "a_l2": l2, "a_masses": masses,
                "a_target": target})


if __name__ == "__main__":
    if len(sys.argv) > 1:  # named cases only, e.g. cloth64_asis
        for name in sys.argv[1:]:
            globals()[f"case_{name}"]()
        sys.exit(0)
    case_springs()
    case_cloth(8, "cloth8")
    case_cloth(64, "cloth64")
    case_cloth_asis()
    case_cloth64_asis()
    case_dirichlet()
    case_sphere()
    case_smooth()
    case_additivity()
    case_mixed()
