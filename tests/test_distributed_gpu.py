"""Shard path of the CUDA engine (mg_mesh_set_owned) on one GPU: every rank
of a world-2/4 partition is built in this process on cuda:0 (the ribbon
state is filled from the global arrays, which is what the halo exchange
delivers — that exchange itself is tested with gloo in test_distributed.py).
Owned rows of gradient, Hessian (pattern bit-exact) and HVP, and the shard
energies summed, must match the reference's golden vectors (<= 1e-10)."""

import numpy as np
import pytest

from golden_util import FLOOR, build_terms, load, rel, rel_scalar

pytestmark = pytest.mark.gpu

CASES = ["cloth64", "spring_grid16", "smooth_ico2", "dirichlet_ico2", "sphere_ico2", "dirichlet_ico2_pinned",
         "mixed_fv_ev_v"]


@pytest.mark.parametrize("mode", ["deterministic", "atomic"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", CASES)
def test_shards_match_reference(name, world, mode):
    from paper_2509_00406_b200.distributed import DistributedProblem, ShardPlan

    d = load(name)
    n = int(d["n"])
    faces = d["faces"]
    edges = d["edges"] if not len(faces) else None
    terms = build_terms(d)
    x, v = d["s0_x"], d["s0_v0"]
    nv = len(d["positions"])
    g = np.full((nv, n), np.nan)
    y = np.full((nv, n), np.nan)
    yp = np.full((nv, n), np.nan)
    e = 0.0
    ep = 0.0
    hrows = {}
    for r in range(world):
        plan = ShardPlan(d["positions"], faces, edges, world, r)
        dp = DistributedProblem(d["positions"], faces, n, terms, fixed_vertices=d["fixed"].tolist(), edges=edges,
                                with_hessian=bool(d["with_hessian"]), accumulation=mode, plan=plan)
        dp.set_x_global(x)
        e += dp.eval_terms()
        own = plan.owned_global
        g[own] = dp.grad_owned().cpu().numpy()
        if dp.problem.with_hessian:
            offs, cols, vals = dp.hess_rows_owned()
            for i, vtx in enumerate(own):
                hrows[vtx] = (cols[offs[i]:offs[i + 1]], vals[offs[i]:offs[i + 1]])
        y[own] = dp.hvp_from_global(v).cpu().numpy()
        yp[own] = dp.hvp_from_global(v, psd_floor=FLOOR).cpu().numpy()
        if "s0_psd_energy" in d and dp.problem.with_hessian:
            ep += dp.eval_terms(psd_floor=FLOOR)
    assert rel_scalar(e, d["s0_energy"]) <= 1e-10
    assert rel(g.ravel(), d["s0_grad"]) <= 1e-10
    assert rel(y.ravel(), d["s0_hvp0"]) <= 1e-10
    assert rel(yp.ravel(), d["s0_hvp_psd0"]) <= 1e-10
    if hrows:
        ro, ci, hv = d["row_offsets"], d["col_indices"], d["s0_hess"]
        scale = np.abs(hv).max()
        for vtx in range(nv):
            lo, hi = ro[vtx], ro[vtx + 1]
            cols, vals = hrows[vtx]
            assert np.array_equal(cols, ci[lo:hi]), vtx
            assert np.abs(vals - hv[lo:hi]).max(initial=0.0) <= 1e-10 * scale
        assert rel_scalar(ep, d["s0_psd_energy"]) <= 1e-10
