"""float32 storage (Problem(dtype=torch.float32), mg_problem_set_storage):
x, gradient, Hessian values, HVP vectors and the builtin terms' attributes
stored in fp32, the edge row kernels computing in fp64. Against the unmodified
reference's float64 golden vectors the results agree within 1e-5 relative
(the north star's fp32 tolerance), the pattern stays bit-exact; problems the
fp32 path does not cover fail loudly."""

import numpy as np
import pytest

from engine_util import engine_problem
from golden_util import FLOOR, load, rel, rel_scalar, states

pytestmark = pytest.mark.gpu

TOL = 1e-5
EDGE_CASES = ["cloth8", "cloth64", "spring_grid16", "spring_pinned", "smooth_ico2", "smooth_ico2_grad"]


@pytest.mark.parametrize("name", EDGE_CASES)
def test_float32_storage_matches_reference(name):
    import torch

    d = load(name)
    p = engine_problem(d, dtype=torch.float32)
    if p.with_hessian:
        h = p.precompute_sparsity()
        assert np.array_equal(h.row_offsets, d["row_offsets"]) and np.array_equal(h.col_indices, d["col_indices"])
        assert h.values_device.dtype == torch.float32
    for s in states(d):
        x = d[f"s{s}_x"]
        if not np.isfinite(x).all():
            continue
        p.x = x
        e = p.eval_terms()
        assert p.grad_device.dtype == torch.float32
        assert rel_scalar(e, d[f"s{s}_energy"]) <= TOL
        assert rel(p.grad, d[f"s{s}_grad"]) <= TOL
        if f"s{s}_hess" in d:
            assert rel(p.hess.values, d[f"s{s}_hess"]) <= TOL
        if f"s{s}_psd_hess" in d:
            e = p.eval_terms(psd_floor=FLOOR)
            assert rel_scalar(e, d[f"s{s}_psd_energy"]) <= TOL
            assert rel(p.hess.values, d[f"s{s}_psd_hess"]) <= TOL
        assert rel_scalar(p.eval_energy_only(x), d[f"s{s}_energy_only"]) <= TOL
        if f"s{s}_v0" in d:
            y = p.hvp(x, d[f"s{s}_v0"])
            assert y.dtype == np.float32
            assert rel(y, d[f"s{s}_hvp0"]) <= TOL
            if f"s{s}_hvp_psd0" in d:
                assert rel(p.hvp(x, d[f"s{s}_v0"], psd_floor=FLOOR), d[f"s{s}_hvp_psd0"]) <= TOL


def test_float32_storage_rejects_other_paths():
    import torch

    d = load("dirichlet_ico2")
    p = engine_problem(d, dtype=torch.float32)
    p.precompute_sparsity()
    p.x = d["s0_x"]
    with pytest.raises(NotImplementedError):
        p.eval_terms()
    with pytest.raises(ValueError):
        engine_problem(load("cloth8"), accumulation="atomic", dtype=torch.float32)
