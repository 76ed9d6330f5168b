"""The sampled-row oracle used by the at-scale parity tests is exact: on
golden problems, the rows it reports equal the whole-mesh oracle's rows
(bit-for-bit pattern rows, values to rounding), and the whole-mesh pattern
restatement equals the reference's golden pattern."""

import numpy as np
import pytest

from golden_util import FLOOR, build_terms, load, oracle_problem, rel
from scale_util import SampledOracle, block_index, dof_index, full_pattern, sample_rows


@pytest.mark.parametrize("name", ["cloth64", "dirichlet_ico2_pinned", "dirichlet_ico2", "sphere_ico2", "smooth_ico2", "mixed_fv_ev_v"])
def test_sampled_rows_equal_full_oracle(name):
    d = load(name)
    terms = build_terms(d)
    nv, n = len(d["positions"]), int(d["n"])
    fixed = d["fixed"].tolist()
    full = oracle_problem(d)
    rows = sample_rows(nv, np.random.default_rng(0), max(3, nv // 5), fixed[:1])
    so = SampledOracle(nv, d["faces"], d["edges"], n, terms, rows, fixed=fixed, with_hessian=bool(d["with_hessian"]))
    assert so.elements <= sum(len(g.ids) for g in full.groups)
    x = d["s0_x"]
    v = np.random.default_rng(1).normal(size=x.size)
    dofs = dof_index(rows, n)
    for floor in ((None, FLOOR) if full.with_hessian else (None,)):
        _, g, h = full.eval_terms(x, psd_floor=floor)
        sg, sh, scols = so.eval_rows(x, psd_floor=floor)
        assert rel(sg, g[dofs]) <= 1e-13
        if h is not None:
            bidx = block_index(full.row_offsets, rows)
            assert np.array_equal(scols, full.col_indices[bidx])
            assert rel(sh, h[bidx]) <= 1e-13
        assert rel(so.hvp_rows(x, v, psd_floor=floor), full.hvp(x, v, psd_floor=floor)[dofs]) <= 1e-13
    if "row_offsets" in d:
        ro, ci = full_pattern(nv, d["faces"], d["edges"], terms, fixed)
        assert np.array_equal(ro, d["row_offsets"]) and np.array_equal(ci, d["col_indices"])
