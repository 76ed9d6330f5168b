"""The oracle is pinned: it reproduces every golden vector produced by the
unmodified reference (tests/golden/make_golden.py) — CPU only."""

import numpy as np
import pytest

from golden_util import FLOOR, cases, load, oracle_problem, rel, rel_scalar, states

TOL = 1e-12


@pytest.mark.parametrize("name", [c for c in cases() if c != "cloth16_asis"])
def test_oracle_matches_reference(name):
    d = load(name)
    op = oracle_problem(d)
    if "row_offsets" in d:
        assert np.array_equal(op.row_offsets, d["row_offsets"])
        assert np.array_equal(op.col_indices, d["col_indices"])
    for s in states(d):
        x = d[f"s{s}_x"]
        e, g, h = op.eval_terms(x)
        assert rel_scalar(e, d[f"s{s}_energy"]) <= TOL
        assert rel(g, d[f"s{s}_grad"]) <= TOL
        if f"s{s}_hess" in d:
            assert rel(h, d[f"s{s}_hess"]) <= TOL
        if f"s{s}_psd_hess" in d:
            e, g, h = op.eval_terms(x, psd_floor=FLOOR)
            assert rel_scalar(e, d[f"s{s}_psd_energy"]) <= TOL
            assert rel(g, d[f"s{s}_psd_grad"]) <= TOL
            assert rel(h, d[f"s{s}_psd_hess"]) <= 1e-11
        assert rel_scalar(op.eval_energy_only(x), d[f"s{s}_energy_only"]) <= TOL
        k = 0
        while f"s{s}_v{k}" in d:
            v = d[f"s{s}_v{k}"]
            assert rel(op.hvp(x, v), d[f"s{s}_hvp{k}"]) <= TOL
            if f"s{s}_hvp_psd{k}" in d:
                assert rel(op.hvp(x, v, psd_floor=FLOOR), d[f"s{s}_hvp_psd{k}"]) <= 1e-11
            k += 1


def test_oracle_cloth_asis_trajectory():
    d = load("cloth16_asis")
    for s in range(int(d["iterates"])):
        d["a_target"] = d[f"s{s}_target"]
        op = oracle_problem(d)
        floor = float(d[f"s{s}_floor"])
        e, g, h = op.eval_terms(d[f"s{s}_x"], psd_floor=None if np.isnan(floor) else floor)
        assert rel_scalar(e, d[f"s{s}_energy"]) <= TOL
        assert rel(g, d[f"s{s}_grad"]) <= TOL
        assert rel(h, d[f"s{s}_hess"]) <= 1e-11


def test_known_answers():
    # single stretched spring, length 2, l=1, k=1 (test_problem.py:106-112)
    d = load("spring_single")
    e, g, _ = oracle_problem(d).eval_terms(d["s0_x"])
    assert e == pytest.approx(4.5, rel=1e-15)
    assert np.allclose(g, [-12, 0, 0, 12, 0, 0])


def test_golden_nan_fields():
    # -log(det<0): NaN energy, finite derivatives
    d = load("sphere_flip")
    assert np.isnan(d["s0_energy"])
    d = load("spring_nan")
    assert np.isnan(d["s0_energy"])


def test_threaded_deterministic_bitwise():
    d = load("spring_grid16")
    r1 = oracle_problem(d, workers=1).eval_terms(d["s0_x"])
    r4 = oracle_problem(d, workers=4).eval_terms(d["s0_x"])
    assert r1[0] == r4[0]
    assert np.array_equal(r1[1], r4[1]) and np.array_equal(r1[2], r4[2])


def bsr_matvec(row_offsets, col_indices, values, r, n=3):
    """y = H r for a block-CSR matrix (host, test helper)."""
    vals = np.asarray(values).reshape(-1, n, n)
    rows = np.repeat(np.arange(len(row_offsets) - 1), np.diff(row_offsets))
    prod = np.einsum("kij,kj->ki", vals, r.reshape(-1, n)[col_indices])
    y = np.zeros((len(row_offsets) - 1, n))
    np.add.at(y, rows, prod)
    return y.ravel()


@pytest.mark.parametrize("s", [0, 3, 7])
def test_oracle_cloth64_asis_trajectory(s):
    """Config 1 as-is at 64x64: Newton iterates of the unmodified ClothSim
    (first, middle and last of its 8 evaluations over 2 steps)."""
    d = load("traj_cloth64_asis")
    assert int(d["iterates"]) == 8
    d["a_target"] = d[f"s{s}_target"]
    op = oracle_problem(d)
    floor = float(d[f"s{s}_floor"])
    e, g, h = op.eval_terms(d[f"s{s}_x"], psd_floor=None if np.isnan(floor) else floor)
    assert rel_scalar(e, d[f"s{s}_energy"]) <= TOL
    assert rel(g, d[f"s{s}_grad"]) <= 1e-11
    assert rel(bsr_matvec(op.row_offsets, op.col_indices, h, d["r"]), d[f"s{s}_hr"]) <= 1e-11
