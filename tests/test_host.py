"""CPU-only checks: the C ABI library loads and exports every declared symbol,
generators reproduce the reference meshes bit for bit, term formulas and
containers behave like the reference's."""

import re
from pathlib import Path

import numpy as np
import pytest

from golden_util import load

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "meshgrad_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*MG_API\s+(?:int|const char\*)\s+(mg_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2509_00406_b200 import _lib

    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert {n for n, _, _ in _lib.SIGNATURES} == set(names)
    assert lib.mg_abi_version() == 1


def test_abi_rejects_null_handles_without_gpu():
    from paper_2509_00406_b200 import _lib

    lib = _lib.load()
    assert lib.mg_eval(None, None, 0, 0.0, None, None, None, None) == _lib.MG_ERR_VALUE
    assert b"NULL" in lib.mg_last_error()


def test_generators_match_reference_meshes():
    from paper_2509_00406_b200.mesh import _host_edges, grid_arrays, icosphere_arrays, punctured_icosphere_arrays

    d = load("cloth8")
    pos, f = grid_arrays(8, 0.1)
    assert np.array_equal(pos, d["positions"]) and np.array_equal(f, d["faces"])
    assert np.array_equal(_host_edges(f, None, 64), d["edges"])
    d = load("smooth_ico2")
    pos, f = icosphere_arrays(2)
    assert np.array_equal(pos, d["positions"]) and np.array_equal(f, d["faces"])
    d = load("dirichlet_ico2")
    pos, f, _ = punctured_icosphere_arrays(2)
    assert np.array_equal(pos, d["positions"]) and np.array_equal(f, d["faces"])


def test_mesh_validation_messages():
    import paper_2509_00406_b200 as mg

    with pytest.raises(mg.MeshError, match="outside"):
        mg.Mesh(np.eye(3), [[0, 1, 5]])
    with pytest.raises(mg.MeshError, match="repeated"):
        mg.Mesh(np.eye(3), [[0, 1, 1]])
    with pytest.raises(mg.MeshError, match="positions"):
        mg.Mesh(np.eye(2), [[0, 1, 1]])
    with pytest.raises(mg.MeshError, match="identical"):
        mg.Mesh(np.eye(3), np.zeros((0, 3)), edges=[[1, 1]])


def test_small_matrix_and_vec_on_plain_floats():
    from paper_2509_00406_b200.active import ActiveVec, SmallMatrix

    m = SmallMatrix([[1.0, 2.0], [3.0, 4.0]])
    assert m.frobenius2() == 30.0
    assert m.det() == -2.0
    inv = m.inverse()
    assert np.allclose(np.array(inv.rows, dtype=float) @ np.array(m.rows), np.eye(2))
    a = ActiveVec([1.0, 2.0, 2.0])
    assert a.norm() == 3.0
    assert list(a.cross([0.0, 0.0, 1.0])) == [2.0, -1.0, 0.0]


def test_no_oracle_imports_in_product():
    pkg = ROOT / "paper_2509_00406_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", f.read_text(), flags=re.M), f
