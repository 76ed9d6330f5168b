"""OBJ load / save (ref mesh.py:376-429): accepted records, error texts with
line numbers, and a save -> load round trip. CPU only (no GPU kernels)."""

import numpy as np
import pytest


def _mg():
    import paper_2509_00406_b200 as mg

    return mg


def test_round_trip_and_suffixes(tmp_path):
    mg = _mg()
    pos, faces = mg.grid_arrays(4, 0.5)
    path = tmp_path / "g.obj"
    mg.save_obj(path, pos, faces)
    m = mg.load_obj(path)
    assert np.array_equal(m.faces, faces)
    assert np.allclose(m.positions, pos, atol=1e-6)
    # vt / vn suffixes and other records are ignored
    text = "# c\no x\nv 0 0 0\nv 1 0 0\nv 0 1 0\nvn 0 0 1\nf 1/1/1 2//1 3\n"
    p = tmp_path / "s.obj"
    p.write_text(text)
    m = mg.load_obj(p)
    assert m.num_faces == 1 and m.num_vertices == 3


@pytest.mark.parametrize("body,msg", [
    ("v 0 0\nf 1 2 3\n", "line 1: vertex record needs 3 coordinates"),
    ("v 0 0 x\n", "line 1: bad vertex coordinate"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\nf 1 2 3 4\n", "line 5: non-triangular face with 4 vertices"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 a 3\n", "line 4: bad face index 'a'"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n", "line 4: face indices must be positive"),
    ("v 0 0 0\n", "no faces"),
])
def test_errors_name_the_line(tmp_path, body, msg):
    mg = _mg()
    p = tmp_path / "bad.obj"
    p.write_text(body)
    with pytest.raises(mg.MeshError, match=msg):
        mg.load_obj(p)
