"""The closed-form-seeded 2x2 / 3x3 spectral clamp (csrc/psd_small.h, used on
the device for vertex and two-point edge Hessians) against the reference's
eigh-based project_psd, on random, degenerate and near-floor spectra."""

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = tmp_path_factory.mktemp("psd") / "libpsd_small_host.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", str(HERE / "native" / "psd_small_host.cpp"),
                    "-o", str(out)], check=True)
    lib = ctypes.CDLL(str(out))
    for name in ("host_project3", "host_project2"):
        getattr(lib, name).argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_double]
    return lib


def ref_project(h, floor):
    w, q = np.linalg.eigh(h)
    w = np.maximum(w, floor)
    out = np.einsum("...ij,...j,...kj->...ik", q, w, q)
    return 0.5 * (out + np.swapaxes(out, -1, -2))


def pack(h):
    n = h.shape[-1]
    idx = [(i, j) for i in range(n) for j in range(i + 1)]
    return np.ascontiguousarray(np.stack([h[..., i, j] for i, j in idx], axis=-1))


def unpack(p, n):
    out = np.zeros(p.shape[:-1] + (n, n))
    k = 0
    for i in range(n):
        for j in range(i + 1):
            out[..., i, j] = out[..., j, i] = p[..., k]
            k += 1
    return out


def run(lib, h, floor):
    n = h.shape[-1]
    p = pack(h)
    fn = lib.host_project3 if n == 3 else lib.host_project2
    fn(p.ctypes.data, len(p), floor)
    return unpack(p, n)


def spectra(rng, n, m):
    q, _ = np.linalg.qr(rng.normal(size=(m, n, n)))
    cases = [rng.normal(size=(m, n)),                                   # generic
             np.repeat(rng.normal(size=(m, 1)), n, axis=1),             # fully degenerate
             np.concatenate([np.repeat(rng.normal(size=(m, 1)), n - 1, axis=1), rng.normal(size=(m, 1))], 1),
             np.concatenate([np.zeros((m, n - 1)), rng.normal(size=(m, 1))], 1),   # zero double root (rest springs)
             rng.normal(size=(m, n)) * 1e-9,                            # all near the floor
             rng.normal(size=(m, n)) * np.array([1.0] + [1e-12] * (n - 1))]
    out = []
    for w in cases:
        out.append(np.einsum("mij,mj,mkj->mik", q, w, q))
    return np.concatenate(out)


@pytest.mark.parametrize("n", [2, 3])
@pytest.mark.parametrize("floor", [1e-9, 1e-3])
def test_matches_eigh_projection(lib, n, floor):
    rng = np.random.default_rng(42 + n)
    h = spectra(rng, n, 400)
    h = 0.5 * (h + np.swapaxes(h, -1, -2))
    got = run(lib, h, floor)
    ref = ref_project(h, floor)
    scale = np.maximum(np.abs(h).max(axis=(1, 2)), floor)
    err = np.abs(got - ref).max(axis=(1, 2)) / scale
    assert err.max() <= 1e-12, err.max()


def test_spring_hessian_structure(lib):
    # 2A of a spring: 4cs I + 8c/l^2 d d^T, compressed (s<0) and at rest (s=0)
    rng = np.random.default_rng(7)
    d = rng.normal(size=(500, 3))
    s = np.concatenate([-np.abs(rng.normal(size=250)) * 1e-2, np.zeros(250)])
    c = 0.5
    h = 2 * (4 * c * s[:, None, None] * np.eye(3) + 8 * c * np.einsum("mi,mj->mij", d, d))
    got = run(lib, h, 1e-9)
    ref = ref_project(h, 1e-9)
    assert (np.abs(got - ref).max(axis=(1, 2)) / np.abs(h).max(axis=(1, 2))).max() <= 1e-12
