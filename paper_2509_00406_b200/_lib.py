"""ctypes binding of the C ABI in include/meshgrad_b200.h.

The shared library is built in-tree (csrc/Makefile -> libmeshgrad_b200.so).
There is no fallback: if the library or a CUDA device is missing, every call
that needs it raises `EngineUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "libmeshgrad_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

# enums (include/meshgrad_b200.h)
MG_OP = {"FV": 0, "EV": 1, "VV": 2, "V": 3}
MG_TERM_INERTIA = 1
MG_TERM_SPRING = 2
MG_TERM_GRAVITY = 3
MG_TERM_EDGE_LENGTH = 4
MG_TERM_SYM_DIRICHLET = 5
MG_TERM_SPHERE = 6
MG_TERM_JIT = 100

MG_ERR_VALUE = 1
MG_ERR_MESH = 2
MG_ERR_STATE = 3
MG_ERR_CUDA = 4
MG_ERR_UNSUPPORTED = 5

# every symbol the header declares: (name, restype, argtypes)
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I64P = ctypes.POINTER(ctypes.c_int64)
_INT = ctypes.c_int
_DBL = ctypes.c_double
SIGNATURES = [
    ("mg_last_error", ctypes.c_char_p, []),
    ("mg_abi_version", _INT, []),
    ("mg_mesh_create", _INT, [_P, _I64, _P, _I64, _I64, _P, _INT, _P, ctypes.POINTER(_P)]),
    ("mg_mesh_counts", _INT, [_P, _I64P, _I64P, _I64P, _I64P]),
    ("mg_mesh_copy_edges", _INT, [_P, _P, _P]),
    ("mg_mesh_copy_vertex_patches", _INT, [_P, _P, _P]),
    ("mg_mesh_set_owned", _INT, [_P, _P, _P]),
    ("mg_mesh_set_row_order", _INT, [_P, _INT, _P]),
    ("mg_mesh_row_order", _INT, [_P, ctypes.POINTER(_INT), ctypes.POINTER(ctypes.c_double)]),
    ("mg_mesh_destroy", _INT, [_P]),
    ("mg_problem_create", _INT, [_P, _INT, _INT, _P, _INT, ctypes.POINTER(_P)]),
    ("mg_problem_add_term", _INT, [_P, _INT, _INT, ctypes.POINTER(_DBL), _INT, ctypes.POINTER(_P), _INT,
                                   ctypes.POINTER(_INT)]),
    ("mg_problem_add_jit_term", _INT, [_P, _INT, _INT, _P, ctypes.POINTER(_P), _INT, ctypes.POINTER(_INT)]),
    ("mg_problem_add_jit_term_sel", _INT, [_P, _INT, _INT, _INT, _P, _I64, _P, ctypes.POINTER(_P), _INT,
                                            ctypes.POINTER(_INT)]),
    ("mg_problem_set_patch_module", _INT, [_P, _P]),
    ("mg_problem_set_row_module", _INT, [_P, _P]),
    ("mg_problem_set_storage", _INT, [_P, _INT]),
    ("mg_problem_set_jit_attr", _INT, [_P, _INT, _INT, _P]),
    ("mg_problem_set_attr", _INT, [_P, _INT, _INT, _P]),
    ("mg_precompute_sparsity", _INT, [_P, _I64P, _P]),
    ("mg_copy_pattern", _INT, [_P, _P, _P, _P]),
    ("mg_eval", _INT, [_P, _P, _INT, _DBL, _P, _P, _P, _P]),
    ("mg_energy", _INT, [_P, _P, _P, _P]),
    ("mg_hvp", _INT, [_P, _P, _P, _INT, _DBL, _P, _P]),
    ("mg_bsr_matvec", _INT, [_P, _P, _P, _P, _P]),
    ("mg_bsr_block_jacobi", _INT, [_P, _P, _P, _P]),
    ("mg_block_apply", _INT, [_P, _P, _P, _P, _P]),
    ("mg_pcg", _INT, [_P, _P, _P, _INT, _DBL, _P, _P, _DBL, _INT, _P, _P, _P, _P]),
    ("mg_problem_destroy", _INT, [_P]),
    ("mg_last_launch_count", _INT, [_P, ctypes.POINTER(_INT)]),
    ("mg_problem_patch_stats", _INT, [_P, _I64P]),
    ("mg_problem_set_timing", _INT, [_P, _INT]),
    ("mg_problem_exact_runs", _INT, [_P, _I64P]),
    ("mg_problem_kernel_time", _INT, [_P, ctypes.POINTER(_DBL), ctypes.POINTER(_INT)]),
]


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library not built or no GPU)."""


class EngineError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    if path is None and os.environ.get("MG_LIB"):
        path = os.environ["MG_LIB"]
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise EngineUnavailable(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_2509_00406_b200/csrc`)"
        )
    lib = ctypes.CDLL(str(p))
    for name, res, args in SIGNATURES:
        if path is not None and os.environ.get("MG_LIB") and not hasattr(lib, name):
            continue  # an A/B build of an older revision (tools/ab_*.sh) may lack newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Raise the Python exception the reference would raise for a status code."""
    if rc == 0:
        return
    msg = _lib.mg_last_error().decode() if _lib is not None else f"status {rc}"
    if rc in (MG_ERR_VALUE, MG_ERR_STATE):
        raise ValueError(msg)
    if rc == MG_ERR_MESH:
        from .mesh import MeshError

        raise MeshError(msg)
    if rc == MG_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise EngineError(rc, msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device: the meshgrad_b200 engine has no CPU fallback")
    return load()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
