"""B200-native per-element forward-mode AD engine for triangle-mesh energies.

Drop-in for the hot path of the reference `meshgrad` package (arXiv
2509.00406): `Problem.eval_terms` (energy, gradient, block-CSR Hessian with
optional per-element PSD clamp), `hvp`, `eval_energy_only` and
`precompute_sparsity`, evaluated by hand-written sm_100a CUDA kernels behind
the C ABI in include/meshgrad_b200.h.
"""

from .active import ActiveVec, SmallMatrix, abs_, cos, exp, log, positive_guard, sin, sqrt
from .mesh import (
    DEFAULT_PATCH_TARGET,
    DEFAULT_VALENCE_CAP,
    Element,
    Mesh,
    MeshError,
    Op,
    SOURCE_KIND,
    generate_grid,
    generate_icosphere,
    grid_arrays,
    icosphere_arrays,
    load_obj,
    punctured_icosphere_arrays,
    save_obj,
)
from .problem import BlockSparseMatrix, Problem, read_matrix_market
from .terms import EdgeLength, Gravity, Inertia, SphereBarrierStretch, Spring, SymDirichlet

__version__ = "0.1.0"

__all__ = [
    "ActiveVec",
    "BlockSparseMatrix",
    "DEFAULT_PATCH_TARGET",
    "DEFAULT_VALENCE_CAP",
    "EdgeLength",
    "Element",
    "Gravity",
    "Inertia",
    "Mesh",
    "MeshError",
    "Op",
    "Problem",
    "SOURCE_KIND",
    "SmallMatrix",
    "SphereBarrierStretch",
    "Spring",
    "SymDirichlet",
    "abs_",
    "cos",
    "exp",
    "generate_grid",
    "generate_icosphere",
    "grid_arrays",
    "icosphere_arrays",
    "load_obj",
    "log",
    "positive_guard",
    "punctured_icosphere_arrays",
    "read_matrix_market",
    "save_obj",
    "sin",
    "sqrt",
]
