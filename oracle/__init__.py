"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference `meshgrad` hot path
(/root/reference/pkg/src/meshgrad/active.py and problem.py), used as the
parity checker for the CUDA engine and as the CPU baseline in bench.py.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import it. The product package never does.

Parity status: PINNED. tests/golden/ holds vectors produced by running the
unmodified reference (tests/golden/make_golden.py, executed in the build
container where /root/reference exists); tests/test_oracle_golden.py checks
this oracle against every one of them.
"""

from .dual import Dual, lift_values
from .engine import OracleProblem, sparsity_pattern

__all__ = ["Dual", "OracleProblem", "lift_values", "sparsity_pattern"]
