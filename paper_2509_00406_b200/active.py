"""Scalar-type-generic containers and elementary functions for term formulas.

The reference writes per-element energies as Python expressions over
`ActiveVec` / `SmallMatrix` of `ActiveScalar`s (`meshgrad/active.py:345-487`).
On this engine the *device* evaluates the builtin terms with CUDA dual numbers
(`csrc/dual.cuh`); the Python formulas below exist so a builtin term can also
be run by any scalar type that supplies the arithmetic protocol (the test
oracle's CPU duals, plain floats / numpy arrays for spot checks).

Nothing in this module differentiates anything: containers forward `+ - * /`
to their components and the elementary functions dispatch to a hook method on
the scalar type (`_mg_sqrt`, `_mg_log`, ...), falling back to numpy for plain
numbers. The reference dispatches the same functions on
`isinstance(a, ActiveScalar)` (`active.py:261-316`); a hook keeps the formulas
independent of any one scalar implementation.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "ActiveVec",
    "SmallMatrix",
    "abs_",
    "cos",
    "exp",
    "log",
    "positive_guard",
    "sin",
    "sqrt",
]


def _dispatch(name, fallback):
    hook = "_mg_" + name

    def fn(a):
        method = getattr(type(a), hook, None)
        if method is not None:
            return method(a)
        return fallback(a)

    fn.__name__ = name
    fn.__doc__ = f"{name}(a): elementwise; scalar types provide `{hook}` (ref active.py:261-316)."
    return fn


sqrt = _dispatch("sqrt", np.sqrt)
log = _dispatch("log", np.log)
exp = _dispatch("exp", np.exp)
sin = _dispatch("sin", np.sin)
cos = _dispatch("cos", np.cos)
abs_ = _dispatch("abs", np.abs)


def _guard_plain(a):
    a = np.asarray(a, dtype=np.float64)
    return np.where(a > 0.0, a, np.nan)


positive_guard = _dispatch("positive_guard", _guard_plain)
positive_guard.__doc__ = (
    "NaN the lanes whose value is not strictly positive; derivatives untouched "
    "(ref active.py:319-327)."
)


class ActiveVec:
    """Fixed-length vector of scalars (ref `ActiveVec`, active.py:345-416).

    Operands that are not ActiveVec are per-component arrays with the component
    on the last axis (a per-element closure array such as `target[v.index]`)."""

    __slots__ = ("comps",)
    __array_ufunc__ = None

    def __init__(self, comps):
        self.comps = tuple(comps)

    def __len__(self):
        return len(self.comps)

    def __iter__(self):
        return iter(self.comps)

    def __getitem__(self, i):
        return self.comps[i]

    def _rhs(self, other, i):
        if isinstance(other, ActiveVec):
            return other.comps[i]
        return np.asarray(other)[..., i]

    def __add__(self, other):
        return ActiveVec([c + self._rhs(other, i) for i, c in enumerate(self.comps)])

    __radd__ = __add__

    def __sub__(self, other):
        return ActiveVec([c - self._rhs(other, i) for i, c in enumerate(self.comps)])

    def __rsub__(self, other):
        return ActiveVec([self._rhs(other, i) - c for i, c in enumerate(self.comps)])

    def __neg__(self):
        return ActiveVec([-c for c in self.comps])

    def __mul__(self, s):
        return ActiveVec([c * s for c in self.comps])

    __rmul__ = __mul__

    def __truediv__(self, s):
        return ActiveVec([c / s for c in self.comps])

    def dot(self, other):
        acc = self.comps[0] * self._rhs(other, 0)
        for i in range(1, len(self.comps)):
            acc = acc + self.comps[i] * self._rhs(other, i)
        return acc

    def norm2(self):
        acc = self.comps[0] * self.comps[0]
        for c in self.comps[1:]:
            acc = acc + c * c
        return acc

    def norm(self):
        return sqrt(self.norm2())

    def normalized(self):
        return self / self.norm()

    def cross(self, other):
        if len(self.comps) != 3:
            raise ValueError("cross product needs 3-D vectors")
        a0, a1, a2 = self.comps
        b0, b1, b2 = (self._rhs(other, i) for i in range(3))
        return ActiveVec([a1 * b2 - a2 * b1, a2 * b0 - a0 * b2, a0 * b1 - a1 * b0])


class SmallMatrix:
    """2x2 / 3x3 matrix of scalars (ref `SmallMatrix`, active.py:419-487)."""

    __slots__ = ("rows",)
    __array_ufunc__ = None

    def __init__(self, rows):
        rows = [list(r) for r in rows]
        if len(rows) not in (2, 3) or any(len(r) != len(rows) for r in rows):
            raise ValueError("SmallMatrix must be 2x2 or 3x3")
        self.rows = rows

    @classmethod
    def from_columns(cls, *cols):
        n = len(cols)
        return cls([[cols[j][i] for j in range(n)] for i in range(n)])

    @property
    def dim(self):
        return len(self.rows)

    def __getitem__(self, ij):
        return self.rows[ij[0]][ij[1]]

    def det(self):
        m = self.rows
        if self.dim == 2:
            return m[0][0] * m[1][1] - m[0][1] * m[1][0]
        minor0 = m[1][1] * m[2][2] - m[1][2] * m[2][1]
        minor1 = m[1][0] * m[2][2] - m[1][2] * m[2][0]
        minor2 = m[1][0] * m[2][1] - m[1][1] * m[2][0]
        return m[0][0] * minor0 - m[0][1] * minor1 + m[0][2] * minor2

    def inverse(self):
        if self.dim != 2:
            raise ValueError("inverse is implemented for 2x2 matrices only")
        d = self.det()
        m = self.rows
        return SmallMatrix([[m[1][1] / d, -m[0][1] / d], [-m[1][0] / d, m[0][0] / d]])

    def frobenius2(self):
        acc = 0.0
        for row in self.rows:
            for e in row:
                acc = e * e + acc
        return acc

    def __matmul__(self, other):
        n = self.dim
        if isinstance(other, SmallMatrix):
            if other.dim != n:
                raise ValueError("dimension mismatch")
            entry = lambda i, j: other.rows[i][j]
        else:
            arr = np.asarray(other)
            entry = lambda i, j: arr[..., i, j]
        out = []
        for i in range(n):
            row = []
            for j in range(n):
                acc = self.rows[i][0] * entry(0, j)
                for k in range(1, n):
                    acc = acc + self.rows[i][k] * entry(k, j)
                row.append(acc)
            out.append(row)
        return SmallMatrix(out)
