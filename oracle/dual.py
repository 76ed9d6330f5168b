"""Batched second-order forward-mode scalar (oracle restatement of
meshgrad/active.py:43-327).

Encoding of the three fields, as in the reference (active.py:8-13):
  jac is None            passive constant
  hes is None            first-order only
  hes is the float 0.0   second order, Hessian structurally zero
  hes ndarray (..., K, K) dense symmetric Hessian
Every rule below states which reference lines it restates; the arithmetic
order matches so the oracle reproduces the reference to the last bit on the
golden vectors wherever summation order does not intervene.
"""

from __future__ import annotations

import numpy as np


def _c1(s):
    """per-lane factor shaped for a gradient (active.py:43-45)"""
    return s[..., None] if np.ndim(s) else s


def _c2(s):
    """per-lane factor shaped for a Hessian (active.py:48-50)"""
    return s[..., None, None] if np.ndim(s) else s


def _is_arr(h):
    return isinstance(h, np.ndarray)


def _h_times(h, s):
    return h * _c2(s) if _is_arr(h) else h


def _h_plus(a, b, sign=1.0):
    """_h_add / _h_sub (active.py:62-93): structural zeros and None pass
    through without touching the other operand."""
    if _is_arr(a) and _is_arr(b):
        return a + b if sign > 0 else a - b
    if _is_arr(a):
        return a
    if _is_arr(b):
        return b if sign > 0 else -b
    if a is None and b is None:
        return None
    return 0.0


def _h_negate(h):
    return -h if _is_arr(h) else h


def _sym_outer(x, y):
    """x y^T + y x^T, bitwise symmetric (active.py:96-99)"""
    return x[..., :, None] * y[..., None, :] + y[..., :, None] * x[..., None, :]


def _self_outer(g):
    return g[..., :, None] * g[..., None, :]


class Dual:
    __slots__ = ("val", "jac", "hes")
    __array_ufunc__ = None

    def __init__(self, val, jac=None, hes=None):
        self.val = val
        self.jac = jac
        self.hes = hes

    # reference-compatible field names (positive_guard-style code reads these)
    @property
    def value(self):
        return self.val

    @property
    def grad(self):
        return self.jac

    @property
    def hess(self):
        return self.hes

    # --- sums (active.py:124-154)
    def __add__(self, o):
        if not isinstance(o, Dual):
            return Dual(self.val + o, self.jac, self.hes)
        v = self.val + o.val
        if self.jac is None:
            return Dual(v, o.jac, o.hes)
        if o.jac is None:
            return Dual(v, self.jac, self.hes)
        return Dual(v, self.jac + o.jac, _h_plus(self.hes, o.hes))

    __radd__ = __add__

    def __sub__(self, o):
        if not isinstance(o, Dual):
            return Dual(self.val - o, self.jac, self.hes)
        v = self.val - o.val
        if o.jac is None:
            return Dual(v, self.jac, self.hes)
        if self.jac is None:
            return Dual(v, -o.jac, _h_negate(o.hes))
        return Dual(v, self.jac - o.jac, _h_plus(self.hes, o.hes, -1.0))

    def __rsub__(self, o):
        if self.jac is None:
            return Dual(o - self.val)
        return Dual(o - self.val, -self.jac, _h_negate(self.hes))

    def __neg__(self):
        if self.jac is None:
            return Dual(-self.val)
        return Dual(-self.val, -self.jac, _h_negate(self.hes))

    # --- products (active.py:156-178)
    def __mul__(self, o):
        if not isinstance(o, Dual):
            if self.jac is None:
                return Dual(self.val * o)
            return Dual(self.val * o, self.jac * _c1(o), _h_times(self.hes, o))
        av, bv = self.val, o.val
        v = av * bv
        if o.jac is None:
            if self.jac is None:
                return Dual(v)
            return Dual(v, self.jac * _c1(bv), _h_times(self.hes, bv))
        if self.jac is None:
            return Dual(v, o.jac * _c1(av), _h_times(o.hes, av))
        g = self.jac * _c1(bv) + o.jac * _c1(av)
        if self.hes is None and o.hes is None:
            return Dual(v, g)
        h = _h_plus(_h_plus(_h_times(self.hes, bv), _h_times(o.hes, av)), _sym_outer(self.jac, o.jac))
        return Dual(v, g, h)

    __rmul__ = __mul__

    # --- quotients (active.py:180-221)
    def __truediv__(self, o):
        if not isinstance(o, Dual):
            with np.errstate(divide="ignore", invalid="ignore"):
                u = np.divide(1.0, o)
            if self.jac is None:
                return Dual(self.val * u)
            return Dual(self.val * u, self.jac * _c1(u), _h_times(self.hes, u))
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            u = np.divide(1.0, o.val)
            v = self.val * u
            if o.jac is None:
                if self.jac is None:
                    return Dual(v)
                return Dual(v, self.jac * _c1(u), _h_times(self.hes, u))
            if self.jac is None:
                return _recip_rule(o, v, u)
            g = (self.jac - _c1(v) * o.jac) * _c1(u)
            if self.hes is None and o.hes is None:
                return Dual(v, g)
            first = _h_plus(_h_times(self.hes, u), _h_times(o.hes, -v * u))
            second = _sym_outer(self.jac, o.jac) * _c2(-u * u) + _self_outer(o.jac) * _c2(2.0 * v * u * u)
            return Dual(v, g, _h_plus(first, second))

    def __rtruediv__(self, o):
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            u = np.divide(1.0, self.val)
            v = o * u
            if self.jac is None:
                return Dual(v)
            return _recip_rule(self, v, u)

    # --- integer powers and abs (active.py:225-249)
    def __pow__(self, p):
        if not isinstance(p, (int, np.integer)):
            raise TypeError("only integer exponents are supported")
        if p == 0:
            return Dual(np.ones_like(np.asarray(self.val, dtype=float)))
        if p == 1:
            return self
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            x = self.val
            f0 = x ** p
            if self.jac is None:
                return Dual(f0)
            f1 = p * x ** (p - 1)
            f2 = p * (p - 1) * x ** (p - 2) if self.hes is not None else None
            return _unary(self, f0, f1, f2)

    def __abs__(self):
        sg = np.sign(self.val)
        if self.jac is None:
            return Dual(np.abs(self.val))
        return Dual(np.abs(self.val), self.jac * _c1(sg), _h_times(self.hes, sg))

    # --- elementary-function hooks (active.py:261-327), see active.py dispatch
    def _mg_sqrt(self):
        with np.errstate(invalid="ignore", divide="ignore"):
            f0 = np.sqrt(self.val)
            if self.jac is None:
                return Dual(f0)
            f1 = 0.5 / f0
            f2 = None if self.hes is None else -0.5 * f1 / self.val
            return _unary(self, f0, f1, f2)

    def _mg_log(self):
        with np.errstate(invalid="ignore", divide="ignore"):
            f0 = np.log(self.val)
            if self.jac is None:
                return Dual(f0)
            f1 = 1.0 / self.val
            f2 = None if self.hes is None else -f1 * f1
            return _unary(self, f0, f1, f2)

    def _mg_exp(self):
        with np.errstate(over="ignore"):
            f0 = np.exp(self.val)
            if self.jac is None:
                return Dual(f0)
            return _unary(self, f0, f0, f0)

    def _mg_sin(self):
        f0 = np.sin(self.val)
        if self.jac is None:
            return Dual(f0)
        return _unary(self, f0, np.cos(self.val), -f0)

    def _mg_cos(self):
        f0 = np.cos(self.val)
        if self.jac is None:
            return Dual(f0)
        return _unary(self, f0, -np.sin(self.val), -f0)

    def _mg_abs(self):
        return abs(self)

    def _mg_positive_guard(self):
        return Dual(np.where(np.asarray(self.val) > 0.0, self.val, np.nan), self.jac, self.hes)


def _recip_rule(b: Dual, v, u):
    """c / b with passive c: v = c*u, u = 1/b (active.py:190-194, 207-221)"""
    g = b.jac * _c1(-v * u)
    if b.hes is None:
        return Dual(v, g)
    return Dual(v, g, _h_plus(_h_times(b.hes, -v * u), _self_outer(b.jac) * _c2(2.0 * v * u * u)))


def _unary(a: Dual, f0, f1, f2):
    """chain rule (active.py:252-258)"""
    g = a.jac * _c1(f1)
    if a.hes is None:
        return Dual(f0, g)
    return Dual(f0, g, _h_plus(_h_times(a.hes, f1), _self_outer(a.jac) * _c2(f2)))


def lift_values(values, with_hessian: bool = True):
    """Seed K variables e_i (active.py:330-342)."""
    values = np.asarray(values, dtype=np.float64)
    k = values.size
    return [Dual(values[i], np.eye(k)[i].copy(), 0.0 if with_hessian else None) for i in range(k)]


def project_psd(h, floor: float) -> np.ndarray:
    """eigh -> clamp -> recompose -> symmetrise (active.py:490-504)."""
    if floor <= 0:
        raise ValueError("floor must be positive")
    h = np.asarray(h, dtype=np.float64)
    w, q = np.linalg.eigh(h)
    w = np.maximum(w, floor)
    out = np.einsum("...ij,...j,...kj->...ik", q, w, q)
    return 0.5 * (out + np.swapaxes(out, -1, -2))
