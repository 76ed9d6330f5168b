"""Tracer + CUDA code generation for arbitrary energy callbacks.

The reference's programming model is a Python callback `fn(handle, nbrs, x)`
over batched `ActiveVec` / `SmallMatrix` values (problem.py:8-14, 440-452).
Here such a callback is run ONCE with symbolic scalars:

  * `x[nbr]` yields an ActiveVec of input variables (slot q, component c);
  * `handle.index` is the real array of element ids, so closure gathers like
    `rest2[edge.index]` evaluate to (M,) / (M, k) numpy arrays; every such
    array meeting a symbolic scalar becomes a per-element *attribute stream*
    (uploaded to the device, read by element id);
  * scalars and 0-d arrays are constants (emitted as exact hex literals);
  * `+ - * /`, unary `-`, integer `**`, `abs` and the module functions
    `sqrt log exp sin cos abs_ positive_guard` are recorded in call order.

The recorded SSA is emitted as a C++ functor over the engine's dual numbers
(csrc/dual.cuh) — the same operation order as the callback, so each mode
rounds like the reference's ActiveScalar — and compiled with nvcc for sm_100a
into a cubin (cached by source hash), which the library loads through the
driver API (`mg_problem_add_jit_term`). The callback must be a pure function
of its inputs (the reference asks the same, problem.py:8-14) and must not
branch on input values.
"""

from __future__ import annotations

import hashlib
import os
import re
import subprocess
from pathlib import Path

import numpy as np

CSRC = Path(__file__).resolve().parent / "csrc"
CACHE = Path(os.environ.get("MG_JIT_CACHE", str(Path(__file__).resolve().parent / "jit_cache")))

__all__ = ["TracedTerm", "trace_callback", "compile_term"]


class _Graph:
    def __init__(self, num_elements):
        self.M = num_elements
        self.lines = []
        self.ops = []  # (name, kind, operand expressions) per line, for structure analysis
        self.attrs = []  # (M,) float64 arrays
        self._attr_ids = {}
        self._pins = []  # keep operand objects alive so their ids stay unique
        self.count = 0

    def new(self, expr, kind="?", args=()):
        name = f"t{self.count}"
        self.count += 1
        self.lines.append(f"auto {name} = {expr};")
        self.ops.append((name, kind, tuple(args)))
        return Sym(self, name)

    def operand(self, v):
        """C++ expression of an operand (symbol, constant or attribute stream)."""
        if isinstance(v, Sym):
            if v.g is not self:
                raise ValueError("symbols from different traces")
            return v.name
        a = np.asarray(v)
        if a.dtype == bool:
            a = a.astype(np.float64)
        per_element = a.ndim == 1 and a.shape[0] == self.M
        if not per_element and (a.ndim == 0 or a.size == 1):  # with M == 1 a (1,) array is still a stream
            return _lit(float(a.reshape(-1)[0]))
        if per_element:
            # the same memory (also different views of it) is one stream
            key = None
            if isinstance(v, np.ndarray):
                key = (v.__array_interface__["data"][0], v.strides, v.shape, v.dtype.str)
            if key is not None and key in self._attr_ids:
                k = self._attr_ids[key]
            else:
                k = len(self.attrs)
                self.attrs.append(np.ascontiguousarray(a, dtype=np.float64))
                if key is not None:
                    self._attr_ids[key] = k
                    self._pins.append(v)
            return f"A[{k}][e]"
        raise ValueError(f"per-element operand must have shape ({self.M},) after indexing, got {a.shape}")


def _lit(x: float) -> str:
    if np.isnan(x):
        return "mg::nan_d()"
    if np.isinf(x):
        return "(1.0 / 0.0)" if x > 0 else "(-1.0 / 0.0)"
    return f"{float(x).hex()}"


class Sym:
    """Symbolic scalar with the reference ActiveScalar's arithmetic protocol."""

    __slots__ = ("g", "name")
    __array_ufunc__ = None  # numpy defers to our reflected operators

    def __init__(self, g, name):
        self.g = g
        self.name = name

    def _bin(self, other, fmt, kind, reflect=False):
        a, b = self.g.operand(self), self.g.operand(other)
        if reflect:
            a, b = b, a
        return self.g.new(fmt.format(a=a, b=b), kind, (a, b))

    def __add__(self, o):
        return self._bin(o, "{a} + {b}", "add")

    def __radd__(self, o):
        return self._bin(o, "{a} + {b}", "add", reflect=True)

    def __sub__(self, o):
        return self._bin(o, "{a} - {b}", "sub")

    def __rsub__(self, o):
        return self._bin(o, "{a} - {b}", "sub", reflect=True)

    def __mul__(self, o):
        return self._bin(o, "{a} * {b}", "mul")

    def __rmul__(self, o):
        return self._bin(o, "{a} * {b}", "mul", reflect=True)

    def __truediv__(self, o):
        return self._bin(o, "{a} / {b}", "div")

    def __rtruediv__(self, o):
        return self._bin(o, "{a} / {b}", "div", reflect=True)

    def __neg__(self):
        return self.g.new(f"-{self.name}", "neg", (self.name,))

    def __pos__(self):
        return self

    def __pow__(self, p):
        if not isinstance(p, (int, np.integer)):
            raise TypeError("only integer exponents are supported")  # active.py:225-227
        if p == 1:
            return self
        return self.g.new(f"mg::powi({self.name}, {int(p)})", "powi", (self.name,))

    def __abs__(self):
        return self.g.new(f"mg::abs_({self.name})", "abs", (self.name,))

    # elementary-function hooks (paper_2509_00406_b200.active dispatch)
    def _mg_sqrt(self):
        return self.g.new(f"sqrt({self.name})", "sqrt", (self.name,))

    def _mg_log(self):
        return self.g.new(f"log({self.name})", "log", (self.name,))

    def _mg_exp(self):
        return self.g.new(f"exp({self.name})", "exp", (self.name,))

    def _mg_sin(self):
        return self.g.new(f"sin({self.name})", "sin", (self.name,))

    def _mg_cos(self):
        return self.g.new(f"cos({self.name})", "cos", (self.name,))

    def _mg_abs(self):
        return self.__abs__()

    def _mg_positive_guard(self):
        return self.g.new(f"positive_guard({self.name})", "guard", (self.name,))

    def __bool__(self):
        raise TypeError("traced callbacks cannot branch on input values")

    def __float__(self):
        raise TypeError("traced callbacks cannot convert inputs to float")


class _Handle:
    __slots__ = ("kind", "index", "slot")

    def __init__(self, kind, index, slot=None):
        self.kind = kind
        self.index = index
        self.slot = slot


class _Vars:
    def __init__(self, vecs):
        self.vecs = vecs

    def __getitem__(self, h):
        if getattr(h, "slot", None) is None:
            raise KeyError("this handle carries no variables")
        return self.vecs[h.slot]


class TracedTerm:
    """Result of tracing: C++ body, attribute streams, shape."""

    def __init__(self, op: str, P: int, n: int, body: list, ret: str, attrs: list, ops: list | None = None):
        self.op, self.P, self.n = op, P, n
        self.body, self.ret, self.attrs = body, ret, attrs
        self.ops = ops or []

    def functor(self, name: str = "Traced") -> str:
        """The recorded SSA as a C++ functor over the engine's duals."""
        lines = "\n      ".join(self.body)
        return f"""struct {name} {{
  template <int N, class S>
  MG_DI auto operator()(const double* const* A, int64_t e, const mg::Vec<S, N>* X) const {{
      using namespace mg;
      (void)A; (void)e;
      {lines}
      return {self.ret};
  }}
}};"""

    def source(self) -> str:
        return f"""// generated by paper_2509_00406_b200/jit.py — traced energy callback
#include "jit_kernel.cuh"

namespace {{
{self.functor()}
}}  // namespace

MG_JIT_INSTANTIATE(Traced, {self.P}, {self.n})
"""


def patch_source(terms: list, n: int) -> str:
    """One module for a problem's traced terms on the patch-owner path
    (csrc/jit_patch.cuh): a functor per term and a policy that runs the V
    terms, then the EV / FV terms, in registration order (like the builtin
    patch kernel), each with its own attribute streams (a.jattr + t * 64)."""
    funcs = "\n".join(t.functor(f"T{i}") for i, t in enumerate(terms))
    vt, et = [], []
    for i, t in enumerate(terms):
        ev = f"mg::patch::JitEval<T{i}, N>{{a.jattr + {i} * mg::patch::JATTR}}"
        if t.op == "V":
            vt.append(f"mg::patch::run_vterm_g<N, MODE, PSD>(a, {ev}, s, oc, eacc);")
        elif t.op in ("EV", "FV"):
            lay = "a.ev" if t.op == "EV" else "a.fv"
            et.append(f"mg::patch::run_eterm_g<{t.P}, N, MODE, PSD>(a, {ev}, {lay}, p, s, oc, eacc);")
        else:
            raise ValueError("patch modules take V / EV / FV traced terms")
    j = "\n    "
    return f"""// generated by paper_2509_00406_b200/jit.py — a problem's traced terms on the patch path
#include "jit_patch.cuh"

namespace {{
{funcs}

struct Policy {{
  template <int N, int MODE, bool PSD>
  MG_DI static void vterms(const mg::patch::PatchArgs& a, const mg::patch::Smem& s, int oc, double& eacc) {{
    (void)a; (void)s; (void)oc; (void)eacc;
    {j.join(vt)}
  }}
  template <int N, int MODE, bool PSD>
  MG_DI static void eterms(const mg::patch::PatchArgs& a, int p, const mg::patch::Smem& s, int oc, double& eacc) {{
    (void)a; (void)p; (void)s; (void)oc; (void)eacc;
    {j.join(et)}
  }}
}};
}}  // namespace

MG_PATCH_JIT_INSTANTIATE(Policy, {n})
"""


_XIN = re.compile(r"^X\[(\d+)\]\[(\d+)\]$")
_ATTR = re.compile(r"A\[(\d+)\]\[e\]")


def _radial(tt: TracedTerm, dsym_of):
    """Shared proof of radial structure (radial_form / radial_vform).
    dsym_of(kind, args) -> (component, sign, C++ expression of d_c) for an
    operation that forms a difference component, None for one that uses the
    inputs otherwise (then the term is not radial), or False when the
    operation does not read an input directly."""
    n = tt.n
    full = tuple(range(n))
    xdep, dsym, sq, post = set(), {}, {}, set()
    dexpr = {}
    r_name = None
    for name, kind, args in tt.ops:
        direct = any(_XIN.match(o) for o in args)
        dep = [o for o in args if _XIN.match(o) or o in xdep]
        if not dep:
            continue
        xdep.add(name)
        if direct:
            got = dsym_of(kind, args)
            if not got:
                return None
            c, sign, expr = got
            dsym[name] = (c, sign)
            dexpr.setdefault(c, expr)
            continue
        if kind == "mul" and len(args) == 2 and args[0] in dsym and args[1] in dsym:
            (ca, sa), (cb, sb) = dsym[args[0]], dsym[args[1]]
            if ca != cb or sa != sb:
                return None
            sq[name] = (ca,)
            continue
        if kind == "add" and len(args) == 2 and args[0] in sq and args[1] in sq:
            comps = tuple(sorted(sq[args[0]] + sq[args[1]]))
            if len(set(comps)) != len(comps):
                return None
            sq[name] = comps
            continue
        for o in dep:  # beyond the quadratic form: inputs only through r
            if o in post:
                continue
            if sq.get(o) == full and (r_name is None or r_name == o):
                r_name = o
                continue
            return None
        post.add(name)
    ret = tt.ret
    if r_name is None:
        if sq.get(ret) != full:  # e.g. the energy |d|^2 itself
            return None
        r_name = ret
    elif ret not in post and ret != r_name:
        return None
    lines = [f"auto {r_name} = R;"] + [ln for (nm, _, _), ln in zip(tt.ops, tt.body) if nm in post]
    return r_name, lines, [dexpr[c] for c in full] if set(dexpr) == set(full) else None


def radial_form(tt: TracedTerm):
    """Prove that an EV callback depends on its vertex positions only through
    r = |x_0 - x_1|^2, from the recorded operations: every use of an input
    is a component difference d_c = x_0[c] - x_1[c] (either orientation),
    those are only squared (d_c * d_c, equal signs) and the squares only
    summed until one symbol r holds each component's square exactly once
    (ActiveVec.norm2 / dot, active.py); every later operation reaches the
    inputs only through r. Returns (r name, [phi lines]) — the operations
    after r, in order, with r bound to the input R — or None.
    (The reference's K = 2n duals of such a term give gradient 2 phi' d and
    Hessian blocks +-(2 phi' I + 4 phi'' d d^T): jit_rows.cuh.)"""
    if tt.op != "EV" or tt.P != 2 or not tt.ops or len(tt.ops) != len(tt.body):
        return None

    def dsym_of(kind, args):
        xin = [_XIN.match(o) for o in args]
        if kind != "sub" or len(args) != 2 or not all(xin):
            return None
        (q0, c0), (q1, c1) = [(int(m.group(1)), int(m.group(2))) for m in xin]
        if c0 != c1 or {q0, q1} != {0, 1}:
            return None
        return c0, 1 if q0 == 0 else -1, ""

    rf = _radial(tt, dsym_of)
    return None if rf is None else (rf[0], rf[1])


def radial_vform(tt: TracedTerm):
    """The same proof for a V callback: the inputs enter only as differences
    d_c = x[c] - t_c with t_c an attribute stream or a constant (either
    orientation; inertia 0.5 m |x - t|^2, apps/cloth.py:102-104), squared and
    summed into r. Returns (r name, [phi lines], [C++ d_c over x[], av[]]) or
    None."""
    if tt.op != "V" or not tt.ops or len(tt.ops) != len(tt.body):
        return None

    def dsym_of(kind, args):
        if kind != "sub" or len(args) != 2:
            return None
        xin = [_XIN.match(o) for o in args]
        if all(xin) or not any(xin):
            return None
        k = 0 if xin[0] else 1
        c = int(xin[k].group(2))
        other = _preloaded(args[1 - k])
        expr = f"x[{c}] - {other}" if k == 0 else f"{other} - x[{c}]"
        return c, 1 if k == 0 else -1, expr

    rf = _radial(tt, dsym_of)
    if rf is None or rf[2] is None:
        return None
    return rf


def _preloaded(text: str) -> str:
    """Attribute-stream reads A[k][e] -> av[k] (values loaded ahead, jit_rows.cuh)."""
    return _ATTR.sub(r"av[\1]", text)


def rows_source(terms: list, n: int) -> str | None:
    """One module for a problem's traced terms on the edge row kernel
    (csrc/jit_rows.cuh), or None unless every term is a V term or an EV term
    radial_form proves radial (and at least one is EV). Attribute streams of
    all terms, in term order, are EvArgs::js; each term's are preloaded into
    av (V terms: per row; EV terms: per incidence, with the gathers)."""
    if not terms or any(t.op not in ("V", "EV") for t in terms) or not any(t.op == "EV" for t in terms):
        return None
    funcs, vcalls, ecalls, vloads, eloads = [], [], [], [], []
    js = nv = ne = 0
    for i, t in enumerate(terms):
        k = len(t.attrs)
        ret = _preloaded(t.ret)
        rv = radial_vform(t) if t.op == "V" else None
        if rv is not None:
            body = "\n      ".join(_preloaded(ln) for ln in rv[1])
            dlines = "\n    ".join(f"d[{c}] = {e};" for c, e in enumerate(rv[2]))
            funcs.append(f"""struct V{i} {{
  template <class S>
  MG_DI auto operator()(const double* av, const S& R) const {{
      using namespace mg;
      (void)av;
      {body}
      return {ret};
  }}
  MG_DI static void dvec(const double* av, const double* x, double* d) {{
    (void)av;
    {dlines}
  }}
}};""")
            vloads += [f"p.v[{nv + j}] = a.js[{js + j}][g];" for j in range(k)]
            vcalls.append(f"{{ double d[N]; V{i}::dvec(p.v + {nv}, xs, d); "
                          f"mg::rows::jit_vradial<N, MODE, PSD>(V{i}{{}}, p.v + {nv}, d, us, a.floor, eacc, vec, dg, "
                          f"finite); }}")
            nv += k
        elif t.op == "V":
            body = "\n      ".join(_preloaded(ln) for ln in t.body)
            funcs.append(f"""struct V{i} {{
  template <int N, class S>
  MG_DI auto operator()(const double* av, const mg::Vec<S, N>* X) const {{
      using namespace mg;
      (void)av;
      {body}
      return {ret};
  }}
}};""")
            vloads += [f"p.v[{nv + j}] = a.js[{js + j}][g];" for j in range(k)]
            vcalls.append(f"mg::rows::jit_vterm<N, MODE, PSD>(V{i}{{}}, p.v + {nv}, fr, xs, us, a.floor, eacc, vec, dg);")
            nv += k
        else:
            rf = radial_form(t)
            if rf is None:
                return None
            body = "\n      ".join(_preloaded(ln) for ln in rf[1])
            funcs.append(f"""struct E{i} {{
  template <class S>
  MG_DI auto operator()(const double* av, const S& R) const {{
      using namespace mg;
      (void)av;
      {body}
      return {ret};
  }}
}};""")
            eloads += [f"p.v[{ne + j}] = a.js[{js + j}][e];" for j in range(k)]
            ecalls.append(f"mg::rows::jit_radial<MODE, NEEDV>(E{i}{{}}, p.v + {ne}, rr, one);")
            ne += k
        js += k
    if js > 24:  # rows::MAX_JS
        return None
    j = "\n    "
    return f"""// generated by paper_2509_00406_b200/jit.py — a problem's traced terms on the edge row kernel
#include "jit_rows.cuh"

namespace {{
{chr(10).join(funcs)}

struct Pol {{
  static constexpr bool kXFreeHvp = false;
  static constexpr bool kVertexOnly = {"true" if ne == 0 else "false"};
  using Store = double;
  template <int N, int MODE>
  MG_DI static mg::rows::JPre<{nv}> vload(const mg::rows::EvArgs& a, int g) {{
    mg::rows::JPre<{nv}> p;
    (void)a; (void)g;
    {j.join(vloads)}
    return p;
  }}
  template <int N, int MODE, bool PSD>
  MG_DI static void vterms(const mg::rows::EvArgs& a, int g, bool fr, const mg::rows::JPre<{nv}>& p, const double* xs,
                           const double* us, double& eacc, double* vec, double* dg, bool& finite) {{
    (void)a; (void)g; (void)fr; (void)p; (void)xs; (void)us; (void)eacc; (void)vec; (void)dg; (void)finite;
    {j.join(vcalls)}
  }}
  template <int MODE>
  MG_DI static mg::rows::JPre<{ne}> eload(const mg::rows::EvArgs& a, uint32_t e) {{
    mg::rows::JPre<{ne}> p;
    (void)a; (void)e;
    {j.join(eloads)}
    return p;
  }}
  template <int MODE, bool NEEDV, class F>
  MG_DI static void eterms(const mg::rows::EvArgs& a, const mg::rows::JPre<{ne}>& p, double rr, uint32_t e, F&& one) {{
    (void)a; (void)e;
    {j.join(ecalls)}
  }}
}};
}}  // namespace

MG_ROWS_JIT_INSTANTIATE(Pol, {n})
"""


def trace_callback(fn, op: str, n: int, num_elements: int, sel=None, index=None) -> TracedTerm:
    """Run `fn(handle, nbrs, x)` once on symbolic inputs (ref problem.py:440-452).
    sel: (M, P) vertex ids of the elements (EV / FV / VV), so that a vertex
    batch's `index` holds the slot's vertex ids like the reference's `_Batch`.
    VV (one valence group): sel rows are the center then its one-ring, `index`
    the centers; the handle is the center (slot 0), nbrs the ring slots."""
    from .active import ActiveVec

    if op == "VV":
        if sel is None or index is None:
            raise ValueError("VV callbacks need the group's neighbourhoods and centers")
        P = int(np.asarray(sel).shape[1])
    else:
        P = {"V": 1, "EV": 2, "FV": 3}[op]
    g = _Graph(num_elements)
    index = np.arange(num_elements, dtype=np.int64) if index is None else np.asarray(index, dtype=np.int64)
    vecs = [ActiveVec([Sym(g, f"X[{q}][{c}]") for c in range(n)]) for q in range(P)]
    kind = {"V": "vertex", "VV": "vertex", "EV": "edge", "FV": "face"}[op]
    handle = _Handle(kind, index, slot=0 if op in ("V", "VV") else None)
    if op != "V" and sel is None:
        raise ValueError("edge / face callbacks need the element vertex lists")
    if op == "V":
        nbrs = (handle,)
    else:
        cols = [_Handle("vertex", np.ascontiguousarray(np.asarray(sel)[:, q], dtype=np.int64), slot=q) for q in range(P)]
        nbrs = tuple(cols[1:]) if op == "VV" else tuple(cols)
    out = fn(handle, nbrs, _Vars(vecs))
    if isinstance(out, Sym):
        ret = out.name
    else:
        ret = g.operand(out) if np.ndim(out) == 0 or np.size(out) == 1 else g.new(g.operand(out), "copy").name
    return TracedTerm(op, P, n, g.lines, ret, g.attrs, g.ops)


_NVCC_FLAGS = ["-cubin", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "--expt-relaxed-constexpr"]
_toolchain_key = None


def _toolchain() -> bytes:
    """Everything a cubin depends on besides the generated source: every
    header under csrc/ (jit_kernel.cuh includes dual.cuh, psd.cuh,
    psd_small.h, ...), the nvcc flags and the nvcc version."""
    global _toolchain_key
    if _toolchain_key is None:
        nvcc = os.environ.get("NVCC", "nvcc")
        try:
            ver = subprocess.run([nvcc, "--version"], capture_output=True, text=True).stdout
        except OSError:
            ver = "no-nvcc"
        parts = [nvcc.encode(), " ".join(_NVCC_FLAGS).encode(), ver.encode()]
        for hdr in sorted(list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))):
            parts += [hdr.name.encode(), hdr.read_bytes()]
        _toolchain_key = b"\0".join(parts)
    return _toolchain_key


def compile_term(tt: TracedTerm) -> bytes:
    """nvcc the traced functor into an sm_100a cubin (cached by source +
    toolchain hash; compiled under a per-process name, then renamed)."""
    return compile_source(tt.source())


def compile_patch(terms: list, n: int) -> bytes:
    """The patch-path module of a problem's traced terms (patch_source)."""
    return compile_source(patch_source(terms, n))


def compile_rows(terms: list, n: int) -> bytes | None:
    """The row-kernel module of a problem's traced terms (rows_source), or None."""
    src = rows_source(terms, n)
    return None if src is None else compile_source(src)


def compile_source(src: str) -> bytes:
    h = hashlib.sha256(src.encode() + _toolchain()).hexdigest()[:20]
    CACHE.mkdir(parents=True, exist_ok=True)
    cubin = CACHE / f"term_{h}.cubin"
    if not cubin.exists():
        tag = f"{os.getpid()}_{os.urandom(4).hex()}"
        cu = CACHE / f"term_{h}.{tag}.cu"
        tmp = CACHE / f"term_{h}.{tag}.cubin.tmp"
        cu.write_text(src)
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, *_NVCC_FLAGS, "-I", str(CSRC), "-o", str(tmp), str(cu)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for traced term:\n{r.stderr[-4000:]}")
        os.replace(tmp, cubin)
        os.replace(cu, CACHE / f"term_{h}.cu")
    return cubin.read_bytes()
