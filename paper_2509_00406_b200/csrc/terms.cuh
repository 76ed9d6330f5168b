// Builtin per-element energies, written once over a generic scalar S
// (Dv / Dg / Dh / Df from dual.cuh). Each body follows the reference
// callback's expression order so every mode rounds like the reference
// (the callbacks live in meshgrad/apps/*.py; file:line per term below).
#pragma once
#include "../../include/meshgrad_b200.h"
#include "dual.cuh"

namespace mg {

// Device-side view of one registered term.
struct TermDev {
  int type;
  int op;
  int P;   // vertices per element
  int pad;
  double c[6];          // scalar params
  const double* a[4];   // attribute arrays (device, caller-owned)
};

template <int TT> struct TermInfo;
template <> struct TermInfo<MG_TERM_INERTIA> { static constexpr int P = 1, OP = MG_OP_V; };
template <> struct TermInfo<MG_TERM_SPRING> { static constexpr int P = 2, OP = MG_OP_EV; };
template <> struct TermInfo<MG_TERM_GRAVITY> { static constexpr int P = 1, OP = MG_OP_V; };
template <> struct TermInfo<MG_TERM_EDGE_LENGTH> { static constexpr int P = 2, OP = MG_OP_EV; };
template <> struct TermInfo<MG_TERM_SYM_DIRICHLET> { static constexpr int P = 3, OP = MG_OP_FV; };
template <> struct TermInfo<MG_TERM_SPHERE> { static constexpr int P = 3, OP = MG_OP_FV; };

// Two-point difference terms: the energy depends on the edge only through
// d = x_i - x_j, so the 2n x 2n Hessian is exactly [[A, -A], [-A, A]] and the
// gradient is [g, -g]. Evaluating a K = n dual on d reproduces the K = 2n
// dual entry for entry: the reference's lifted d carries gradient e_c - e_{n+c},
// every later operation is entrywise, and the off-diagonal entries differ only
// by exact sign flips (active.py:156-258). Half the variables, a quarter of
// the Hessian work, and the PSD clamp reduces to an n x n eigenproblem.
template <int TT> struct TwoPoint { static constexpr bool value = false; };
template <> struct TwoPoint<MG_TERM_SPRING> { static constexpr bool value = true; };
template <> struct TwoPoint<MG_TERM_EDGE_LENGTH> { static constexpr bool value = true; };

// Radial two-point terms: E = phi(r) with r = |x_i - x_j|^2. The n x n block
// is then A = 2 phi'(r) I + 4 phi''(r) d d^T, so value, gradient and Hessian
// follow from a one-variable second-order dual on r, and the block's spectrum
// is known in closed form: 2 phi' (n-1 times, transverse) and
// 2 phi' + 4 phi'' r (along d). Results agree with the full dual to rounding.
template <int TT> struct Radial { static constexpr bool value = false; };
template <> struct Radial<MG_TERM_SPRING> { static constexpr bool value = true; };
template <> struct Radial<MG_TERM_EDGE_LENGTH> { static constexpr bool value = true; };

// phi(r) of a radial term given the element's attribute value a0 (the spring's
// squared rest length; unused by the edge length)
template <int TT, class S>
MG_DI auto radial_phi(const TermDev& t, double a0, const S& r) {
  if constexpr (TT == MG_TERM_SPRING) {
    auto s = r / a0 - 1.0;
    return (s * s) * (t.c[0] * a0);
  } else {
    static_assert(TT == MG_TERM_EDGE_LENGTH, "not a radial term");
    (void)t;
    (void)a0;
    return r;
  }
}
template <int TT> struct RadialAttr { static constexpr bool value = TT == MG_TERM_SPRING; };

template <int TT, class S>
MG_DI auto term_eval_radial(const TermDev& t, int64_t e, const S& r) {
  return radial_phi<TT>(t, RadialAttr<TT>::value ? t.a[0][e] : 0.0, r);
}

template <int TT, int N, class S>
MG_DI auto term_eval_diff(const TermDev& t, int64_t e, const Vec<S, N>& d) {
  if constexpr (TT == MG_TERM_SPRING) {
    const double l2 = t.a[0][e];
    auto s = norm2(d) / l2 - 1.0;
    return (s * s) * (t.c[0] * l2);
  } else {
    static_assert(TT == MG_TERM_EDGE_LENGTH, "not a two-point term");
    return norm2(d);
  }
}

// e: element id (== vertex id for V terms); vid: the element's P vertex ids;
// X: the P lifted per-vertex variable vectors.
template <int TT, int N, class S>
MG_DI auto term_eval(const TermDev& t, int64_t e, const int* vid, const Vec<S, N>* X) {
  if constexpr (TT == MG_TERM_INERTIA) {
    // d = x[v] - target[v]; 0.5 * m[v] * d.norm2()          (cloth.py:102-104)
    auto d = vsub(X[0], t.a[1] + e * N);
    return norm2(d) * (0.5 * t.a[0][e]);
  } else if constexpr (TT == MG_TERM_SPRING) {
    // d = x_i - x_j; s = d.norm2()/l2 - 1; (c * l2) * (s*s)   (cloth.py:106-110)
    const double l2 = t.a[0][e];
    auto d = vsub(X[0], X[1]);
    auto s = norm2(d) / l2 - 1.0;
    return (s * s) * (t.c[0] * l2);
  } else if constexpr (TT == MG_TERM_GRAVITY) {
    // (-h2) * (m[v] * x[v].dot(g))                            (cloth.py:112-113)
    return (dot(X[0], t.c + 1) * t.a[0][e]) * (-t.c[0]);
  } else if constexpr (TT == MG_TERM_EDGE_LENGTH) {
    // (x_i - x_j).norm2()                                     (smooth.py:27-28)
    return norm2(vsub(X[0], X[1]));
  } else if constexpr (TT == MG_TERM_SYM_DIRICHLET) {
    static_assert(N == 2, "symmetric Dirichlet is a UV (n = 2) energy");
    // param.py:170-177
    const double* R = t.a[0] + e * 4;  // rest_inv[f], row-major 2x2
    auto d1 = vsub(X[1], X[0]);
    auto d2 = vsub(X[2], X[0]);
    // SmallMatrix([[d1x, d2x], [d1y, d2y]]) @ R  (active.py:469-487)
    auto j00 = d1[0] * R[0] + d2[0] * R[2];
    auto j01 = d1[0] * R[1] + d2[0] * R[3];
    auto j10 = d1[1] * R[0] + d2[1] * R[2];
    auto j11 = d1[1] * R[1] + d2[1] * R[3];
    auto det = positive_guard(j00 * j11 - j01 * j10);
    // frobenius2: acc = e*e + acc, acc starting at 0.0 (active.py:462-467)
    auto fro = j00 * j00 + 0.0;
    fro = j01 * j01 + fro;
    fro = j10 * j10 + fro;
    fro = j11 * j11 + fro;
    return (fro + fro / (det * det)) * t.a[1][e];
  } else {
    static_assert(TT == MG_TERM_SPHERE, "unknown term");
    static_assert(N == 2, "sphere energy uses 2 tangent variables per vertex");
    // sphere.py:71-99: p_q = normalize(x0*b1 + x1*b2 + s) per vertex
    using S3 = decltype(X[0][0] * 1.0 + X[0][0] * 1.0 + 1.0);
    using SP = decltype(S3{} / sqrt(norm2(Vec<S3, 3>{})));
    Vec<SP, 3> p[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int64_t v = vid[q];
      const double* s = t.a[0] + v * 3;
      const double* b1 = t.a[1] + v * 3;
      const double* b2 = t.a[2] + v * 3;
      Vec<S3, 3> r;
#pragma unroll
      for (int c = 0; c < 3; ++c) r[c] = X[q][0] * b1[c] + X[q][1] * b2[c] + s[c];
      auto nrm = sqrt(norm2(r));
#pragma unroll
      for (int c = 0; c < 3; ++c) p[q][c] = r[c] / nrm;
    }
    const bool barrier = t.c[0] != 0.0, stretch = t.c[1] != 0.0;
    using SR = decltype(p[0][0] * p[0][0] + 0.0);
    SR total{};
    if (barrier) {
      // SmallMatrix.from_columns(p0, p1, p2).det(): m_ij = p_j[i] (active.py:432-453)
      auto det = p[0][0] * (p[1][1] * p[2][2] - p[2][1] * p[1][2]) -
                 p[1][0] * (p[0][1] * p[2][2] - p[2][1] * p[0][2]) +
                 p[2][0] * (p[0][1] * p[1][2] - p[1][1] * p[0][2]);
      total = -log(det) + 0.0;
    }
    if (stretch) {
      auto a = norm2(vsub(p[0], p[1]));
      auto b = norm2(vsub(p[1], p[2]));
      auto c = norm2(vsub(p[2], p[0]));
      if (barrier) total = total + a + b + c;
      else total = a + 0.0 + b + c;
    }
    return total;
  }
}

}  // namespace mg
