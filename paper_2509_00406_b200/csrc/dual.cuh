// Device dual numbers for per-element forward-mode AD (sm_100a).
//
// Restates the arithmetic of the reference's batched `ActiveScalar`
// (meshgrad/active.py:102-327) for ONE element per thread, with everything in
// registers and the local variable count K a compile-time constant:
//
//   Dv<K>        value-only ("passive" lift, problem.py:425-426). A wrapper
//                rather than a bare double so divisions follow the reference
//                (value * (1/b), active.py:180-190) bit for bit.
//   Dg<K>        value + gradient[K]            (gradient mode, hess None)
//   Dh<K,Z>      value + gradient + packed symmetric Hessian (K(K+1)/2).
//                Z == true is the reference's *structural zero* Hessian
//                (hess == 0.0, active.py:8-13): it carries no storage and the
//                product rule skips it exactly as `_h_scale/_h_add` do, so
//                NaN/Inf behaviour matches the reference per entry.
//   Df<K,Z>      forward-over-forward dual for matrix-free HVP: value,
//                gradient, directional derivative vd = g.w and gd = H.w
//                (O(K) per op instead of O(K^2)). Z as above for gd.
//
// The gradient is deliberately dense (no compile-time sparsity folding):
// the reference multiplies real zero entries, so 0*Inf -> NaN spreads through
// a gradient exactly as in numpy.
//
// Primal values are computed with explicitly rounded operations
// (__dadd_rn / __dmul_rn, which the compiler never fuses into an FMA) so a
// callback's value is bitwise the reference's numpy value for the same
// operation order. This matters where the primal itself is ill-conditioned:
// the sphere barrier's det[p0 p1 p2] at icosphere(10) is the difference of
// O(1) products ~1e-6 apart, and a fused rounding there moves every face
// gradient by ~1e-10 relative. Derivative parts may fuse.
//
// Packed Hessian index for i >= j: i*(i+1)/2 + j. Every product-rule update
// is computed once per unordered pair, so the assembled blocks are bitwise
// symmetric by construction (the reference guarantees the same, active.py:19-21).
#pragma once
#include <cmath>
#include <cstdint>

#define MG_DI __device__ __forceinline__

namespace mg {

MG_DI constexpr int tri(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }
template <int K> struct TriN { static constexpr int value = K * (K + 1) / 2; };

MG_DI double nan_d() { return __longlong_as_double(0x7ff8000000000000LL); }

// --------------------------------------------------------------------------
// value-only
template <int K>
struct Dv {
  double v;
};

template <int K> MG_DI Dv<K> operator+(Dv<K> a, Dv<K> b) { return {__dadd_rn(a.v, b.v)}; }
template <int K> MG_DI Dv<K> operator+(Dv<K> a, double b) { return {__dadd_rn(a.v, b)}; }
template <int K> MG_DI Dv<K> operator+(double b, Dv<K> a) { return {__dadd_rn(a.v, b)}; }
template <int K> MG_DI Dv<K> operator-(Dv<K> a, Dv<K> b) { return {__dsub_rn(a.v, b.v)}; }
template <int K> MG_DI Dv<K> operator-(Dv<K> a, double b) { return {__dsub_rn(a.v, b)}; }
template <int K> MG_DI Dv<K> operator-(double b, Dv<K> a) { return {__dsub_rn(b, a.v)}; }
template <int K> MG_DI Dv<K> operator-(Dv<K> a) { return {-a.v}; }
template <int K> MG_DI Dv<K> operator*(Dv<K> a, Dv<K> b) { return {__dmul_rn(a.v, b.v)}; }
template <int K> MG_DI Dv<K> operator*(Dv<K> a, double b) { return {__dmul_rn(a.v, b)}; }
template <int K> MG_DI Dv<K> operator*(double b, Dv<K> a) { return {__dmul_rn(a.v, b)}; }
template <int K> MG_DI Dv<K> operator/(Dv<K> a, Dv<K> b) { double u = 1.0 / b.v; return {__dmul_rn(a.v, u)}; }
template <int K> MG_DI Dv<K> operator/(Dv<K> a, double b) { double u = 1.0 / b; return {__dmul_rn(a.v, u)}; }
template <int K> MG_DI Dv<K> operator/(double a, Dv<K> b) { double u = 1.0 / b.v; return {__dmul_rn(a, u)}; }
template <int K> MG_DI Dv<K> sqrt(Dv<K> a) { return {::sqrt(a.v)}; }
template <int K> MG_DI Dv<K> log(Dv<K> a) { return {::log(a.v)}; }
template <int K> MG_DI Dv<K> exp(Dv<K> a) { return {::exp(a.v)}; }
template <int K> MG_DI Dv<K> sin(Dv<K> a) { return {::sin(a.v)}; }
template <int K> MG_DI Dv<K> cos(Dv<K> a) { return {::cos(a.v)}; }
template <int K> MG_DI Dv<K> positive_guard(Dv<K> a) { return {a.v > 0.0 ? a.v : nan_d()}; }

// --------------------------------------------------------------------------
// gradient mode
template <int K>
struct Dg {
  double v;
  double g[K];
};

template <int K> MG_DI Dg<K> operator+(const Dg<K>& a, const Dg<K>& b) {
  Dg<K> r; r.v = __dadd_rn(a.v, b.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] + b.g[i];
  return r;
}
template <int K> MG_DI Dg<K> operator+(const Dg<K>& a, double b) { Dg<K> r = a; r.v = __dadd_rn(a.v, b); return r; }
template <int K> MG_DI Dg<K> operator+(double b, const Dg<K>& a) { return a + b; }
template <int K> MG_DI Dg<K> operator-(const Dg<K>& a, const Dg<K>& b) {
  Dg<K> r; r.v = __dsub_rn(a.v, b.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] - b.g[i];
  return r;
}
template <int K> MG_DI Dg<K> operator-(const Dg<K>& a, double b) { Dg<K> r = a; r.v = __dsub_rn(a.v, b); return r; }
template <int K> MG_DI Dg<K> operator-(const Dg<K>& a) {
  Dg<K> r; r.v = -a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = -a.g[i];
  return r;
}
template <int K> MG_DI Dg<K> operator-(double b, const Dg<K>& a) {
  Dg<K> r; r.v = __dsub_rn(b, a.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = -a.g[i];
  return r;
}
template <int K> MG_DI Dg<K> operator*(const Dg<K>& a, double c) {
  Dg<K> r; r.v = __dmul_rn(a.v, c);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] * c;
  return r;
}
template <int K> MG_DI Dg<K> operator*(double c, const Dg<K>& a) { return a * c; }
template <int K> MG_DI Dg<K> operator*(const Dg<K>& a, const Dg<K>& b) {
  Dg<K> r; r.v = __dmul_rn(a.v, b.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] * b.v + b.g[i] * a.v;
  return r;
}
template <int K> MG_DI Dg<K> operator/(const Dg<K>& a, double b) { double u = 1.0 / b; return a * u; }
template <int K> MG_DI Dg<K> operator/(const Dg<K>& a, const Dg<K>& b) {
  double u = 1.0 / b.v;
  Dg<K> r; r.v = __dmul_rn(a.v, u);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = (a.g[i] - r.v * b.g[i]) * u;
  return r;
}
template <int K> MG_DI Dg<K> operator/(double a, const Dg<K>& b) {
  double u = 1.0 / b.v;
  Dg<K> r; r.v = __dmul_rn(a, u);
  double f = -r.v * u;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = b.g[i] * f;
  return r;
}
template <int K> MG_DI Dg<K> chain1(const Dg<K>& a, double f0, double f1) {
  Dg<K> r; r.v = f0;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] * f1;
  return r;
}
template <int K> MG_DI Dg<K> sqrt(const Dg<K>& a) { double f0 = ::sqrt(a.v); return chain1(a, f0, 0.5 / f0); }
template <int K> MG_DI Dg<K> log(const Dg<K>& a) { return chain1(a, ::log(a.v), 1.0 / a.v); }
template <int K> MG_DI Dg<K> exp(const Dg<K>& a) { double f0 = ::exp(a.v); return chain1(a, f0, f0); }
template <int K> MG_DI Dg<K> sin(const Dg<K>& a) { return chain1(a, ::sin(a.v), ::cos(a.v)); }
template <int K> MG_DI Dg<K> cos(const Dg<K>& a) { return chain1(a, ::cos(a.v), -::sin(a.v)); }
template <int K> MG_DI Dg<K> positive_guard(const Dg<K>& a) { Dg<K> r = a; r.v = a.v > 0.0 ? a.v : nan_d(); return r; }

// --------------------------------------------------------------------------
// Hessian mode. Z == true: structurally zero Hessian (no storage).
template <int K, bool Z> struct Dh;

template <int K>
struct Dh<K, true> {
  static constexpr bool kZero = true;
  double v;
  double g[K];
};

template <int K>
struct Dh<K, false> {
  static constexpr bool kZero = false;
  double v;
  double g[K];
  double h[TriN<K>::value];
};

namespace detail {
// _h_add / _h_sub / _h_scale of active.py:52-93 over the compile-time encoding.
template <int K, bool ZA, bool ZB>
MG_DI void h_add(Dh<K, ZA && ZB>& r, const Dh<K, ZA>& a, const Dh<K, ZB>& b) {
  if constexpr (!ZA && !ZB) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = a.h[i] + b.h[i];
  } else if constexpr (!ZA) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = a.h[i];
  } else if constexpr (!ZB) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = b.h[i];
  }
}
template <int K, bool ZA, bool ZB>
MG_DI void h_sub(Dh<K, ZA && ZB>& r, const Dh<K, ZA>& a, const Dh<K, ZB>& b) {
  if constexpr (!ZA && !ZB) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = a.h[i] - b.h[i];
  } else if constexpr (!ZA) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = a.h[i];
  } else if constexpr (!ZB) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = -b.h[i];
  }
}
}  // namespace detail

template <int K, bool ZA, bool ZB>
MG_DI Dh<K, ZA && ZB> operator+(const Dh<K, ZA>& a, const Dh<K, ZB>& b) {
  Dh<K, ZA && ZB> r; r.v = __dadd_rn(a.v, b.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] + b.g[i];
  detail::h_add<K, ZA, ZB>(r, a, b);
  return r;
}
template <int K, bool Z> MG_DI Dh<K, Z> operator+(const Dh<K, Z>& a, double b) { Dh<K, Z> r = a; r.v = __dadd_rn(a.v, b); return r; }
template <int K, bool Z> MG_DI Dh<K, Z> operator+(double b, const Dh<K, Z>& a) { return a + b; }
template <int K, bool ZA, bool ZB>
MG_DI Dh<K, ZA && ZB> operator-(const Dh<K, ZA>& a, const Dh<K, ZB>& b) {
  Dh<K, ZA && ZB> r; r.v = __dsub_rn(a.v, b.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] - b.g[i];
  detail::h_sub<K, ZA, ZB>(r, a, b);
  return r;
}
template <int K, bool Z> MG_DI Dh<K, Z> operator-(const Dh<K, Z>& a, double b) { Dh<K, Z> r = a; r.v = __dsub_rn(a.v, b); return r; }
template <int K, bool Z> MG_DI Dh<K, Z> operator-(const Dh<K, Z>& a) {
  Dh<K, Z> r; r.v = -a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = -a.g[i];
  if constexpr (!Z) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = -a.h[i];
  }
  return r;
}
template <int K, bool Z> MG_DI Dh<K, Z> operator-(double b, const Dh<K, Z>& a) {
  Dh<K, Z> r = -a; r.v = __dsub_rn(b, a.v); return r;
}
template <int K, bool Z> MG_DI Dh<K, Z> operator*(const Dh<K, Z>& a, double c) {
  Dh<K, Z> r; r.v = __dmul_rn(a.v, c);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] * c;
  if constexpr (!Z) {
#pragma unroll
    for (int i = 0; i < TriN<K>::value; ++i) r.h[i] = a.h[i] * c;
  }
  return r;
}
template <int K, bool Z> MG_DI Dh<K, Z> operator*(double c, const Dh<K, Z>& a) { return a * c; }

// product rule, active.py:156-178:
//   h = (a.h*bv + b.h*av) + (ga gb^T + gb ga^T)
template <int K, bool ZA, bool ZB>
MG_DI Dh<K, false> operator*(const Dh<K, ZA>& a, const Dh<K, ZB>& b) {
  Dh<K, false> r; r.v = __dmul_rn(a.v, b.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] * b.v + b.g[i] * a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double os = a.g[i] * b.g[j] + b.g[i] * a.g[j];
      if constexpr (!ZA && !ZB) r.h[tri(i, j)] = (a.h[tri(i, j)] * b.v + b.h[tri(i, j)] * a.v) + os;
      else if constexpr (!ZA) r.h[tri(i, j)] = a.h[tri(i, j)] * b.v + os;
      else if constexpr (!ZB) r.h[tri(i, j)] = b.h[tri(i, j)] * a.v + os;
      else r.h[tri(i, j)] = os;
    }
  }
  return r;
}
template <int K, bool Z> MG_DI Dh<K, Z> operator/(const Dh<K, Z>& a, double b) { double u = 1.0 / b; return a * u; }

// quotient rule, active.py:180-205:
//   u = 1/bv, v = av*u, g = (ga - v gb) u,
//   h = (a.h u + b.h (-v u)) + (sym(ga,gb)(-u u) + gb gb^T (2 v u u))
template <int K, bool ZA, bool ZB>
MG_DI Dh<K, false> operator/(const Dh<K, ZA>& a, const Dh<K, ZB>& b) {
  double u = 1.0 / b.v;
  Dh<K, false> r; r.v = __dmul_rn(a.v, u);
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = (a.g[i] - r.v * b.g[i]) * u;
  const double cb = -r.v * u, cs = -u * u, cq = 2.0 * r.v * u * u;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double tail = (a.g[i] * b.g[j] + b.g[i] * a.g[j]) * cs + (b.g[i] * b.g[j]) * cq;
      if constexpr (!ZA && !ZB) r.h[tri(i, j)] = (a.h[tri(i, j)] * u + b.h[tri(i, j)] * cb) + tail;
      else if constexpr (!ZA) r.h[tri(i, j)] = a.h[tri(i, j)] * u + tail;
      else if constexpr (!ZB) r.h[tri(i, j)] = b.h[tri(i, j)] * cb + tail;
      else r.h[tri(i, j)] = tail;
    }
  }
  return r;
}
// passive numerator, active.py:207-221
template <int K, bool Z>
MG_DI Dh<K, false> operator/(double a, const Dh<K, Z>& b) {
  double u = 1.0 / b.v;
  Dh<K, false> r; r.v = __dmul_rn(a, u);
  const double cb = -r.v * u, cq = 2.0 * r.v * u * u;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = b.g[i] * cb;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double q = (b.g[i] * b.g[j]) * cq;
      if constexpr (!Z) r.h[tri(i, j)] = b.h[tri(i, j)] * cb + q;
      else r.h[tri(i, j)] = q;
    }
  }
  return r;
}
// unary chain rule, active.py:252-258: h = a.h f1 + (g g^T) f2
template <int K, bool Z>
MG_DI Dh<K, false> chain2(const Dh<K, Z>& a, double f0, double f1, double f2) {
  Dh<K, false> r; r.v = f0;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] * f1;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double q = (a.g[i] * a.g[j]) * f2;
      if constexpr (!Z) r.h[tri(i, j)] = a.h[tri(i, j)] * f1 + q;
      else r.h[tri(i, j)] = q;
    }
  }
  return r;
}
template <int K, bool Z> MG_DI Dh<K, false> sqrt(const Dh<K, Z>& a) {
  double f0 = ::sqrt(a.v), f1 = 0.5 / f0;
  return chain2(a, f0, f1, -0.5 * f1 / a.v);
}
template <int K, bool Z> MG_DI Dh<K, false> log(const Dh<K, Z>& a) {
  double f1 = 1.0 / a.v;
  return chain2(a, ::log(a.v), f1, -f1 * f1);
}
template <int K, bool Z> MG_DI Dh<K, false> exp(const Dh<K, Z>& a) { double f0 = ::exp(a.v); return chain2(a, f0, f0, f0); }
template <int K, bool Z> MG_DI Dh<K, false> sin(const Dh<K, Z>& a) { double f0 = ::sin(a.v); return chain2(a, f0, ::cos(a.v), -f0); }
template <int K, bool Z> MG_DI Dh<K, false> cos(const Dh<K, Z>& a) { double f0 = ::cos(a.v); return chain2(a, f0, -::sin(a.v), -f0); }
template <int K, bool Z> MG_DI Dh<K, Z> positive_guard(const Dh<K, Z>& a) { Dh<K, Z> r = a; r.v = a.v > 0.0 ? a.v : nan_d(); return r; }

// --------------------------------------------------------------------------
// forward-over-forward (HVP) mode. gd = H w, vd = g.w.  Z: H structurally 0.
template <int K, bool Z> struct Df;

template <int K>
struct Df<K, true> {
  static constexpr bool kZero = true;
  double v, vd;
  double g[K];
};
template <int K>
struct Df<K, false> {
  static constexpr bool kZero = false;
  double v, vd;
  double g[K];
  double gd[K];
};

template <int K, bool ZA, bool ZB>
MG_DI Df<K, ZA && ZB> operator+(const Df<K, ZA>& a, const Df<K, ZB>& b) {
  Df<K, ZA && ZB> r; r.v = __dadd_rn(a.v, b.v); r.vd = a.vd + b.vd;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] + b.g[i];
  if constexpr (!ZA && !ZB) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = a.gd[i] + b.gd[i];
  } else if constexpr (!ZA) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = a.gd[i];
  } else if constexpr (!ZB) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = b.gd[i];
  }
  return r;
}
template <int K, bool Z> MG_DI Df<K, Z> operator+(const Df<K, Z>& a, double b) { Df<K, Z> r = a; r.v = __dadd_rn(a.v, b); return r; }
template <int K, bool Z> MG_DI Df<K, Z> operator+(double b, const Df<K, Z>& a) { return a + b; }
template <int K, bool Z> MG_DI Df<K, Z> operator-(const Df<K, Z>& a) {
  Df<K, Z> r; r.v = -a.v; r.vd = -a.vd;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = -a.g[i];
  if constexpr (!Z) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = -a.gd[i];
  }
  return r;
}
template <int K, bool ZA, bool ZB>
MG_DI Df<K, ZA && ZB> operator-(const Df<K, ZA>& a, const Df<K, ZB>& b) {
  Df<K, ZA && ZB> r; r.v = __dsub_rn(a.v, b.v); r.vd = a.vd - b.vd;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] - b.g[i];
  if constexpr (!ZA && !ZB) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = a.gd[i] - b.gd[i];
  } else if constexpr (!ZA) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = a.gd[i];
  } else if constexpr (!ZB) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = -b.gd[i];
  }
  return r;
}
template <int K, bool Z> MG_DI Df<K, Z> operator-(const Df<K, Z>& a, double b) { Df<K, Z> r = a; r.v = __dsub_rn(a.v, b); return r; }
template <int K, bool Z> MG_DI Df<K, Z> operator-(double b, const Df<K, Z>& a) { Df<K, Z> r = -a; r.v = __dsub_rn(b, a.v); return r; }
template <int K, bool Z> MG_DI Df<K, Z> operator*(const Df<K, Z>& a, double c) {
  Df<K, Z> r; r.v = __dmul_rn(a.v, c); r.vd = a.vd * c;
#pragma unroll
  for (int i = 0; i < K; ++i) r.g[i] = a.g[i] * c;
  if constexpr (!Z) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.gd[i] = a.gd[i] * c;
  }
  return r;
}
template <int K, bool Z> MG_DI Df<K, Z> operator*(double c, const Df<K, Z>& a) { return a * c; }
// (H_a bv + H_b av + ga gb^T + gb ga^T) w
template <int K, bool ZA, bool ZB>
MG_DI Df<K, false> operator*(const Df<K, ZA>& a, const Df<K, ZB>& b) {
  Df<K, false> r; r.v = __dmul_rn(a.v, b.v); r.vd = a.vd * b.v + b.vd * a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    r.g[i] = a.g[i] * b.v + b.g[i] * a.v;
    double os = a.g[i] * b.vd + b.g[i] * a.vd;
    if constexpr (!ZA && !ZB) r.gd[i] = (a.gd[i] * b.v + b.gd[i] * a.v) + os;
    else if constexpr (!ZA) r.gd[i] = a.gd[i] * b.v + os;
    else if constexpr (!ZB) r.gd[i] = b.gd[i] * a.v + os;
    else r.gd[i] = os;
  }
  return r;
}
template <int K, bool Z> MG_DI Df<K, Z> operator/(const Df<K, Z>& a, double b) { double u = 1.0 / b; return a * u; }
template <int K, bool ZA, bool ZB>
MG_DI Df<K, false> operator/(const Df<K, ZA>& a, const Df<K, ZB>& b) {
  double u = 1.0 / b.v;
  Df<K, false> r; r.v = __dmul_rn(a.v, u); r.vd = (a.vd - r.v * b.vd) * u;
  const double cb = -r.v * u, cs = -u * u, cq = 2.0 * r.v * u * u;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    r.g[i] = (a.g[i] - r.v * b.g[i]) * u;
    double tail = (a.g[i] * b.vd + b.g[i] * a.vd) * cs + (b.g[i] * b.vd) * cq;
    if constexpr (!ZA && !ZB) r.gd[i] = (a.gd[i] * u + b.gd[i] * cb) + tail;
    else if constexpr (!ZA) r.gd[i] = a.gd[i] * u + tail;
    else if constexpr (!ZB) r.gd[i] = b.gd[i] * cb + tail;
    else r.gd[i] = tail;
  }
  return r;
}
template <int K, bool Z>
MG_DI Df<K, false> operator/(double a, const Df<K, Z>& b) {
  double u = 1.0 / b.v;
  Df<K, false> r; r.v = __dmul_rn(a, u);
  const double cb = -r.v * u, cq = 2.0 * r.v * u * u;
  r.vd = b.vd * cb;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    r.g[i] = b.g[i] * cb;
    double q = (b.g[i] * b.vd) * cq;
    if constexpr (!Z) r.gd[i] = b.gd[i] * cb + q;
    else r.gd[i] = q;
  }
  return r;
}
template <int K, bool Z>
MG_DI Df<K, false> chainf(const Df<K, Z>& a, double f0, double f1, double f2) {
  Df<K, false> r; r.v = f0; r.vd = a.vd * f1;
  const double s = a.vd * f2;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    r.g[i] = a.g[i] * f1;
    double q = a.g[i] * s;
    if constexpr (!Z) r.gd[i] = a.gd[i] * f1 + q;
    else r.gd[i] = q;
  }
  return r;
}
template <int K, bool Z> MG_DI Df<K, false> sqrt(const Df<K, Z>& a) {
  double f0 = ::sqrt(a.v), f1 = 0.5 / f0;
  return chainf(a, f0, f1, -0.5 * f1 / a.v);
}
template <int K, bool Z> MG_DI Df<K, false> log(const Df<K, Z>& a) {
  double f1 = 1.0 / a.v;
  return chainf(a, ::log(a.v), f1, -f1 * f1);
}
template <int K, bool Z> MG_DI Df<K, false> exp(const Df<K, Z>& a) { double f0 = ::exp(a.v); return chainf(a, f0, f0, f0); }
template <int K, bool Z> MG_DI Df<K, false> sin(const Df<K, Z>& a) { double f0 = ::sin(a.v); return chainf(a, f0, ::cos(a.v), -f0); }
template <int K, bool Z> MG_DI Df<K, false> cos(const Df<K, Z>& a) { double f0 = ::cos(a.v); return chainf(a, f0, -::sin(a.v), -f0); }
template <int K, bool Z> MG_DI Df<K, Z> positive_guard(const Df<K, Z>& a) { Df<K, Z> r = a; r.v = a.v > 0.0 ? a.v : nan_d(); return r; }

// --------------------------------------------------------------------------
// small fixed vectors of scalars (ActiveVec, active.py:345-416)
template <class S, int N>
struct Vec {
  S c[N];
  MG_DI S& operator[](int i) { return c[i]; }
  MG_DI const S& operator[](int i) const { return c[i]; }
};

template <class S, int N> MG_DI auto vsub(const Vec<S, N>& a, const Vec<S, N>& b) {
  Vec<decltype(a.c[0] - b.c[0]), N> r;
#pragma unroll
  for (int i = 0; i < N; ++i) r.c[i] = a.c[i] - b.c[i];
  return r;
}
template <class S, int N> MG_DI Vec<S, N> vsub(const Vec<S, N>& a, const double* b) {
  Vec<S, N> r;
#pragma unroll
  for (int i = 0; i < N; ++i) r.c[i] = a.c[i] - b[i];
  return r;
}
// norm2: acc = c0*c0; acc = acc + ci*ci  (active.py:387-391)
template <class S, int N> MG_DI auto norm2(const Vec<S, N>& a) {
  auto acc = a.c[0] * a.c[0];
#pragma unroll
  for (int i = 1; i < N; ++i) acc = acc + a.c[i] * a.c[i];
  return acc;
}
// dot with a passive vector (active.py:381-385)
template <class S, int N> MG_DI S dot(const Vec<S, N>& a, const double* b) {
  S acc = a.c[0] * b[0];
#pragma unroll
  for (int i = 1; i < N; ++i) acc = acc + a.c[i] * b[i];
  return acc;
}

}  // namespace mg
