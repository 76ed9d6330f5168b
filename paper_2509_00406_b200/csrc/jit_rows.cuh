// Edge row kernels for traced (JIT) energy terms.
//
// When every EV callback of a problem depends on the vertex positions only
// through r = |x_i - x_j|^2 (the tracer proves this on the recorded SSA,
// paper_2509_00406_b200/jit.py: radial_form), the problem's traced terms run
// on the builtin terms' edge row kernel (edge_rows.cuh) instead of the patch
// kernel. jit.py emits
//   * per V term a functor over the engine's duals on the row's own vertex
//     (K = n: the reference's lift of a one-vertex element), evaluated with
//     the same lift / _extract / PSD epilogue as the patch kernel
//     (elem_eval.cuh), so its values are the exact path's;
//   * per EV term the callback's operations AFTER r as a function phi(r) of
//     one variable, evaluated on a second-order one-variable dual: phi, phi'
//     and phi'' give the edge's gradient 2 phi' d, its 6x6 Hessian
//     [[A,-A],[-A,A]] with A = 2 phi' I + 4 phi'' d d^T, and the block's PSD
//     clamp in closed form (the reference differentiates the same
//     expression with K = 2n duals; the values agree to rounding);
//   * a policy that runs them (attribute streams preloaded with the
//     incidence gathers, `av[k]` in the functors) and MG_ROWS_JIT_INSTANTIATE.
// A non-finite value raises the redo flag; the problem's traced patch module
// then re-runs the call with the full duals (the reference's NaN placement).
#pragma once
#include "edge_rows.cuh"
#include "elem_eval.cuh"
#include "jit_kernel.cuh"

namespace mg {
namespace rows {

// a V-term functor as an element evaluator (elem_eval.cuh)
template <class FN, int N>
struct JitVEval {
  const double* av;
  template <class S>
  MG_DI auto operator()(int64_t, const int*, const Vec<S, N>* X) const {
    return FN{}.template operator()<N>(av, X);
  }
};

// one traced V term at the row's vertex (the lift of a one-vertex element)
template <int N, int MODE, bool PSD, class FN>
MG_DI void jit_vterm(const FN&, const double* av, bool fr, const double* xs, const double* us, double floor,
                     double& eacc, double* vec, double* dg) {
  const double* xr[1] = {xs};
  const double* wr[1] = {us};
  const int vid = 0;
  ElemOutP<1, N, MODE, PSD> o;
  eval_element_f<1, N, MODE, PSD>(JitVEval<FN, N>{av}, 0, &vid, xr, wr, &fr, floor, o);
  eacc += o.val;
#pragma unroll
  for (int c = 0; c < N; ++c) vec[c] += o.g[c];
  if constexpr (MODE == MODE_HESS) {
    if (o.has_h)
#pragma unroll
      for (int k = 0; k < TriN<N>::value; ++k) dg[k] += o.h[k];
  }
}

template <class R> MG_DI double jr_value(const R& r) { return r.v; }
MG_DI double jr_value(double r) { return r; }
template <class R> MG_DI double jr_d1(const R& r) { return r.g[0]; }
MG_DI double jr_d1(double) { return 0.0; }
template <class R> MG_DI double jr_d2(const R& r) {
  if constexpr (R::kZero) return 0.0;
  else return r.h[0];
}
MG_DI double jr_d2(double) { return 0.0; }

// one traced V term the tracer proved radial in d = x - t (t an attribute
// or constant vector; jit.py radial_vform): E = phi(|d|^2) on a one-variable
// second-order dual, gradient 2 phi' d, Hessian A = 2 phi' I + 4 phi'' d d^T
// (clamped in closed form under a PSD floor). A non-finite value clears
// `finite` (the patch module's exact re-run then places NaN like the reference).
template <int N, int MODE, bool PSD, class PHI>
MG_DI void jit_vradial(const PHI& phi, const double* av, const double* d, const double* us, double floor,
                       double& eacc, double* vec, double* dg, bool& finite) {
  double rr = 0.0;
#pragma unroll
  for (int c = 0; c < N; ++c) rr = d[c] * d[c] + rr;
  double pv, p1, p2;
  if constexpr (MODE == MODE_GRAD || MODE == MODE_ENERGY) {
    Dg<1> R;
    R.v = rr;
    R.g[0] = 1.0;
    const auto r = phi(av, R);
    pv = jr_value(r);
    p1 = jr_d1(r);
    p2 = 0.0;
  } else {
    Dh<1, true> R;
    R.v = rr;
    R.g[0] = 1.0;
    const auto r = phi(av, R);
    pv = jr_value(r);
    p1 = jr_d1(r);
    p2 = jr_d2(r);
  }
  finite &= isfinite(pv + p1 + p2);
  eacc += pv;
  if constexpr (MODE == MODE_GRAD || MODE == MODE_HESS) {
#pragma unroll
    for (int c = 0; c < N; ++c) vec[c] += 2.0 * p1 * d[c];
  }
  if constexpr (MODE == MODE_HESS || MODE == MODE_HVP) {
    double ci = 2.0 * p1, cd = 4.0 * p2;
    if constexpr (PSD) radial_clamp_fast(ci, cd, rr, floor);
    if constexpr (MODE == MODE_HESS) {
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c) dg[tri(i, c)] += cd * d[i] * d[c] + (i == c ? ci : 0.0);
    } else {
      double du = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) du += d[c] * us[c];
#pragma unroll
      for (int i = 0; i < N; ++i) vec[i] += ci * us[i] + cd * d[i] * du;
    }
  }
}

// phi, phi', phi'' of one traced radial EV term at r (gradient mode: a
// first-order dual, phi'' = 0)
template <int MODE, bool NEEDV, class PHI, class F>
MG_DI void jit_radial(const PHI& phi, const double* av, double rr, F&& one) {
  double pv, p1, p2;
  if constexpr (MODE == MODE_GRAD) {
    Dg<1> R;
    R.v = rr;
    R.g[0] = 1.0;
    const auto r = phi(av, R);
    pv = jr_value(r);
    p1 = jr_d1(r);
    p2 = 0.0;
  } else {
    Dh<1, true> R;
    R.v = rr;
    R.g[0] = 1.0;
    const auto r = phi(av, R);
    pv = jr_value(r);
    p1 = jr_d1(r);
    p2 = jr_d2(r);
  }
  const bool ok = NEEDV ? isfinite(pv + p1 + p2) : isfinite(p1 + p2);
  one(ok, pv, p1, p2);
}

// preloaded attribute values of a row module (V streams per row, EV streams
// per incidence)
template <int K> struct JPre { double v[K > 0 ? K : 1]; };

}  // namespace rows
}  // namespace mg

#define MG_ROWS_JIT_KERNEL(POL, N, NAME, MODE, PSD)                                                                \
  extern "C" __global__ void __launch_bounds__(mg::rows::FastCfg<MODE, PSD>::BLOCK,                              \
                                               (mg::rows::FastMinb<MODE, PSD, POL::kXFreeHvp>::v))                 \
      NAME(const __grid_constant__ mg::rows::EvArgs a) {                                                           \
    mg::rows::rows_fast_body<N, MODE, PSD, POL>(a);                                                                \
  }

#define MG_ROWS_JIT_INSTANTIATE(POL, N)                              \
  MG_ROWS_JIT_KERNEL(POL, N, mg_rows_grad, mg::MODE_GRAD, false)     \
  MG_ROWS_JIT_KERNEL(POL, N, mg_rows_hess, mg::MODE_HESS, false)     \
  MG_ROWS_JIT_KERNEL(POL, N, mg_rows_hess_psd, mg::MODE_HESS, true)  \
  MG_ROWS_JIT_KERNEL(POL, N, mg_rows_hvp, mg::MODE_HVP, false)       \
  MG_ROWS_JIT_KERNEL(POL, N, mg_rows_hvp_psd, mg::MODE_HVP, true)
