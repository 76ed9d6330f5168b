// Per-element evaluation shared by the patch kernels: lift (unit seeds,
// free-masked), term_eval, and the reference's `_extract` epilogue
// (problem.py:454-476: structural zero, symmetrise, optional PSD clamp).
#pragma once
#include "mg_internal.cuh"
#include "psd.cuh"

namespace mg {

// Evaluate one element: dual result -> value + per-slot contributions.
//   MODE_GRAD: g[K];  MODE_HESS: g[K] and packed h (valid flag);
//   MODE_HVP: hv[K] (H v, PSD-clamped if requested).
template <int P_, int N, int MODE, bool PSD>
struct ElemOutP {
  static constexpr int P = P_, K = P * N;
  double val;
  double g[K];
  double h[(MODE == MODE_HESS) ? TriN<K>::value : 1];
  bool has_h;
};
template <int TT, int N, int MODE, bool PSD>
using ElemOut = ElemOutP<TermInfo<TT>::P, N, MODE, PSD>;

// the term as an evaluator: ev(e, vid, X) -> dual result (builtin terms here;
// traced callbacks supply their generated functor, jit_patch.cuh)
template <int TT, int N>
struct BuiltinEval {
  const TermDev& t;
  template <class S>
  MG_DI auto operator()(int64_t e, const int* vid, const Vec<S, N>* X) const { return term_eval<TT, N>(t, e, vid, X); }
};

template <int P, int N, int MODE, bool PSD, class EV>
__device__ __forceinline__ void eval_element_f(const EV& ev, int64_t e, const int* vid, const double* const* xr,
                                               const double* const* wr, const bool* fr, double floor,
                                               ElemOutP<P, N, MODE, PSD>& o);

template <int TT, int N, int MODE, bool PSD>
__device__ __forceinline__ void eval_element(const TermDev& t, int64_t e, const int* vid, const double* const* xr,
                                             const double* const* wr, const bool* fr, double floor,
                                             ElemOut<TT, N, MODE, PSD>& o) {
  eval_element_f<TermInfo<TT>::P, N, MODE, PSD>(BuiltinEval<TT, N>{t}, e, vid, xr, wr, fr, floor, o);
}

template <int P, int N, int MODE, bool PSD, class EV>
__device__ __forceinline__ void eval_element_f(const EV& ev, int64_t e, const int* vid, const double* const* xr,
                                               const double* const* wr, const bool* fr, double floor,
                                               ElemOutP<P, N, MODE, PSD>& o) {
  constexpr int K = P * N;
  if constexpr (MODE == MODE_ENERGY) {
    Vec<Dv<K>, N> X[P];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < N; ++c) X[q][c].v = xr[q][c];
    o.val = ev(e, vid, X).v;
  } else if constexpr (MODE == MODE_GRAD) {
    Vec<Dg<K>, N> X[P];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        X[q][c].v = xr[q][c];
#pragma unroll
        for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c) ? 1.0 : 0.0;
      }
    auto r = ev(e, vid, X);
    o.val = r.v;
#pragma unroll
    for (int i = 0; i < K; ++i) o.g[i] = r.g[i];
  } else if constexpr (MODE == MODE_HESS || (MODE == MODE_HVP && PSD)) {
    Vec<Dh<K, true>, N> X[P];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        X[q][c].v = xr[q][c];
#pragma unroll
        for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c) ? 1.0 : 0.0;
      }
    auto r = ev(e, vid, X);
    using R = decltype(r);
    o.val = r.v;
    if constexpr (MODE == MODE_HESS) {
#pragma unroll
      for (int i = 0; i < K; ++i) o.g[i] = r.g[i];
    }
    o.has_h = !R::kZero || PSD;
    double h[TriN<K>::value];
    if constexpr (R::kZero) {
#pragma unroll
      for (int i = 0; i < TriN<K>::value; ++i) h[i] = 0.0;
    } else {
#pragma unroll
      for (int i = 0; i < TriN<K>::value; ++i) h[i] = r.h[i];
    }
    if constexpr (PSD) {
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (!fr[q])
#pragma unroll
          for (int c = 0; c < N; ++c)
#pragma unroll
            for (int j = 0; j < K; ++j) h[tri(q * N + c, j)] = 0.0;
      extract_psd<P, N>(h, floor);
    } else {
#pragma unroll
      for (int i = 0; i < TriN<K>::value; ++i) h[i] = 0.5 * (h[i] + h[i]);
    }
    if constexpr (MODE == MODE_HESS) {
#pragma unroll
      for (int i = 0; i < TriN<K>::value; ++i) o.h[i] = h[i];
    } else {
      double vl[K];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) vl[q * N + c] = fr[q] ? wr[q][c] : 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) acc += h[tri(i, j)] * vl[j];
        o.g[i] = o.has_h ? acc : 0.0;
      }
    }
  } else {  // HVP without PSD: forward-over-forward
    Vec<Df<K, true>, N> X[P];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        X[q][c].v = xr[q][c];
        X[q][c].vd = fr[q] ? wr[q][c] : 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c) ? 1.0 : 0.0;
      }
    auto r = ev(e, vid, X);
    using R = decltype(r);
    o.val = r.v;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if constexpr (R::kZero) o.g[i] = 0.0;
      else o.g[i] = r.gd[i];
    }
  }
}

// Fixed-order block sum over NT threads (warp shuffle tree, then thread 0
// over the warp sums); valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum_fixed(double v) {
  __shared__ double ws[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) r += ws[i];
  return r;
}

}  // namespace mg
