// Element kernels for traced (JIT) energy terms.
//
// paper_2509_00406_b200/jit.py traces a user callback written against the
// reference's ActiveVec / SmallMatrix API (the reference callback protocol,
// problem.py:8-14, 440-452) into an SSA expression and emits a functor
//
//   struct F { template <int N, class S>
//              MG_DI auto operator()(const double* const* A, int64_t e, const Vec<S, N>* X) const; };
//
// whose body replays the recorded operations, in the recorded order, on the
// engine's dual numbers (dual.cuh). MG_JIT_INSTANTIATE(F, P, N) then emits the
// extern "C" kernels the library launches through the driver API
// (mg_problem_add_jit_term): one element per thread, the reference's lift /
// _extract / scatter pipeline (problem.py:420-476, 526-544), fp64 atomics into
// zeroed outputs and fixed-order per-block energy partials.
#pragma once
#include "dual.cuh"
#include "jit_abi.h"
#include "psd.cuh"

namespace mg {

// integer power (active.py:225-243): f0 = v^p, f1 = p v^(p-1), f2 = p (p-1) v^(p-2)
MG_DI double jit_ipow(double v, int p) {
  double r = 1.0, b = v;
  int q = p < 0 ? -p : p;
  while (q) {
    if (q & 1) r *= b;
    b *= b;
    q >>= 1;
  }
  return p < 0 ? 1.0 / r : r;
}
MG_DI double powi(double a, int p) { return p == 0 ? 1.0 : jit_ipow(a, p); }
template <int K> MG_DI Dv<K> powi(Dv<K> a, int p) { return {p == 0 ? 1.0 : jit_ipow(a.v, p)}; }
template <int K> MG_DI Dg<K> powi(const Dg<K>& a, int p) {
  if (p == 0) { Dg<K> r; r.v = 1.0; for (int i = 0; i < K; ++i) r.g[i] = 0.0; return r; }
  if (p == 1) return a;
  return chain1(a, jit_ipow(a.v, p), p * jit_ipow(a.v, p - 1));
}
template <int K, bool Z> MG_DI Dh<K, false> powi(const Dh<K, Z>& a, int p) {
  if (p == 0) return chain2(a, 1.0, 0.0, 0.0);
  return chain2(a, jit_ipow(a.v, p), p * jit_ipow(a.v, p - 1), p * (p - 1) * jit_ipow(a.v, p - 2));
}
template <int K, bool Z> MG_DI Df<K, false> powi(const Df<K, Z>& a, int p) {
  if (p == 0) return chainf(a, 1.0, 0.0, 0.0);
  return chainf(a, jit_ipow(a.v, p), p * jit_ipow(a.v, p - 1), p * (p - 1) * jit_ipow(a.v, p - 2));
}
// |a| with derivative sign(a) (0 at the kink) and no curvature (active.py:245-249)
MG_DI double jit_sign(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : (v == 0.0 ? 0.0 : v)); }
MG_DI double abs_(double a) { return ::fabs(a); }
template <int K> MG_DI Dv<K> abs_(Dv<K> a) { return {::fabs(a.v)}; }
template <int K> MG_DI Dg<K> abs_(const Dg<K>& a) { return chain1(a, ::fabs(a.v), jit_sign(a.v)); }
template <int K, bool Z> MG_DI Dh<K, false> abs_(const Dh<K, Z>& a) { return chain2(a, ::fabs(a.v), jit_sign(a.v), 0.0); }
template <int K, bool Z> MG_DI Df<K, false> abs_(const Df<K, Z>& a) { return chainf(a, ::fabs(a.v), jit_sign(a.v), 0.0); }
MG_DI double positive_guard(double a) { return a > 0.0 ? a : nan_d(); }

MG_DI void jit_put_vec(const JitArgs& a, double* out, int64_t e, int P, int q, int N, int c, int v, double val) {
  if (a.sv) a.sv[(e * P + q) * N + c] = val;
  else atomicAdd(out + (int64_t)v * N + c, val);
}

template <class R> MG_DI double jit_value(const R& r) { return r.v; }
MG_DI double jit_value(double r) { return r; }

template <class F, int P, int N, int MODE, bool PSD>
MG_DI void jit_element(const JitArgs& a) {
  constexpr int K = P * N;
  const int64_t e = blockIdx.x * (int64_t)JIT_TPB + threadIdx.x;
  double ev = 0.0;
  if (e < a.M) {
    int vid[P];
#pragma unroll
    for (int q = 0; q < P; ++q) vid[q] = a.sel ? a.sel[e * P + q] : (int)e;
    bool fr[P];
#pragma unroll
    for (int q = 0; q < P; ++q) fr[q] = !a.fixed || !a.fixed[vid[q]];
    F f;
    if constexpr (MODE == JIT_ENERGY) {
      Vec<Dv<K>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) X[q][c].v = a.x[(int64_t)vid[q] * N + c];
      ev = jit_value(f.template operator()<N>(a.attrs, e, X));
    } else if constexpr (MODE == JIT_GRAD) {
      Vec<Dg<K>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          X[q][c].v = a.x[(int64_t)vid[q] * N + c];
#pragma unroll
          for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c && fr[q]) ? 1.0 : 0.0;
        }
      auto r = f.template operator()<N>(a.attrs, e, X);
      ev = r.v;
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (fr[q])
#pragma unroll
          for (int c = 0; c < N; ++c) jit_put_vec(a, a.grad, e, P, q, N, c, vid[q], r.g[q * N + c]);
    } else if constexpr (MODE == JIT_HESS || (MODE == JIT_HVP && PSD)) {
      Vec<Dh<K, true>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          X[q][c].v = a.x[(int64_t)vid[q] * N + c];
#pragma unroll
          for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c && fr[q]) ? 1.0 : 0.0;
        }
      auto r = f.template operator()<N>(a.attrs, e, X);
      using R = decltype(r);
      ev = r.v;
      if constexpr (MODE == JIT_HESS) {
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (fr[q])
#pragma unroll
            for (int c = 0; c < N; ++c) jit_put_vec(a, a.grad, e, P, q, N, c, vid[q], r.g[q * N + c]);
      }
      if constexpr (!R::kZero || PSD) {
        double h[TriN<K>::value];
        if constexpr (R::kZero) {
#pragma unroll
          for (int i = 0; i < TriN<K>::value; ++i) h[i] = 0.0;
        } else {
#pragma unroll
          for (int i = 0; i < TriN<K>::value; ++i) h[i] = r.h[i];
        }
        if constexpr (PSD) extract_psd<P, N>(h, a.floor);
        else {
#pragma unroll
          for (int i = 0; i < TriN<K>::value; ++i) h[i] = 0.5 * (h[i] + h[i]);
        }
        if constexpr (MODE == JIT_HESS) {
          const int32_t* b = a.bids + e * P * P;
#pragma unroll
          for (int q1 = 0; q1 < P; ++q1)
#pragma unroll
            for (int q2 = 0; q2 < P; ++q2) {
              const int32_t bid = b[q1 * P + q2];
              if (bid >= 0) {
                if (a.sh) {
                  double* dst = a.sh + ((e * P + q1) * P + q2) * N * N;
#pragma unroll
                  for (int rr = 0; rr < N; ++rr)
#pragma unroll
                    for (int cc = 0; cc < N; ++cc) dst[rr * N + cc] = h[tri(q1 * N + rr, q2 * N + cc)];
                } else {
                  double* dst = a.hess + (int64_t)bid * N * N;
#pragma unroll
                  for (int rr = 0; rr < N; ++rr)
#pragma unroll
                    for (int cc = 0; cc < N; ++cc) atomicAdd(dst + rr * N + cc, h[tri(q1 * N + rr, q2 * N + cc)]);
                }
              }
            }
        } else {
          double vl[K];
#pragma unroll
          for (int q = 0; q < P; ++q)
#pragma unroll
            for (int c = 0; c < N; ++c) vl[q * N + c] = fr[q] ? a.w[(int64_t)vid[q] * N + c] : 0.0;
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (fr[q])
#pragma unroll
              for (int c = 0; c < N; ++c) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < K; ++j) acc += h[tri(q * N + c, j)] * vl[j];
                jit_put_vec(a, a.y, e, P, q, N, c, vid[q], acc);
              }
        }
      } else if constexpr (MODE == JIT_HESS) {
        if (a.sh) {  // structural-zero Hessian: zero blocks for the gather
          const int32_t* b = a.bids + e * P * P;
          for (int k = 0; k < P * P; ++k)
            if (b[k] >= 0)
              for (int i = 0; i < N * N; ++i) a.sh[(e * P * P + k) * N * N + i] = 0.0;
        }
      }
    } else {  // JIT_HVP without PSD: forward-over-forward
      Vec<Df<K, true>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          X[q][c].v = a.x[(int64_t)vid[q] * N + c];
          X[q][c].vd = fr[q] ? a.w[(int64_t)vid[q] * N + c] : 0.0;
#pragma unroll
          for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c && fr[q]) ? 1.0 : 0.0;
        }
      auto r = f.template operator()<N>(a.attrs, e, X);
      using R = decltype(r);
      if constexpr (!R::kZero) {
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (fr[q])
#pragma unroll
            for (int c = 0; c < N; ++c) jit_put_vec(a, a.y, e, P, q, N, c, vid[q], r.gd[q * N + c]);
      } else if (a.sv) {
        for (int i = 0; i < P * N; ++i) a.sv[e * P * N + i] = 0.0;
      }
    }
  }
  if constexpr (MODE != JIT_HVP) {
    if (a.owned && e < a.M && !a.owned[a.sel ? a.sel[e * P] : e]) ev = 0.0;
    // fixed-order block sum
    __shared__ double ws[JIT_TPB / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ev += __shfl_down_sync(0xffffffffu, ev, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = ev;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < JIT_TPB / 32; ++i) s += ws[i];
      a.partials[blockIdx.x] = s;
    }
  }
}

}  // namespace mg

#define MG_JIT_KERNEL(F, P, N, NAME, MODE, PSD)                                           \
  extern "C" __global__ void __launch_bounds__(mg::JIT_TPB) NAME(const __grid_constant__ mg::JitArgs a) { \
    mg::jit_element<F, P, N, MODE, PSD>(a);                                                \
  }

#define MG_JIT_INSTANTIATE(F, P, N)                                \
  MG_JIT_KERNEL(F, P, N, mg_jit_energy, mg::JIT_ENERGY, false)     \
  MG_JIT_KERNEL(F, P, N, mg_jit_grad, mg::JIT_GRAD, false)         \
  MG_JIT_KERNEL(F, P, N, mg_jit_hess, mg::JIT_HESS, false)         \
  MG_JIT_KERNEL(F, P, N, mg_jit_hess_psd, mg::JIT_HESS, true)      \
  MG_JIT_KERNEL(F, P, N, mg_jit_hvp, mg::JIT_HVP, false)           \
  MG_JIT_KERNEL(F, P, N, mg_jit_hvp_psd, mg::JIT_HVP, true)
