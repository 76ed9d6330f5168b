// Deterministic patch-owner assembly: one CTA per vertex patch.
//
// A CTA owns R consecutive rows (Morton order) of the gradient / HVP / block
// Hessian. It
//   1. stages x (and the HVP direction) of its owned + ribbon vertices in
//      shared memory,
//   2. evaluates the V terms of its owned vertices (one thread per row),
//   3. evaluates every EV / FV element incident to an owned row (ribbon
//      elements are evaluated by each owning patch), holding the element's
//      dual-number result in registers, and adds the owned-row parts into
//      shared-memory row accumulators in conflict-free color phases
//      (elements are pre-sorted by color: a fixed, race-free summation order),
//   4. writes each owned row once, coalesced: no memset, no atomics, bitwise
//      reproducible.
// The energy is summed per patch over the elements whose first vertex is
// owned, then reduced in fixed order.
//
// Term types dispatch at runtime inside the kernel (warp-uniform switch);
// families bound which types are compiled in, to keep register allocation of
// light problems (cloth) independent of heavy terms (sphere).
#include "mg_internal.cuh"
#include "psd.cuh"

namespace mg {

namespace {

constexpr int PT = 128;  // threads per patch CTA
constexpr int MAXT = 8;

struct OpView {
  const int32_t* off;
  const int32_t* elem;
  const uint16_t* local;
  const uint8_t* pos;
  const uint8_t* color;
};

struct PatchArgs {
  int R;
  int nterms;
  int64_t V;
  const int32_t* vtx_off;
  const int32_t* vtx;
  const int32_t* hloc;
  const uint8_t* diag_pos;
  const int64_t* row_offsets;
  const uint8_t* fixed;
  const double* x;
  const double* w;
  double* grad;
  double* hess;
  double* y;
  double* partials;
  double floor;
  OpView ev, fv;
  TermDev terms[MAXT];
};

// shared-memory carve-up
struct Smem {
  double* xs;     // (nvp, N)
  double* ws;     // (nvp, N)   HVP direction
  double* acc;    // (R, N)     grad / y rows
  double* hacc;   // (blocks, N, N)
  int* vid;       // (nvp)
  int* hl;        // (R)
  uint8_t* fx;    // (nvp)
};

template <int N, int MODE>
__device__ __forceinline__ Smem carve(double* base, int R, int nvp_max, int blocks_max) {
  Smem s;
  double* d = base;
  s.xs = d; d += (size_t)nvp_max * N;
  s.ws = d; if (MODE == MODE_HVP) d += (size_t)nvp_max * N;
  s.acc = d; d += (size_t)R * N;
  s.hacc = d; if (MODE == MODE_HESS) d += (size_t)blocks_max * N * N;
  int* i = reinterpret_cast<int*>(d);
  s.vid = i; i += nvp_max;
  s.hl = i; i += R;
  s.fx = reinterpret_cast<uint8_t*>(i);
  return s;
}

__device__ double block_sum(double v) {
  __shared__ double ws[PT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < PT / 32; ++i) r += ws[i];
  return r;
}

// Evaluate one element: dual result -> value + per-slot contributions.
//   MODE_GRAD: g[K];  MODE_HESS: g[K] and packed h (valid flag);
//   MODE_HVP: hv[K] (H v, PSD-clamped if requested).
template <int TT, int N, int MODE, bool PSD>
struct ElemOut {
  static constexpr int P = TermInfo<TT>::P, K = P * N;
  double val;
  double g[K];
  double h[(MODE == MODE_HESS) ? TriN<K>::value : 1];
  bool has_h;
};

template <int TT, int N, int MODE, bool PSD>
__device__ __forceinline__ void eval_element(const TermDev& t, int64_t e, const int* vid, const double* const* xr,
                                             const double* const* wr, const bool* fr, double floor,
                                             ElemOut<TT, N, MODE, PSD>& o) {
  constexpr int P = TermInfo<TT>::P, K = P * N;
  if constexpr (MODE == MODE_ENERGY) {
    Vec<Dv<K>, N> X[P];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < N; ++c) X[q][c].v = xr[q][c];
    o.val = term_eval<TT, N>(t, e, vid, X).v;
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
    auto r = term_eval<TT, N>(t, e, vid, X);
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
    auto r = term_eval<TT, N>(t, e, vid, X);
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
    auto r = term_eval<TT, N>(t, e, vid, X);
    using R = decltype(r);
    o.val = r.v;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if constexpr (R::kZero) o.g[i] = 0.0;
      else o.g[i] = r.gd[i];
    }
  }
}

// V terms: one thread per owned row, no conflicts.
template <int TT, int N, int MODE, bool PSD>
__device__ __forceinline__ void run_vterm(const PatchArgs& a, const TermDev& t, const Smem& s, int oc,
                                          double& eacc) {
  for (int r = threadIdx.x; r < oc; r += PT) {
    const int v = s.vid[r];
    const bool fr = !s.fx[r];
    const double* xr[1] = {s.xs + r * N};
    const double* wr[1] = {s.ws + r * N};
    ElemOut<TT, N, MODE, PSD> o;
    eval_element<TT, N, MODE, PSD>(t, v, &v, xr, wr, &fr, a.floor, o);
    eacc += o.val;
    if (fr) {
      if constexpr (MODE != MODE_ENERGY) {
#pragma unroll
        for (int c = 0; c < N; ++c) s.acc[r * N + c] += o.g[c];
      }
      if constexpr (MODE == MODE_HESS) {
        const int dp = a.diag_pos[v];
        if (o.has_h && dp != 255) {
          double* blk = s.hacc + (size_t)(s.hl[r] + dp) * N * N;
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) blk[i * N + j] += o.h[tri(i, j)];
        }
      }
    }
  }
}

// EV / FV terms over the patch's element list, in color phases.
template <int TT, int N, int MODE, bool PSD>
__device__ __forceinline__ void run_eterm(const PatchArgs& a, const TermDev& t, const OpView& L, int p,
                                          const Smem& s, int oc, double& eacc) {
  constexpr int P = TermInfo<TT>::P;
  const int j0 = L.off[p], j1 = L.off[p + 1];
  for (int base = j0; base < j1; base += PT) {
    const int j = base + threadIdx.x;
    const bool act = j < j1;
    int lq[P], vid[P];
    bool fr[P];
    int color = -1;
    ElemOut<TT, N, MODE, PSD> o;
    if (act) {
      const int64_t e = L.elem[j];
      color = L.color[j];
      const double* xr[P];
      const double* wr[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        lq[q] = L.local[(int64_t)j * P + q];
        vid[q] = s.vid[lq[q]];
        fr[q] = !s.fx[lq[q]];
        xr[q] = s.xs + lq[q] * N;
        wr[q] = s.ws + lq[q] * N;
      }
      eval_element<TT, N, MODE, PSD>(t, e, vid, xr, wr, fr, a.floor, o);
      if (lq[0] < oc) eacc += o.val;
    }
    const int clo = L.color[base];
    const int chi = L.color[min(base + PT, j1) - 1];
    for (int c = clo; c <= chi; ++c) {
      if (act && color == c) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
          if (lq[q] < oc && fr[q]) {
            if constexpr (MODE != MODE_ENERGY) {
#pragma unroll
              for (int cc = 0; cc < N; ++cc) s.acc[lq[q] * N + cc] += o.g[q * N + cc];
            }
            if constexpr (MODE == MODE_HESS) {
              if (o.has_h) {
                const uint8_t* pq = L.pos + ((int64_t)j * P + q) * P;
                const int hb = s.hl[lq[q]];
#pragma unroll
                for (int q2 = 0; q2 < P; ++q2) {
                  const int ps = pq[q2];
                  if (ps != 255) {
                    double* blk = s.hacc + (size_t)(hb + ps) * N * N;
#pragma unroll
                    for (int i = 0; i < N; ++i)
#pragma unroll
                      for (int k = 0; k < N; ++k) blk[i * N + k] += o.h[tri(q * N + i, q2 * N + k)];
                  }
                }
              }
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

// type masks of the compiled families
constexpr unsigned bit(int t) { return 1u << t; }
constexpr unsigned FAM_LIGHT = bit(MG_TERM_INERTIA) | bit(MG_TERM_SPRING) | bit(MG_TERM_GRAVITY) | bit(MG_TERM_EDGE_LENGTH);
constexpr unsigned FAM_UV = FAM_LIGHT | bit(MG_TERM_SYM_DIRICHLET);
constexpr unsigned FAM_ALL = FAM_UV | bit(MG_TERM_SPHERE);

template <int N, unsigned FAM, int MODE, bool PSD>
__global__ void __launch_bounds__(PT) k_patch(const __grid_constant__ PatchArgs a, int nvp_max, int blocks_max) {
  extern __shared__ __align__(16) double smem[];
  const int p = blockIdx.x;
  const int R = a.R;
  const int64_t own0 = (int64_t)p * R;
  const int oc = (int)min((int64_t)R, a.V - own0);
  const int v0 = a.vtx_off[p];
  const int nvp = a.vtx_off[p + 1] - v0;
  Smem s = carve<N, MODE>(smem, R, nvp_max, blocks_max);

  // stage patch vertices
  for (int i = threadIdx.x; i < nvp; i += PT) {
    const int g = a.vtx[v0 + i];
    s.vid[i] = g;
    s.fx[i] = a.fixed ? a.fixed[g] : 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nvp * N; i += PT) {
    const int li = i / N, c = i - li * N;
    const int64_t g = s.vid[li];
    s.xs[i] = a.x[g * N + c];
    if constexpr (MODE == MODE_HVP) s.ws[i] = a.w[g * N + c];
  }
  for (int i = threadIdx.x; i < oc * N; i += PT) s.acc[i] = 0.0;
  int nblk = 0;
  if constexpr (MODE == MODE_HESS) {
    for (int r = threadIdx.x; r < oc; r += PT) s.hl[r] = a.hloc[own0 + r];
    const int64_t last = own0 + oc - 1;
    const int lv = a.vtx[v0 + oc - 1];
    nblk = a.hloc[last] + (int)(a.row_offsets[lv + 1] - a.row_offsets[lv]);
    for (int i = threadIdx.x; i < nblk * N * N; i += PT) s.hacc[i] = 0.0;
  }
  __syncthreads();

  double eacc = 0.0;
  for (int ti = 0; ti < a.nterms; ++ti) {
    const TermDev& t = a.terms[ti];
    if (t.op != MG_OP_V) continue;
    switch (t.type) {
      case MG_TERM_INERTIA:
        if constexpr ((FAM & bit(MG_TERM_INERTIA)) != 0) run_vterm<MG_TERM_INERTIA, N, MODE, PSD>(a, t, s, oc, eacc);
        break;
      case MG_TERM_GRAVITY:
        if constexpr ((FAM & bit(MG_TERM_GRAVITY)) != 0) run_vterm<MG_TERM_GRAVITY, N, MODE, PSD>(a, t, s, oc, eacc);
        break;
      default: break;
    }
  }
  __syncthreads();
  for (int ti = 0; ti < a.nterms; ++ti) {
    const TermDev& t = a.terms[ti];
    switch (t.type) {
      case MG_TERM_SPRING:
        if constexpr ((FAM & bit(MG_TERM_SPRING)) != 0) run_eterm<MG_TERM_SPRING, N, MODE, PSD>(a, t, a.ev, p, s, oc, eacc);
        break;
      case MG_TERM_EDGE_LENGTH:
        if constexpr ((FAM & bit(MG_TERM_EDGE_LENGTH)) != 0) run_eterm<MG_TERM_EDGE_LENGTH, N, MODE, PSD>(a, t, a.ev, p, s, oc, eacc);
        break;
      case MG_TERM_SYM_DIRICHLET:
        if constexpr ((FAM & bit(MG_TERM_SYM_DIRICHLET)) != 0 && N == 2) run_eterm<MG_TERM_SYM_DIRICHLET, N, MODE, PSD>(a, t, a.fv, p, s, oc, eacc);
        break;
      case MG_TERM_SPHERE:
        if constexpr ((FAM & bit(MG_TERM_SPHERE)) != 0 && N == 2) run_eterm<MG_TERM_SPHERE, N, MODE, PSD>(a, t, a.fv, p, s, oc, eacc);
        break;
      default: break;
    }
  }
  __syncthreads();

  // write owned rows once
  double* vout = MODE == MODE_HVP ? a.y : a.grad;
  for (int i = threadIdx.x; i < oc * N; i += PT) {
    const int r = i / N, c = i - r * N;
    vout[(int64_t)s.vid[r] * N + c] = s.acc[i];
  }
  if constexpr (MODE == MODE_HESS) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int r = wid; r < oc; r += PT / 32) {
      const int g = s.vid[r];
      const int64_t ro = a.row_offsets[g];
      const int cnt = (int)(a.row_offsets[g + 1] - ro) * N * N;
      const double* src = s.hacc + (size_t)s.hl[r] * N * N;
      double* dst = a.hess + ro * N * N;
      for (int k = lane; k < cnt; k += 32) dst[k] = src[k];
    }
  }
  if constexpr (MODE != MODE_HVP) {
    const double tot = block_sum(eacc);
    if (threadIdx.x == 0) a.partials[p] = tot;
  }
}


// ---------------------------------------------------------------------------
// Two-point edge fast path (every term is a V term or a two-point EV term:
// cloth, smoothing). Per patch CTA:
//   stage 1  every patch edge once: K = n dual on d = x_i - x_j (bitwise equal
//            to the reference's K = 2n dual, see TwoPoint in terms.cuh); the
//            result (value, g, A or its PSD clamp, floor shift) goes to a
//            shared-memory scratch slot;
//   stage 2  one thread per owned row: V terms + its incident edges in column
//            order (fixed summation order -> bitwise reproducible), gradient /
//            HVP row written, diagonal block kept in shared memory;
//   stage 3  one warp per owned row writes the row's blocks with coalesced
//            stores: off-diagonal block (i,j) = -M_e + delta_e I of the unique
//            edge (i,j), diagonal = the stage-2 sum.
// No color phases: three barriers per patch.
struct EvArgs {
  int R;
  int nterms;
  int64_t V;
  const int32_t* vtx_off;
  const int32_t* vtx;
  const int32_t* ev_off;
  const int32_t* ev_elem;
  const uint16_t* ev_local;
  const int32_t* rinc_off;
  const uint32_t* rinc;
  const int32_t* hloc;
  const uint8_t* diag_pos;
  const int64_t* row_offsets;
  const uint8_t* fixed;
  const double* x;
  const double* w;
  double* grad;
  double* hess;
  double* y;
  double* partials;
  double floor;
  TermDev terms[MAXT];
};

template <int N, int MODE, bool PSD>
struct EvLayout {
  static constexpr int T = TriN<N>::value;
  // scratch doubles per edge
  static constexpr int SW = MODE == MODE_GRAD ? 1 + N : MODE == MODE_HESS ? 1 + N + T + 1 : (PSD ? 2 * N : N);
};

template <int N, int MODE, bool PSD>
__device__ __forceinline__ void ev_stage1_edge(const EvArgs& a, int64_t e, const double* xa, const double* xb,
                                               const double* wa, const double* wb, bool fa, bool fb, double* out) {
  using L = EvLayout<N, MODE, PSD>;
  constexpr int T = L::T;
  double acc[L::SW];
#pragma unroll
  for (int i = 0; i < L::SW; ++i) acc[i] = 0.0;
  for (int ti = 0; ti < a.nterms; ++ti) {
    const TermDev& t = a.terms[ti];
    if (t.op != MG_OP_EV) continue;
    const int tt = t.type;
    if constexpr (MODE == MODE_GRAD) {
      Vec<Dg<N>, N> d;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        d[c].v = xa[c] - xb[c];
#pragma unroll
        for (int i = 0; i < N; ++i) d[c].g[i] = (i == c) ? 1.0 : 0.0;
      }
      auto r = tt == MG_TERM_SPRING ? term_eval_diff<MG_TERM_SPRING, N>(t, e, d) : term_eval_diff<MG_TERM_EDGE_LENGTH, N>(t, e, d);
      acc[0] += r.v;
#pragma unroll
      for (int i = 0; i < N; ++i) acc[1 + i] += r.g[i];
    } else if constexpr (MODE == MODE_HESS || (MODE == MODE_HVP && PSD)) {
      Vec<Dh<N, true>, N> d;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        d[c].v = xa[c] - xb[c];
#pragma unroll
        for (int i = 0; i < N; ++i) d[c].g[i] = (i == c) ? 1.0 : 0.0;
      }
      auto r = tt == MG_TERM_SPRING ? term_eval_diff<MG_TERM_SPRING, N>(t, e, d) : term_eval_diff<MG_TERM_EDGE_LENGTH, N>(t, e, d);
      double h[T];
#pragma unroll
      for (int i = 0; i < T; ++i) h[i] = 0.5 * (r.h[i] + r.h[i]);
      double dl = 0.0;
      if constexpr (PSD) {
        if (all_finite<N>(h)) {
          if (fa && fb) {
#pragma unroll
            for (int i = 0; i < T; ++i) h[i] = 2.0 * h[i];
            project_if_needed<N>(h, a.floor);
#pragma unroll
            for (int i = 0; i < T; ++i) h[i] = 0.5 * h[i];
            dl = 0.5 * a.floor;
          } else if (fa || fb) {
            project_if_needed<N>(h, a.floor);
          }
        }
      }
      if constexpr (MODE == MODE_HESS) {
        acc[0] += r.v;
#pragma unroll
        for (int i = 0; i < N; ++i) acc[1 + i] += r.g[i];
#pragma unroll
        for (int i = 0; i < T; ++i) acc[1 + N + i] += h[i];
        acc[1 + N + T] += dl;
      } else {
        // y_a = M (wa - wb) + dl (wa + wb), y_b = -M (wa - wb) + dl (wa + wb);
        // one free endpoint: y_free = P(A) w_free
        double wd[N], ws[N];
#pragma unroll
        for (int c = 0; c < N; ++c) {
          const double ua = fa ? wa[c] : 0.0, ub = fb ? wb[c] : 0.0;
          wd[c] = ua - ub;
          ws[c] = ua + ub;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double m = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) m += h[tri(i, j)] * wd[j];
          acc[i] += m + dl * ws[i];
          acc[N + i] += -m + dl * ws[i];
        }
      }
    } else {  // HVP, forward-over-forward on d with direction (wa - wb) (free-masked)
      Vec<Df<N, true>, N> d;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        d[c].v = xa[c] - xb[c];
        d[c].vd = (fa ? wa[c] : 0.0) - (fb ? wb[c] : 0.0);
#pragma unroll
        for (int i = 0; i < N; ++i) d[c].g[i] = (i == c) ? 1.0 : 0.0;
      }
      auto r = tt == MG_TERM_SPRING ? term_eval_diff<MG_TERM_SPRING, N>(t, e, d) : term_eval_diff<MG_TERM_EDGE_LENGTH, N>(t, e, d);
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] += r.gd[i];
    }
  }
#pragma unroll
  for (int i = 0; i < L::SW; ++i) out[i] = acc[i];
}

template <int N, int MODE, bool PSD>
__global__ void __launch_bounds__(PT) k_patch_ev(const __grid_constant__ EvArgs a, int nvp_max, int ne_max,
                                                  int blocks_max) {
  using L = EvLayout<N, MODE, PSD>;
  constexpr int T = L::T, SW = L::SW, NN = N * N;
  extern __shared__ __align__(16) double smem[];
  const int p = blockIdx.x;
  const int R = a.R;
  const int64_t own0 = (int64_t)p * R;
  const int oc = (int)min((int64_t)R, a.V - own0);
  const int v0 = a.vtx_off[p];
  const int nvp = a.vtx_off[p + 1] - v0;
  const int j0 = a.ev_off[p];
  const int ne = a.ev_off[p + 1] - j0;

  double* xs = smem;
  double* ws = xs + (size_t)nvp_max * N;
  double* scr = ws + (MODE == MODE_HVP ? (size_t)nvp_max * N : 0);
  double* rdiag = scr + (size_t)ne_max * SW;
  int64_t* sro = reinterpret_cast<int64_t*>(rdiag + (MODE == MODE_HESS ? (size_t)R * T : 0));
  int* vid = reinterpret_cast<int*>(sro + (MODE == MODE_HESS ? R : 0));
  int* shl = vid + nvp_max;
  int* slen = shl + R;
  int16_t* map = reinterpret_cast<int16_t*>(slen + R);
  uint8_t* fx = reinterpret_cast<uint8_t*>(map + (MODE == MODE_HESS ? blocks_max : 0));

  // stage 0: patch vertices
  for (int i = threadIdx.x; i < nvp; i += PT) {
    const int g = a.vtx[v0 + i];
    vid[i] = g;
    fx[i] = a.fixed ? a.fixed[g] : 0;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      xs[i * N + c] = a.x[(int64_t)g * N + c];
      if constexpr (MODE == MODE_HVP) ws[i * N + c] = a.w[(int64_t)g * N + c];
    }
  }
  if constexpr (MODE == MODE_HESS) {
    for (int r = threadIdx.x; r < oc; r += PT) {
      const int g = a.vtx[v0 + r];
      const int64_t ro = a.row_offsets[g];
      sro[r] = ro;
      slen[r] = (int)(a.row_offsets[g + 1] - ro);
      shl[r] = a.hloc[own0 + r];
    }
  }
  __syncthreads();

  // stage 1: every patch edge once (records of the next edge prefetched)
  {
    int jj = threadIdx.x;
    int64_t e = 0;
    uint32_t lab = 0;
    if (jj < ne) {
      e = a.ev_elem[j0 + jj];
      lab = reinterpret_cast<const uint32_t*>(a.ev_local)[j0 + jj];
    }
    for (; jj < ne; jj += PT) {
      const int64_t ce = e;
      const uint32_t clab = lab;
      if (jj + PT < ne) {
        e = a.ev_elem[j0 + jj + PT];
        lab = reinterpret_cast<const uint32_t*>(a.ev_local)[j0 + jj + PT];
      }
      const int la = clab & 0xffff, lb = clab >> 16;
      ev_stage1_edge<N, MODE, PSD>(a, ce, xs + la * N, xs + lb * N, ws + la * N, ws + lb * N, !fx[la], !fx[lb],
                                   scr + (size_t)jj * SW);
    }
  }
  __syncthreads();

  // stage 2: one thread per owned row
  double eacc = 0.0;
  for (int r = threadIdx.x; r < oc; r += PT) {
    const int g = vid[r];
    const bool fr = !fx[r];
    double vec[N];
    double dg[T];
#pragma unroll
    for (int i = 0; i < N; ++i) vec[i] = 0.0;
#pragma unroll
    for (int i = 0; i < T; ++i) dg[i] = 0.0;
    // V terms
    for (int ti = 0; ti < a.nterms; ++ti) {
      const TermDev& t = a.terms[ti];
      if (t.op != MG_OP_V) continue;
      const double* xr[1] = {xs + r * N};
      const double* wr[1] = {ws + r * N};
      const int vv = g;
      if (t.type == MG_TERM_INERTIA) {
        ElemOut<MG_TERM_INERTIA, N, MODE, PSD> o;
        eval_element<MG_TERM_INERTIA, N, MODE, PSD>(t, g, &vv, xr, wr, &fr, a.floor, o);
        eacc += o.val;
#pragma unroll
        for (int i = 0; i < N; ++i) vec[i] += o.g[i];
        if constexpr (MODE == MODE_HESS) {
          if (o.has_h)
#pragma unroll
            for (int i = 0; i < T; ++i) dg[i] += o.h[i];
        }
      } else if (t.type == MG_TERM_GRAVITY) {
        ElemOut<MG_TERM_GRAVITY, N, MODE, PSD> o;
        eval_element<MG_TERM_GRAVITY, N, MODE, PSD>(t, g, &vv, xr, wr, &fr, a.floor, o);
        eacc += o.val;
#pragma unroll
        for (int i = 0; i < N; ++i) vec[i] += o.g[i];
        if constexpr (MODE == MODE_HESS) {
          if (o.has_h)
#pragma unroll
            for (int i = 0; i < T; ++i) dg[i] += o.h[i];
        }
      }
    }
    // incident edges, column order
    const int k0 = a.rinc_off[own0 + r], k1 = a.rinc_off[own0 + r + 1];
    for (int k = k0; k < k1; ++k) {
      const uint32_t rec = a.rinc[k];
      const int jj = rec & 0xffff;
      const int q = (rec >> 16) & 1;
      const double* sc = scr + (size_t)jj * SW;
      if constexpr (MODE == MODE_GRAD || MODE == MODE_HESS) {
        if (q == 0) eacc += sc[0];
        const double sg = q == 0 ? 1.0 : -1.0;
#pragma unroll
        for (int i = 0; i < N; ++i) vec[i] += sg * sc[1 + i];
      }
      if constexpr (MODE == MODE_HESS) {
        const double dl = sc[1 + N + T];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int c = 0; c <= i; ++c) dg[tri(i, c)] += sc[1 + N + tri(i, c)] + (i == c ? dl : 0.0);
        const int pos = rec >> 24;
        if (pos != 255) map[shl[r] + pos] = (int16_t)jj;
      }
      if constexpr (MODE == MODE_HVP) {
        if constexpr (PSD) {
#pragma unroll
          for (int i = 0; i < N; ++i) vec[i] += sc[q * N + i];
        } else {
          const double sg = q == 0 ? 1.0 : -1.0;
#pragma unroll
          for (int i = 0; i < N; ++i) vec[i] += sg * sc[i];
        }
      }
    }
    double* vout = MODE == MODE_HVP ? a.y : a.grad;
#pragma unroll
    for (int i = 0; i < N; ++i) vout[(int64_t)g * N + i] = fr ? vec[i] : 0.0;
    if constexpr (MODE == MODE_HESS) {
#pragma unroll
      for (int i = 0; i < T; ++i) rdiag[r * T + i] = dg[i];
      const int dp = a.diag_pos[g];
      if (fr && dp != 255) map[shl[r] + dp] = -1;
    }
  }
  if constexpr (MODE == MODE_HESS) {
    __syncthreads();
    // stage 3: one warp per owned row, coalesced block writes. Each lane owns
    // a fixed (block-in-group, entry) slot: BPW = 32 / NN blocks per pass.
    constexpr int BPW = 32 / NN;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int lb = lane / NN, lrc = lane - lb * NN, li = lrc / N, lc = lrc - li * N;
    const int ltri = li >= lc ? li * (li + 1) / 2 + lc : lc * (lc + 1) / 2 + li;
    const bool ldiag = li == lc;
    if (lb < BPW) {
      for (int r = wid; r < oc; r += PT / 32) {
        const int len = slen[r];
        double* dst = a.hess + sro[r] * NN;
        const int hb = shl[r];
        const double* rd = rdiag + r * T;
        for (int b = lb; b < len; b += BPW) {
          const int jj = map[hb + b];
          double v;
          if (jj < 0) {
            v = rd[ltri];
          } else {
            const double* sc = scr + (size_t)jj * SW;
            v = -sc[1 + N + ltri] + (ldiag ? sc[1 + N + T] : 0.0);
          }
          dst[b * NN + lrc] = v;
        }
      }
    }
  }
  if constexpr (MODE != MODE_HVP) {
    const double tot = block_sum(eacc);
    if (threadIdx.x == 0) a.partials[p] = tot;
  }
}

size_t ev_smem_bytes(int N, int mode, bool psd, int R, int nvp_max, int ne_max, int blocks_max) {
  const int T = N * (N + 1) / 2;
  const int SW = mode == MODE_GRAD ? 1 + N : mode == MODE_HESS ? 1 + N + T + 1 : (psd ? 2 * N : N);
  size_t b = 8 * ((size_t)nvp_max * N + (mode == MODE_HVP ? (size_t)nvp_max * N : 0) + (size_t)ne_max * SW +
                  (mode == MODE_HESS ? (size_t)R * T + R : 0));
  b += 4 * ((size_t)nvp_max + 2 * R) + (mode == MODE_HESS ? 2 * (size_t)blocks_max : 0) + nvp_max + 16;
  return b;
}

template <int N, int MODE, bool PSD>
void launch_ev(const EvArgs& a, int64_t np, int nvp_max, int ne_max, int blocks_max, cudaStream_t st) {
  auto kern = k_patch_ev<N, MODE, PSD>;
  const size_t sm = ev_smem_bytes(N, MODE, PSD, a.R, nvp_max, ne_max, blocks_max);
  if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "patch does not fit in shared memory");
  MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  kern<<<(unsigned)np, PT, sm, st>>>(a, nvp_max, ne_max, blocks_max);
  MG_LAUNCH_CHECK();
}

template <int N>
void launch_ev_mode(const EvArgs& a, int64_t np, int nvp, int ne, int nb, Mode mode, bool psd, cudaStream_t st) {
  switch (mode) {
    case MODE_GRAD: launch_ev<N, MODE_GRAD, false>(a, np, nvp, ne, nb, st); break;
    case MODE_HESS:
      if (psd) launch_ev<N, MODE_HESS, true>(a, np, nvp, ne, nb, st);
      else launch_ev<N, MODE_HESS, false>(a, np, nvp, ne, nb, st);
      break;
    case MODE_HVP:
      if (psd) launch_ev<N, MODE_HVP, true>(a, np, nvp, ne, nb, st);
      else launch_ev<N, MODE_HVP, false>(a, np, nvp, ne, nb, st);
      break;
    default: throw Error(MG_ERR_UNSUPPORTED, "edge fast path assembles grad / Hessian / HVP only");
  }
}


size_t smem_bytes(int N, int mode, int R, int nvp_max, int blocks_max) {
  size_t d = (size_t)nvp_max * N + (mode == MODE_HVP ? (size_t)nvp_max * N : 0) + (size_t)R * N +
             (mode == MODE_HESS ? (size_t)blocks_max * N * N : 0);
  return d * 8 + (size_t)(nvp_max + R) * 4 + (size_t)nvp_max + 16;
}

template <int N, unsigned FAM, int MODE, bool PSD>
void launch_fam(const PatchArgs& a, int64_t np, int nvp_max, int blocks_max, cudaStream_t st) {
  auto kern = k_patch<N, FAM, MODE, PSD>;
  const size_t sm = smem_bytes(N, MODE, a.R, nvp_max, blocks_max);
  if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "patch does not fit in shared memory");
  MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  kern<<<(unsigned)np, PT, sm, st>>>(a, nvp_max, blocks_max);
  MG_LAUNCH_CHECK();
}

template <int N, unsigned FAM>
void launch_mode(const PatchArgs& a, int64_t np, int nvp, int nb, Mode mode, bool psd, cudaStream_t st) {
  switch (mode) {
    case MODE_GRAD: launch_fam<N, FAM, MODE_GRAD, false>(a, np, nvp, nb, st); break;
    case MODE_HESS:
      if (psd) launch_fam<N, FAM, MODE_HESS, true>(a, np, nvp, nb, st);
      else launch_fam<N, FAM, MODE_HESS, false>(a, np, nvp, nb, st);
      break;
    case MODE_HVP:
      if (psd) launch_fam<N, FAM, MODE_HVP, true>(a, np, nvp, nb, st);
      else launch_fam<N, FAM, MODE_HVP, false>(a, np, nvp, nb, st);
      break;
    default: throw Error(MG_ERR_UNSUPPORTED, "patch kernels assemble grad / Hessian / HVP only");
  }
}

}  // namespace

bool patch_supported(const Problem& p) {
  if (p.terms.empty() || p.terms.size() > MAXT) return false;
  if (p.n != 2 && p.n != 3) return false;
  for (auto& t : p.terms)
    if (t.dev.op == MG_OP_VV) return false;
  return p.mesh->patches.num > 0;
}

int64_t launch_patch(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  const Mesh& m = *p.mesh;
  if (p.ev_fast) {
    EvArgs a;
    a.R = m.patches.R;
    a.nterms = (int)p.terms.size();
    a.V = m.Vr;
    a.vtx_off = p.vtx_off.p;
    a.vtx = p.vtx.p;
    a.ev_off = p.lay[0].off.p;
    a.ev_elem = p.lay[0].elem.p;
    a.ev_local = p.lay[0].local.p;
    a.rinc_off = p.rinc_off.p;
    a.rinc = p.rinc.p;
    a.hloc = p.hloc.p;
    a.diag_pos = p.diag_pos.p;
    a.row_offsets = p.row_offsets.p;
    a.fixed = p.any_fixed ? p.fixed.p : nullptr;
    a.x = c.x;
    a.w = c.w;
    a.grad = c.grad;
    a.hess = c.hess;
    a.y = c.y;
    a.partials = c.partials + partial_offset;
    a.floor = c.floor;
    for (int i = 0; i < a.nterms; ++i) a.terms[i] = p.terms[i].dev;
    const int64_t np = m.patches.num;
    if (p.n == 3) launch_ev_mode<3>(a, np, p.max_patch_vertices, p.max_patch_elems, p.max_patch_blocks, mode, c.psd, c.stream);
    else launch_ev_mode<2>(a, np, p.max_patch_vertices, p.max_patch_elems, p.max_patch_blocks, mode, c.psd, c.stream);
    return mode == MODE_HVP ? 0 : np;
  }
  PatchArgs a;
  a.R = m.patches.R;
  a.nterms = (int)p.terms.size();
  a.V = m.Vr;
  a.vtx_off = p.vtx_off.p;
  a.vtx = p.vtx.p;
  a.hloc = p.hloc.p;
  a.diag_pos = p.diag_pos.p;
  a.row_offsets = p.row_offsets.p;
  a.fixed = p.any_fixed ? p.fixed.p : nullptr;
  a.x = c.x;
  a.w = c.w;
  a.grad = c.grad;
  a.hess = c.hess;
  a.y = c.y;
  a.partials = c.partials + partial_offset;
  a.floor = c.floor;
  const OpLayout& ev = p.lay[0];
  const OpLayout& fv = p.lay[1];
  a.ev = OpView{ev.off.p, ev.elem.p, ev.local.p, ev.pos.p, ev.color.p};
  a.fv = OpView{fv.off.p, fv.elem.p, fv.local.p, fv.pos.p, fv.color.p};
  unsigned used = 0;
  for (int i = 0; i < a.nterms; ++i) {
    a.terms[i] = p.terms[i].dev;
    used |= 1u << p.terms[i].dev.type;
  }
  const int64_t np = m.patches.num;
  const int nvp = p.max_patch_vertices, nb = p.max_patch_blocks;
  if (p.n == 3) {
    if (used & ~FAM_LIGHT) throw Error(MG_ERR_UNSUPPORTED, "term not available for var_dim 3");
    launch_mode<3, FAM_LIGHT>(a, np, nvp, nb, mode, c.psd, c.stream);
  } else {
    if (used & bit(MG_TERM_SPHERE)) launch_mode<2, FAM_ALL>(a, np, nvp, nb, mode, c.psd, c.stream);
    else if (used & bit(MG_TERM_SYM_DIRICHLET)) launch_mode<2, FAM_UV>(a, np, nvp, nb, mode, c.psd, c.stream);
    else launch_mode<2, FAM_LIGHT>(a, np, nvp, nb, mode, c.psd, c.stream);
  }
  return mode == MODE_HVP ? 0 : np;
}

}  // namespace mg
