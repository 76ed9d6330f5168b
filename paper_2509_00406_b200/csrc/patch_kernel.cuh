// Patch-owner assembly kernel body, shared by the library's builtin terms
// (patch_kernels.cu) and traced callbacks (jit_patch.cuh, compiled at runtime
// with the generated functors): see patch_kernels.cu for the algorithm.
// A policy type supplies the terms:
//   template <int N, int MODE, bool PSD> static void vterms(a, s, oc, eacc);
//   template <int N, int MODE, bool PSD> static void eterms(a, p, s, oc, eacc);
// using run_vterm_g / run_eterm_g with an evaluator ev(e, vid, X).
#pragma once
#include "elem_eval.cuh"
#include "mg_internal.cuh"
#include "psd.cuh"

namespace mg {
namespace patch {

constexpr int PT = 128;  // threads per patch CTA
constexpr int MAXT = 8;
constexpr int JATTR = 64;  // attribute streams per traced term (== JIT_MAX_ATTRS)

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
  int64_t np;        // patches
  const int* redo;   // non-null: run only if *redo != 0 (exact re-run after a fast kernel)
  int* exact_runs;   // incremented once per executed re-run
  int64_t np_total;  // energy partials the reduction reads (> np: zero-fill the rest on a re-run)
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
  const double* const* jattr;  // traced terms: (nterms, JATTR) attribute stream pointers (device)
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

// V terms: one thread per owned row, no conflicts.
template <int N, int MODE, bool PSD, class EVAL>
__device__ __forceinline__ void run_vterm_g(const PatchArgs& a, const EVAL& ev, const Smem& s, int oc,
                                            double& eacc) {
  for (int r = threadIdx.x; r < oc; r += PT) {
    const int v = s.vid[r];
    const bool fr = !s.fx[r];
    const double* xr[1] = {s.xs + r * N};
    const double* wr[1] = {s.ws + r * N};
    ElemOutP<1, N, MODE, PSD> o;
    eval_element_f<1, N, MODE, PSD>(ev, v, &v, xr, wr, &fr, a.floor, o);
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
template <int P, int N, int MODE, bool PSD, class EVAL>
__device__ __forceinline__ void run_eterm_g(const PatchArgs& a, const EVAL& ev, const OpView& L, int p,
                                            const Smem& s, int oc, double& eacc) {
  const int j0 = L.off[p], j1 = L.off[p + 1];
  for (int base = j0; base < j1; base += PT) {
    const int j = base + threadIdx.x;
    const bool act = j < j1;
    int lq[P], vid[P];
    bool fr[P];
    int color = -1;
    ElemOutP<P, N, MODE, PSD> o;
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
      eval_element_f<P, N, MODE, PSD>(ev, e, vid, xr, wr, fr, a.floor, o);
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

// The kernel body: one CTA per patch (grid-stride over patches).
template <int N, int MODE, bool PSD, class Pol>
__device__ __forceinline__ void patch_body(const PatchArgs& a, int nvp_max, int blocks_max) {

  extern __shared__ __align__(16) double smem[];
  if (a.redo && *(volatile const int*)a.redo == 0) return;
  if (a.redo && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.exact_runs, 1);
  if constexpr (MODE != MODE_HVP) {
    for (int64_t i = a.np + blockIdx.x * (int64_t)PT + threadIdx.x; i < a.np_total; i += (int64_t)gridDim.x * PT)
      a.partials[i] = 0.0;
  }
  for (int64_t pp = blockIdx.x; pp < a.np; pp += gridDim.x) {
  __syncthreads();
  const int p = (int)pp;
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
  Pol::template vterms<N, MODE, PSD>(a, s, oc, eacc);
  __syncthreads();
  Pol::template eterms<N, MODE, PSD>(a, p, s, oc, eacc);
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
  }  // patches

}

// shared memory of one patch CTA
inline size_t smem_bytes(int N, int mode, int R, int nvp_max, int blocks_max) {
  size_t d = (size_t)nvp_max * N + (mode == MODE_HVP ? (size_t)nvp_max * N : 0) + (size_t)R * N +
             (mode == MODE_HESS ? (size_t)blocks_max * N * N : 0);
  return d * 8 + (size_t)(nvp_max + R) * 4 + (size_t)nvp_max + 16;
}

}  // namespace patch
}  // namespace mg
