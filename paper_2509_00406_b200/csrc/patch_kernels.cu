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
#include "elem_eval.cuh"

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
  }  // patches
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
  int64_t grid = np;
  if (a.redo) {  // exact re-run: a small persistent grid that exits unless the flag is raised
    int dev = 0, sms = 148;
    MG_CUDA(cudaGetDevice(&dev));
    MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = np < (int64_t)sms * 4 ? np : (int64_t)sms * 4;
  }
  kern<<<(unsigned)grid, PT, sm, st>>>(a, nvp_max, blocks_max);
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
    if (t.dev.op == MG_OP_VV || t.jit) return false;
  return p.mesh->patches.num > 0;
}

int64_t launch_patch(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  const Mesh& m = *p.mesh;
  if (p.ev_fast) return launch_patch_ev(p, mode, c, partial_offset);
  int64_t n_fast = 0;
  // face row kernels: Dirichlet in every mode; sphere for gradient / HVP
  const bool fast = p.fv_fast && (p.terms[0].dev.type != MG_TERM_SPHERE || mode == MODE_GRAD || mode == MODE_HVP);
  if (fast) n_fast = launch_patch_fv(p, mode, c, partial_offset);
  PatchArgs a;
  a.R = m.patches.R;
  a.nterms = (int)p.terms.size();
  a.V = m.Vr;
  a.np = m.patches.num;
  a.redo = fast ? p.redo.p : nullptr;  // after a face row kernel: exact re-run only on its flag
  a.exact_runs = p.exact_runs.p;
  a.np_total = n_fast;
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
  if (!fast) timing_begin(p, c.stream);
  if (p.n == 3) {
    if (used & ~FAM_LIGHT) throw Error(MG_ERR_UNSUPPORTED, "term not available for var_dim 3");
    launch_mode<3, FAM_LIGHT>(a, np, nvp, nb, mode, c.psd, c.stream);
  } else {
    if (used & bit(MG_TERM_SPHERE)) launch_mode<2, FAM_ALL>(a, np, nvp, nb, mode, c.psd, c.stream);
    else if (used & bit(MG_TERM_SYM_DIRICHLET)) launch_mode<2, FAM_UV>(a, np, nvp, nb, mode, c.psd, c.stream);
    else launch_mode<2, FAM_LIGHT>(a, np, nvp, nb, mode, c.psd, c.stream);
  }
  if (!fast) timing_end(p, c.stream);
  if (mode == MODE_HVP) return 0;
  return np > n_fast ? np : n_fast;
}

}  // namespace mg
