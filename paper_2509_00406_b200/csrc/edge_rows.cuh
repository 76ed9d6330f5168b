// Edge row kernel body, shared by the library's builtin radial terms
// (edge_kernels.cu) and traced callbacks whose edge terms the tracer proved
// radial (jit_rows.cuh, compiled at runtime with the generated functors).
// See edge_kernels.cu for the algorithm. A policy type supplies the terms:
//
//   static constexpr bool kXFreeHvp;   // EV Hessian independent of x (the
//                                      // unclamped HVP reads directions only)
//   static constexpr bool kVertexOnly; // no per-edge attribute: the gradient /
//                                      // HVP kernels may read 32-bit records
//   template <int N, int MODE> static auto vload(const EvArgs&, int g);
//       V-term attribute loads, issued before the incidence gathers
//   template <int N, int MODE, bool PSD> static void vterms(a, g, fr, pre, xs, us, eacc, vec, dg, finite);
//       the row's V terms: energy, gradient / H u into vec, Hessian into dg
//       (closed forms that can miss the reference's NaN placement clear finite)
//   template <int MODE> static auto eload(const EvArgs&, uint32_t e);
//       per-edge attribute loads of one incidence (issued with the gathers)
//   template <int MODE, bool NEEDV, class EP, class F> static void eterms(a, ep, rr, e, one);
//       phi, phi', phi'' of every radial EV term at r = |d|^2, handed to
//       one(ok, phi, phi', phi'')
//   using Store = double | float;      // storage of x, w, outputs, attributes
#pragma once
#include "mg_internal.cuh"
#include "stage.cuh"

namespace mg {
namespace rows {

constexpr int PT = EV_ROW_BLOCK;  // rows (threads) per CTA
constexpr int MAXT = 8;
constexpr int MAX_JS = 24;        // traced attribute streams of a row module (all terms)

struct EvArgs {
  int nterms;
  int64_t V;  // owned rows (patch order)
  const int32_t* order;      // (V) vertex of each row
  const uint8_t* pfix;       // (V) pinned flag of each row
  const uint32_t* rmeta;     // (V) incidence count (sat. 255) | pinned << 8 | diagonal position << 16
  const uint64_t* ell;       // (EV_ELL_K, V) first incidences, slot-major
  int64_t es;                // slot stride of ell / ell32 (V padded to whole row blocks; rmeta / order padded too)
  const uint32_t* ell32;     // (EV_ELL_K, V) vertex-only 32-bit records for the gradient / HVP kernels
                             // when no EV term reads a per-edge attribute (patch_setup.cu k_ell32), or null
  const int32_t* rinc_off;   // (V+1)
  const uint64_t* rrec;      // lo: edge | slot << 31, hi: other | pinned(other) << 31
  const int64_t* prow_ro;
  const int32_t* prow_len;
  const uint8_t* prow_dp;
  const int32_t* hoff;
  const double* x;
  const double* w;
  double* grad;
  double* hess;
  double* y;
  double* partials;
  int* redo;  // raised by the radial kernel on a non-finite lane
  int* exact_runs;
  int nev, nvt;                 // compacted term lists (indices into terms)
  int ev_idx[MAXT], vt_idx[MAXT];
  const double* ev_a0;          // per-edge attribute of ev_idx[0] (prefetched), or null
  // staged tiles (k_tile_ev): see Problem::tiles_ready
  const int2* tcnt;
  const uint32_t* tv;
  const uint64_t* te;
  const uint16_t* islot;
  const uint16_t* islot8;  // (V, 8): a row's first 8 slots, one 16-byte load
  int max_v, max_e;
  int64_t np_total;  // energy partials the reduction reads (the exact re-run zero-fills past its own)
  double floor;
  TermDev terms[MAXT];
  const double* js[MAX_JS];  // traced terms: attribute streams of the row module, terms in order
};

MG_DI void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// dst[0..n) = src[0..n) (doubles), src in shared memory with the same 16-byte
// phase as dst: 8-byte head / tail stores plus one bulk (TMA) copy of the
// aligned middle. The caller waits for the bulk group before leaving.
MG_DI void row_store_bulk(double* dst, const double* src, int n) {
  int k0 = 0;
  if (reinterpret_cast<uintptr_t>(dst) & 15) {
    if (n > 0) dst[0] = src[0];
    k0 = 1;
  }
  int m = n - k0;
  if (m <= 0) return;
  if (m & 1) {
    dst[n - 1] = src[n - 1];
    --m;
  }
  if (m > 0) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(src + k0);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst + k0), "r"(sa), "r"((uint32_t)m * 8u) : "memory");
  }
}

// the same for floats (fp32 storage): 4-byte head until dst is 16-byte
// aligned, one bulk copy of the aligned middle, 4-byte tail
MG_DI void row_store_bulk_f(float* dst, const float* src, int n) {
  int k0 = 0;
  while (k0 < n && (reinterpret_cast<uintptr_t>(dst + k0) & 15)) {
    dst[k0] = src[k0];
    ++k0;
  }
  int m = (n - k0) & ~3;
  for (int k = k0 + m; k < n; ++k) dst[k] = src[k];
  if (m > 0) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(src + k0);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst + k0), "r"(sa), "r"((uint32_t)m * 4u) : "memory");
  }
}

// 1/x to full fp64 precision without the IEEE division sequence: hardware
// reciprocal estimate + two Newton steps (non-finite / zero inputs give
// non-finite results, which send the call to the exact kernel)
MG_DI double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Storage of the per-vertex / per-element streams: fp64 (the reference's), or
// fp32 (Problem(dtype=float32): half the bytes; arithmetic stays fp64). The
// EvArgs pointers are typed double and reinterpreted by the storage type.
template <class T> MG_DI double ldv(const double* p, int64_t i) { return (double)reinterpret_cast<const T*>(p)[i]; }
template <class T> MG_DI void stv(double* p, int64_t i, double v) { reinterpret_cast<T*>(p)[i] = (T)v; }

// Closed-form clamp of a radial block c_i I + c_d d d^T (r = |d|^2): the
// transverse eigenvalue is c_i, the axial one c_i + c_d r. Already above the
// floor -> unchanged (the reference's eigh recomposition equals the input to
// rounding); otherwise Q max(L, f) Q^T = m_t I + (m_d - m_t) d d^T / r.
MG_DI void radial_clamp_fast(double& ci, double& cd, double r, double f) {
  const double lt = ci, ld = ci + cd * r;
  if (lt > f && ld > f) return;
  const double mt = lt > f ? lt : f, md = ld > f ? ld : f;
  ci = mt;
  cd = r > 0.0 ? (md - mt) * rcp_fast(r) : 0.0;
}

// incidences per row held in registers (the rest are streamed) and the
// occupancy target: the Hessian kernel is bounded by its shared-memory row
// buffers anyway; the smem-free HVP / gradient kernels trade prefetch depth
// for more resident warps
#ifndef EV_HESS_MINB
#define EV_HESS_MINB 1
#endif
#ifndef EV_FLAT_BLOCK
#define EV_FLAT_BLOCK 64
#endif
// 1: gradient / HVP kernels walk row blocks grid-stride too, with the next
// row's level-1 streams in flight (A/B knob)
#ifndef EV_FLAT_PERSIST
#define EV_FLAT_PERSIST 0
#endif
// gradient / HVP kernels: persistent CTAs whose row blocks' level-1 streams
// (ELL records, meta words, row order) arrive by bulk (TMA) copies EV_STAGES
// blocks ahead into a shared-memory ring (0: per-thread loads)
#ifndef EV_STAGED
#define EV_STAGED 1
#endif
#ifndef EV_STAGED_HESS
#define EV_STAGED_HESS 1  // headline 0.617 -> 0.543 ms (cloth 2048^2 grad+H(psd)), plain 0.553 -> 0.485
#endif
#ifndef EV_STAGES_HESS
// one stage: the next block's streams are issued as soon as this block's are
// read, a whole block's compute ahead, and the 4.3 KB saved lets 6 instead of
// 5 CTAs (32 KB row buffers) share an SM: headline 0.542 -> 0.485 ms
#define EV_STAGES_HESS 1
#endif
#ifndef EV_STAGES
#define EV_STAGES 1  // cloth HVP 0.190 -> 0.173 ms staged (2240^2); smoothing HVP 0.271 at 1 or 2, 0.295 at 3 (1: 1% faster)
#endif
// MAXI: incidences in flight; BLOCK: threads per CTA (the Hessian kernel's CTA
// is its row-buffer group, EV_ROW_BLOCK); MINB: CTAs per SM to fit
template <int MODE, bool PSD> struct FastCfg {
  static constexpr int MAXI = EV_ELL_K, BLOCK = EV_ROW_BLOCK, MINB = EV_HESS_MINB;
};
#ifndef EV_HVP_MAXI
#define EV_HVP_MAXI 4  // 5 / 6: config-5 HVP 1.726 / 1.868 vs 1.676 ms (6 at 640 threads: 2.83)
#endif
#ifndef EV_XFREE_MAXI
#define EV_XFREE_MAXI 6  // incidences in flight of the x-free HVP (directions only): 0.313 -> 0.278 ms at 4 -> 6 (smoothing, icosphere(10))
#endif
#ifndef EV_HVP_THREADS
#define EV_HVP_THREADS 512  // measured: 0.269 ms vs 0.288 at 640 (row-kernel spring HVP, 2048^2)
#endif
template <> struct FastCfg<MODE_HVP, false> {
  static constexpr int MAXI = EV_HVP_MAXI, BLOCK = EV_FLAT_BLOCK, MINB = EV_HVP_THREADS / EV_FLAT_BLOCK;
};
#ifndef EV_HVP_PSD_THREADS
#define EV_HVP_PSD_THREADS 512  // 640: 0.275 vs 0.234 ms (clamped HVP, 2240^2)
#endif
#ifndef EV_GRAD_THREADS
#define EV_GRAD_THREADS 640  // with 6 incidences in flight; 768 with 4: config-5 gradient 1.453 vs 1.483 ms, smoothing gradient 0.280 vs 0.301 (6 at 512: 1.565; 5 at 640 / 768: 1.463 / 1.660)
#endif
#ifndef EV_HVP_PSD_MAXI
#define EV_HVP_PSD_MAXI 4  // 6: clamped cloth HVP 0.241 vs 0.234 ms (2240^2), 0.274 at 384 threads
#endif
#ifndef EV_GRAD_MAXI
#define EV_GRAD_MAXI 6  // the gradient rows' incidences in flight (EV_GRAD_THREADS)
#endif
template <> struct FastCfg<MODE_HVP, true> {
  static constexpr int MAXI = EV_HVP_PSD_MAXI, BLOCK = EV_FLAT_BLOCK, MINB = EV_HVP_PSD_THREADS / EV_FLAT_BLOCK;
};
template <> struct FastCfg<MODE_GRAD, false> {
  static constexpr int MAXI = EV_GRAD_MAXI, BLOCK = EV_FLAT_BLOCK, MINB = EV_GRAD_THREADS / EV_FLAT_BLOCK;
};
#ifndef EV_ENERGY_THREADS
#define EV_ENERGY_THREADS 768  // 512 / 640 / 1024: 0.146 / 0.128 / 0.160 vs 0.129 ms (cloth 2048^2 energy probe)
#endif
template <> struct FastCfg<MODE_ENERGY, false> {  // the energy probe: first-vertex edges only
  static constexpr int MAXI = 6, BLOCK = EV_FLAT_BLOCK, MINB = EV_ENERGY_THREADS / EV_FLAT_BLOCK;
};
// the x-free HVP holds only directions: full occupancy (64 registers; 1280 /
// 1536 threads per SM measured 0.510 / 0.639 ms vs 0.274, smoothing HVP)
template <int MODE, bool PSD, bool XFREE_HVP> struct FastMinb {
  static constexpr int v = (MODE == MODE_HVP && !PSD && XFREE_HVP) ? 1024 / EV_FLAT_BLOCK : FastCfg<MODE, PSD>::MINB;
};

// Radial row kernel body: one thread per owned row, d = x_row - x_other
// (radial terms are even in d, so no orientation bookkeeping). A row's first
// MAXI incidences are fetched in two batched levels (records, then neighbour
// x and edge attributes) so their latencies overlap.
template <int N, int MODE, bool PSD, class Pol>
MG_DI void rows_fast_body(const EvArgs& a) {
  constexpr int T = TriN<N>::value, NN = N * N;
  using ST = typename Pol::Store;
  constexpr bool F32 = sizeof(ST) == 4;  // fp32 storage
  constexpr int PTB = FastCfg<MODE, PSD>::BLOCK;
  // e.g. the edge length's Hessian 2 [[I,-I],[-I,I]] does not depend on x
  // (apps/smooth.py:27-28): its unclamped HVP reads only the direction
  constexpr bool XFREE = MODE == MODE_HVP && !PSD && Pol::kXFreeHvp;
  constexpr int MAXI = XFREE ? EV_XFREE_MAXI : FastCfg<MODE, PSD>::MAXI;
  extern __shared__ __align__(16) double hbuf[];
  // Row blocks are walked grid-stride (a persistent grid for the Hessian, one
  // block per CTA otherwise); the level-1 streams of the thread's next row are
  // loaded while it works on the current one.
  struct L1 {
    int g = 0;
    uint32_t meta = 0;
    int64_t ro = 0;
    int ho = 0;
    uint64_t rc[EV_ELL_K];
  };
  // level 1: static per-row streams, all indexed by the row alone
  // (coalesced): vertex, meta word, row start / buffer offset, ELL records.
  // The gradient / HVP kernels read 32-bit vertex-only records when no term
  // needs the edge id (half the bytes) and expand them to the 64-bit form here.
  auto load_l1 = [&](int64_t r, L1& l) {
    if (r >= a.V) return;
    l.g = a.order ? a.order[r] : (int)r;  // null: identity row order
    l.meta = a.rmeta[r];
    if constexpr (MODE == MODE_HESS) {
      l.ro = a.prow_ro[r];
      l.ho = a.hoff[r];
#pragma unroll
      for (int j = 0; j < EV_ELL_K; ++j) l.rc[j] = a.ell[(int64_t)j * a.es + r];
    } else if (Pol::kVertexOnly) {  // vertex-only records (no per-edge attribute is read)
#pragma unroll
      for (int j = 0; j < EV_ELL_K; ++j) {
        const uint32_t q = a.ell32[(int64_t)j * a.es + r];
        const uint32_t o = q & 0x7fffffffu;
        const uint32_t lo = (uint32_t)(o < (uint32_t)l.g) << 31;  // edge id unused; first vertex: o > g
        l.rc[j] = (uint64_t)lo | ((uint64_t)q << 32);
      }
    } else {
#pragma unroll
      for (int j = 0; j < EV_ELL_K; ++j) l.rc[j] = a.ell[(int64_t)j * a.es + r];
    }
  };
  const int64_t nblk = (a.V + PTB - 1) / PTB;
  bool finite = true;
  L1 cur, nxt;
  constexpr bool STAGED = MODE != MODE_HESS ? EV_STAGED : EV_STAGED_HESS;
  constexpr bool PERSIST = !STAGED && (MODE == MODE_HESS || EV_FLAT_PERSIST);
  constexpr bool HS = MODE == MODE_HESS;  // the Hessian's stages also carry row starts and row-buffer offsets
  if constexpr (PERSIST) load_l1((int64_t)blockIdx.x * PTB + threadIdx.x, cur);
  // staged level 1 (see EV_STAGED): ring of EV_STAGES stages, each one row
  // block's slot-major ELL slices, meta words and row order
  // (vertex-only problems always carry the 32-bit records: patch_setup.cu)
  constexpr bool vo = Pol::kVertexOnly;
  constexpr int ST_ELL = EV_ELL_K * PTB * ((vo && !HS) ? 4 : 8);
  constexpr int ST_RO = ST_ELL + 2 * PTB * 4, ST_HO = ST_RO + PTB * 8;
  constexpr int ST_BYTES = HS ? ST_HO + PTB * 4 : ST_RO;
  constexpr int NST = HS ? EV_STAGES_HESS : EV_STAGES;
  __shared__ __align__(128) unsigned char stg[STAGED ? NST : 1][STAGED ? ST_BYTES : 16];
  __shared__ __align__(8) uint64_t sbar[NST];
  auto stage_issue = [&](int st, int64_t b) {  // one thread
    constexpr bool v32 = vo && !HS;
    constexpr uint32_t esz = v32 ? 4u : 8u;
    mbar_expect_tx(&sbar[st], EV_ELL_K * PTB * esz + PTB * 4 + (a.order ? PTB * 4 : 0) + (HS ? PTB * 12 : 0));
#pragma unroll
    for (int j = 0; j < EV_ELL_K; ++j) {
      const void* src = v32 ? (const void*)(a.ell32 + (int64_t)j * a.es + b * PTB)
                            : (const void*)(a.ell + (int64_t)j * a.es + b * PTB);
      bulk_g2s(stg[st] + j * PTB * esz, src, PTB * esz, &sbar[st]);
    }
    bulk_g2s(stg[st] + ST_ELL, a.rmeta + b * PTB, PTB * 4, &sbar[st]);
    if (a.order) bulk_g2s(stg[st] + ST_ELL + PTB * 4, a.order + b * PTB, PTB * 4, &sbar[st]);
    if constexpr (HS) {
      bulk_g2s(stg[st] + ST_RO, a.prow_ro + b * PTB, PTB * 8, &sbar[st]);
      bulk_g2s(stg[st] + ST_HO, a.hoff + b * PTB, PTB * 4, &sbar[st]);
    }
  };
  if constexpr (STAGED) {
    if (threadIdx.x == 0) {
      for (int st = 0; st < NST; ++st) mbar_init(&sbar[st], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int st = 0; st < NST; ++st) {
        const int64_t b = blockIdx.x + (int64_t)st * gridDim.x;
        if (b < nblk) stage_issue(st, b);
      }
  }
  int it = 0;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
  const int64_t row = blk * PTB + threadIdx.x;
  if constexpr (STAGED) {
    const int st = it % NST;
    mbar_wait(&sbar[st], (uint32_t)(it / NST) & 1u);
    const unsigned char* sp = stg[st];
    cur.g = a.order ? reinterpret_cast<const int32_t*>(sp + ST_ELL + PTB * 4)[threadIdx.x] : (int)row;
    cur.meta = reinterpret_cast<const uint32_t*>(sp + ST_ELL)[threadIdx.x];
    if constexpr (HS) {
      cur.ro = reinterpret_cast<const int64_t*>(sp + ST_RO)[threadIdx.x];
      cur.ho = reinterpret_cast<const int32_t*>(sp + ST_HO)[threadIdx.x];
    }
#pragma unroll
    for (int j = 0; j < EV_ELL_K; ++j) {
      if (vo && !HS) {
        const uint32_t q = reinterpret_cast<const uint32_t*>(sp)[j * PTB + threadIdx.x];
        const uint32_t lo = (uint32_t)((q & 0x7fffffffu) < (uint32_t)cur.g) << 31;
        cur.rc[j] = (uint64_t)lo | ((uint64_t)q << 32);
      } else {
        cur.rc[j] = reinterpret_cast<const uint64_t*>(sp)[j * PTB + threadIdx.x];
      }
    }
    __syncthreads();  // every thread has read the stage: refill it
    if (threadIdx.x == 0 && blk + (int64_t)NST * gridDim.x < nblk) {
      // the threads' generic-proxy reads of the stage before the bulk copy's
      // async-proxy writes into it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      stage_issue(st, blk + (int64_t)NST * gridDim.x);
    }
  } else if constexpr (PERSIST) {
    if (blk + gridDim.x < nblk) load_l1(row + (int64_t)gridDim.x * PTB, nxt);
  } else {
    load_l1(row, cur);
  }
  double eacc = 0.0;
  if (row < a.V) {
    const int g = cur.g;
    const uint32_t meta = cur.meta;
    const int64_t ro = cur.ro;
    const int ho = cur.ho;
    uint64_t rc[EV_ELL_K];
#pragma unroll
    for (int j = 0; j < EV_ELL_K; ++j) rc[j] = cur.rc[j];
    (void)ro;
    // the previous row's bulk copy must have read this thread's row buffer
    if constexpr (MODE == MODE_HESS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    // level 2: own x / w, issued before anything waits on the meta word (with
    // the identity row order g is the row itself, so these do not wait on
    // level 1 at all); the pinned mask is applied after the load
    double xs[N], us[N];
#pragma unroll
    for (int c = 0; c < N; ++c) {
      xs[c] = ldv<ST>(a.x, (int64_t)g * N + c);
      if constexpr (MODE == MODE_HVP) us[c] = ldv<ST>(a.w, (int64_t)g * N + c);
      else us[c] = 0.0;
    }
    const auto vpre = Pol::template vload<N, MODE>(a, g);
    // level 3: neighbour x (w) and the edge attributes, kept MAXI incidences
    // ahead of the compute (a rolling window over the ELL slots). Unused ELL
    // slots hold record 0 (edge 0, vertex 0), so the loads are unconditional
    // (no wait on the incidence count) and their values are never used.
    using EP = decltype(Pol::template eload<MODE>(a, 0u));
    double xo[EV_ELL_K][N], uo[EV_ELL_K][N];
    EP ep[EV_ELL_K];
    auto issue = [&](int j) {
      const uint32_t hi = (uint32_t)(rc[j] >> 32);
      const int64_t o = hi & 0x7fffffffu;
      const bool fo = !(hi >> 31);
      // the energy probe evaluates an edge at its first vertex only
      const bool need = MODE != MODE_ENERGY || !((uint32_t)rc[j] >> 31);
#pragma unroll
      for (int c = 0; c < N; ++c) {
        xo[j][c] = (!XFREE && need) ? ldv<ST>(a.x, o * N + c) : 0.0;
        if constexpr (MODE == MODE_HVP) {
          const double wv = ldv<ST>(a.w, o * N + c);
          uo[j][c] = fo ? wv : 0.0;
        } else {
          uo[j][c] = 0.0;
        }
      }
      if (need) ep[j] = Pol::template eload<MODE>(a, (uint32_t)rc[j] & 0x7fffffffu);
    };
#pragma unroll
    for (int j = 0; j < MAXI; ++j) issue(j);
    const bool fr = !((meta >> 8) & 1);
    const int dp = (int)(meta >> 16) & 0xff;
    const int cnt = (meta & 0xff) < 255 ? (int)(meta & 0xff) : a.rinc_off[row + 1] - a.rinc_off[row];
    if constexpr (MODE == MODE_HVP) {
#pragma unroll
      for (int c = 0; c < N; ++c) us[c] = fr ? us[c] : 0.0;
    }
    double vec[N], dg[T];
#pragma unroll
    for (int i = 0; i < N; ++i) vec[i] = 0.0;
#pragma unroll
    for (int i = 0; i < T; ++i) dg[i] = 0.0;
    // V terms (their attribute loads overlapped the level-3 loads)
    if constexpr (MODE == MODE_ENERGY) eacc += Pol::template venergy<N>(a, g, vpre, xs);
    else Pol::template vterms<N, MODE, PSD>(a, g, fr, vpre, xs, us, eacc, vec, dg, finite);
    double* hrow = hbuf + ho;
    // fp32 storage: the row built as floats in the row's (double-sized) slot of
    // the buffer, shifted so its 16-byte phase matches the destination's
    ST* grow = reinterpret_cast<ST*>(hbuf) + 2 * ho + (int)(((uint64_t)ro * NN - 2 * (uint64_t)ho) & 3u);
    (void)grow;
    int pos = 0;
    // one incidence: contributions to this row
    auto incidence = [&](uint64_t r64, const double* xo_, const double* uo_, const EP& av) {
      const uint32_t lo = (uint32_t)r64, hi = (uint32_t)(r64 >> 32);
      const uint32_t e = lo & 0x7fffffffu;
      const bool first = (lo >> 31) == 0;  // the row is the edge's first vertex
      const bool fo = !(hi >> 31);
      if constexpr (MODE == MODE_ENERGY) {
        if (first) {
          double d[N];
#pragma unroll
          for (int c = 0; c < N; ++c) d[c] = __dsub_rn(xs[c], xo_[c]);
          eacc += Pol::template evalue<N>(a, av, d, e);
        }
        return;
      }
      double d[N], rr = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        d[c] = XFREE ? 0.0 : xs[c] - xo_[c];
        rr = d[c] * d[c] + rr;
      }
      double gam = 0.0, ci_s = 0.0, cd_s = 0.0, dl = 0.0, val = 0.0;
      auto one_term = [&](bool ok, double pv, double p1, double p2) {
        finite &= ok;
        val += pv;
        gam += 2.0 * p1;
        if constexpr (MODE != MODE_GRAD) {
          double ci = 2.0 * p1, cd = 4.0 * p2, sh = 0.0;
          if constexpr (PSD) {
            if (fr && fo) {  // [[A,-A],[-A,A]]: clamp 2A, halve, shift floor/2
              ci *= 2.0; cd *= 2.0;
              radial_clamp_fast(ci, cd, rr, a.floor);
              ci *= 0.5; cd *= 0.5;
              sh = 0.5 * a.floor;
            } else if (fr || fo) {
              radial_clamp_fast(ci, cd, rr, a.floor);
            }
          }
          ci_s += ci;
          cd_s += cd;
          dl += sh;
        }
      };
      Pol::template eterms<MODE, MODE != MODE_HVP>(a, av, rr, e, one_term);
      if constexpr (MODE != MODE_HVP) {
        if (first) eacc += val;  // an edge's energy counts at its first vertex
      }
      if constexpr (MODE == MODE_GRAD || MODE == MODE_HESS) {
#pragma unroll
        for (int i = 0; i < N; ++i) vec[i] += gam * d[i];
      }
      if constexpr (MODE == MODE_HVP) {  // y_row = M (u_row - u_other) + dl (u_row + u_other)
        if constexpr (XFREE) {  // M = ci I (the axial coefficient is exactly zero)
#pragma unroll
          for (int i = 0; i < N; ++i) vec[i] += ci_s * (us[i] - uo_[i]);
        } else {
          double dw = 0.0;
#pragma unroll
          for (int c = 0; c < N; ++c) dw += d[c] * (us[c] - uo_[c]);
#pragma unroll
          for (int i = 0; i < N; ++i) {
            if constexpr (PSD) vec[i] += ci_s * (us[i] - uo_[i]) + cd_s * d[i] * dw + dl * (us[i] + uo_[i]);
            else vec[i] += ci_s * (us[i] - uo_[i]) + cd_s * d[i] * dw;  // dl is zero without a clamp
          }
        }
      }
      if constexpr (MODE == MODE_HESS) {
        // t = cd d d^T (6 unique products) feeds both the diagonal sum and the
        // edge's off-diagonal block -t + (dl - ci) I
        double cdd[N], t[T];
#pragma unroll
        for (int i = 0; i < N; ++i) cdd[i] = cd_s * d[i];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int c = 0; c <= i; ++c) t[tri(i, c)] = cdd[i] * d[c];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int c = 0; c <= i; ++c) dg[tri(i, c)] += t[tri(i, c)] + (i == c ? ci_s + dl : 0.0);
        if (fr && fo) {
          if (dp != 255 && pos == dp) ++pos;  // leave the diagonal's slot
          double blk[NN];
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int c = 0; c < N; ++c) blk[i * N + c] = -t[tri(i, c)] + (i == c ? dl - ci_s : 0.0);
          if constexpr (F32) {
            ST* dst = grow + pos * NN;
#pragma unroll
            for (int k = 0; k < NN; ++k) dst[k] = (ST)blk[k];
          } else {
            double* dst = hrow + pos * NN;
#pragma unroll
            for (int k = 0; k < NN; ++k) dst[k] = blk[k];
          }
          ++pos;
        }
      }
    };
#pragma unroll
    for (int j = 0; j < EV_ELL_K; ++j) {
      if (j + MAXI < EV_ELL_K) issue(j + MAXI);
      if (j < cnt) incidence(rc[j], xo[j], uo[j], ep[j]);
    }
    for (int k = EV_ELL_K; k < cnt; ++k) {  // high-valence rows: the CSR tail
      const uint64_t r64 = a.rrec[a.rinc_off[row] + k];
      const int64_t o = (uint32_t)(r64 >> 32) & 0x7fffffffu;
      const bool fo = !(r64 >> 63);
      double x1[N], u1[N];
#pragma unroll
      for (int c = 0; c < N; ++c) {
        x1[c] = ldv<ST>(a.x, o * N + c);
        if constexpr (MODE == MODE_HVP) u1[c] = fo ? ldv<ST>(a.w, o * N + c) : 0.0;
        else u1[c] = 0.0;
      }
      const EP av = Pol::template eload<MODE>(a, (uint32_t)r64 & 0x7fffffffu);
      incidence(r64, x1, u1, av);
    }
    double* vout = MODE == MODE_HVP ? a.y : a.grad;
    if constexpr (MODE != MODE_ENERGY) {
#pragma unroll
      for (int i = 0; i < N; ++i) stv<ST>(vout, (int64_t)g * N + i, fr ? vec[i] : 0.0);
    }
    if constexpr (MODE == MODE_HESS) {
      if (fr && dp != 255) {
        if constexpr (F32) {
          ST* dst = grow + dp * NN;
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int c = 0; c < N; ++c) dst[i * N + c] = (ST)dg[tri(i, c)];
        } else {
          double* dst = hrow + dp * NN;
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int c = 0; c < N; ++c) dst[i * N + c] = dg[tri(i, c)];
        }
      }
      // blocks written: off-diagonals, plus the diagonal if the walk never passed it
      const int len = (fr && dp != 255) ? (pos > dp + 1 ? pos : dp + 1) : pos;
      if (len > 0) {
        fence_proxy_async_smem();
        if constexpr (F32)
          row_store_bulk_f(reinterpret_cast<float*>(a.hess) + ro * NN, reinterpret_cast<const float*>(grow), len * NN);
        else
          row_store_bulk(a.hess + ro * NN, hrow, len * NN);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if constexpr (MODE != MODE_HVP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(0xffffffffu, eacc, o);
    if ((threadIdx.x & 31) == 0) a.partials[row >> 5] = eacc;
  }
  if constexpr (PERSIST) cur = nxt;
  else if constexpr (!STAGED) break;  // one row block per CTA (unstaged gradient / HVP)
  }
  if (!finite) *a.redo = 1;
  if constexpr (MODE == MODE_HESS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

}  // namespace rows
}  // namespace mg
