// Edge row kernel: the patch-owner assembly specialised to problems whose
// terms are V terms and radial EV terms E = phi(|x_i - x_j|^2) (cloth
// springs, smoothing).
//
// One thread per owned row; rows in patch (Morton) order, EV_ROW_BLOCK rows
// per CTA, so a CTA's rows and their neighbours are spatially compact and the
// neighbours' x hit L1/L2. A thread
//   * evaluates its V terms,
//   * walks its incident edges in column order (records built at setup) and
//     evaluates each from a one-variable dual on r = |d|^2 (Radial in
//     terms.cuh) with the closed-form PSD clamp; non-finite lanes take the
//     exact K = n dual so NaN / Inf land where the reference puts them,
//   * accumulates gradient / HVP row and diagonal block in registers in that
//     fixed order (bitwise reproducible), writes each off-diagonal block of its
//     row into a shared-memory row buffer in output layout as it goes,
//   * and streams the finished row to HBM with one bulk (TMA) copy.
// No barriers, no atomics, no memset: every output byte is written once; an
// edge is evaluated by each of its two owner rows (recompute instead of
// communicate). The energy counts every element once (edges at their first
// vertex) through fixed-order per-warp partials.
#include <cstring>

#include "edge_rows.cuh"
#include "elem_eval.cuh"
#include "mg_internal.cuh"
#include "psd.cuh"

namespace mg {

namespace {

using namespace rows;

// per-edge record (doubles) and per-row V-term accumulator widths
template <int N, int MODE, bool PSD>
struct EvRec {
  static constexpr int T = TriN<N>::value;
  // HESS: [g (N), A + dl I (T)];  GRAD: [g];  HVP: [y_a] or, with PSD, [y_a, y_b]
  static constexpr int SW = MODE == MODE_HESS ? N + T : (MODE == MODE_HVP && PSD) ? 2 * N : N;
  static constexpr int VW = MODE == MODE_HESS ? N + T : N;
};


template <class Q>
MG_DI double hess00(const Q& q) {
  if constexpr (Q::kZero) return 0.0;
  else return q.h[0];
}

// Closed-form clamp of a radial block c_i I + c_d d d^T (r = |d|^2): the
// transverse eigenvalue is c_i, the axial one c_i + c_d r. Already above the
// floor -> unchanged (the reference's eigh recomposition equals the input to
// rounding); otherwise Q max(L, f) Q^T = m_t I + (m_d - m_t) d d^T / r.
MG_DI void radial_clamp(double& ci, double& cd, double r, double f) {
  const double lt = ci, ld = ci + cd * r;
  if (lt > f && ld > f) return;
  const double mt = lt > f ? lt : f, md = ld > f ? ld : f;
  ci = mt;
  cd = r > 0.0 ? (md - mt) / r : 0.0;
}

// Radial evaluation of one patch edge (sum over the EV terms). Returns false
// when any intermediate is non-finite (the caller then takes edge_dual).
//   val: energy;  rec: record (EvRec);  dl: floor shift of the off-diagonal
//   blocks (HESS): block(a,b) = -(A) + dl I = -rec_A + 2 dl I.
template <int N, int MODE, bool PSD>
MG_DI bool edge_radial(const EvArgs& a, int64_t e, const double* xa, const double* xb, const double* wa,
                       const double* wb, bool fa, bool fb, double& val, double* rec, double& dl) {
  using L = EvRec<N, MODE, PSD>;
  double d[N];
  double rr = 0.0;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    d[c] = xa[c] - xb[c];
    rr = d[c] * d[c] + rr;
  }
  double gam = 0.0;  // sum of 2 phi'
  double ci_s = 0.0, cd_s = 0.0;
  double yacc[2 * N];
#pragma unroll
  for (int i = 0; i < 2 * N; ++i) yacc[i] = 0.0;
  bool ok = true;
  val = 0.0;
  dl = 0.0;
  for (int ti = 0; ti < a.nterms; ++ti) {
    const TermDev& t = a.terms[ti];
    if (t.op != MG_OP_EV) continue;
    if constexpr (MODE == MODE_GRAD) {
      Dg<1> r;
      r.v = rr;
      r.g[0] = 1.0;
      auto q = t.type == MG_TERM_SPRING ? term_eval_radial<MG_TERM_SPRING>(t, e, r)
                                        : term_eval_radial<MG_TERM_EDGE_LENGTH>(t, e, r);
      ok &= isfinite(q.v) && isfinite(q.g[0]);
      val += q.v;
      gam += 2.0 * q.g[0];
    } else {
      Dh<1, true> r;
      r.v = rr;
      r.g[0] = 1.0;
      double pv, p1, p2;
      if (t.type == MG_TERM_SPRING) {
        auto q = term_eval_radial<MG_TERM_SPRING>(t, e, r);
        pv = q.v; p1 = q.g[0]; p2 = hess00(q);
      } else {
        auto q = term_eval_radial<MG_TERM_EDGE_LENGTH>(t, e, r);
        pv = q.v; p1 = q.g[0]; p2 = hess00(q);
      }
      ok &= isfinite(pv) && isfinite(p1) && isfinite(p2);
      val += pv;
      gam += 2.0 * p1;
      double ci = 2.0 * p1, cd = 4.0 * p2, sh = 0.0;
      if constexpr (PSD) {
        if (fa && fb) {  // spectrum of [[A,-A],[-A,A]] = 2 eig(A) U {0}: clamp 2A, halve, shift floor/2
          ci *= 2.0; cd *= 2.0;
          radial_clamp(ci, cd, rr, a.floor);
          ci *= 0.5; cd *= 0.5;
          sh = 0.5 * a.floor;
        } else if (fa || fb) {
          radial_clamp(ci, cd, rr, a.floor);
        }
      }
      if constexpr (MODE == MODE_HESS) {
        ci_s += ci;
        cd_s += cd;
        dl += sh;
      } else {  // HVP: y_a = M (wa - wb) + sh (wa + wb), y_b = -M (wa - wb) + sh (wa + wb)
        double wd[N], ws[N], dw = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) {
          const double ua = fa ? wa[c] : 0.0, ub = fb ? wb[c] : 0.0;
          wd[c] = ua - ub;
          ws[c] = ua + ub;
          dw += d[c] * wd[c];
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double m = ci * wd[i] + cd * d[i] * dw;
          yacc[i] += m + sh * ws[i];
          yacc[N + i] += -m + sh * ws[i];
        }
      }
    }
  }
  if (!ok) return false;
  if constexpr (MODE == MODE_GRAD || MODE == MODE_HESS) {
#pragma unroll
    for (int i = 0; i < N; ++i) rec[i] = gam * d[i];
  }
  if constexpr (MODE == MODE_HESS) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) rec[N + tri(i, j)] = cd_s * d[i] * d[j] + (i == j ? ci_s + dl : 0.0);
  }
  if constexpr (MODE == MODE_HVP) {
#pragma unroll
    for (int i = 0; i < L::SW; ++i) rec[i] = yacc[i];
  }
  return true;
}

// Exact path: K = n dual on d = x_a - x_b (bitwise equal to the reference's
// K = 2n dual, TwoPoint in terms.cuh), packed n x n blocks, generic clamp.

template <int N, int MODE, bool PSD>
MG_DI void edge_dual(const EvArgs& a, int64_t e, const double* xa, const double* xb, const double* wa,
                     const double* wb, bool fa, bool fb, double& val, double* rec, double& dl) {
  constexpr int T = TriN<N>::value;
  using L = EvRec<N, MODE, PSD>;
  double acc[L::SW];
#pragma unroll
  for (int i = 0; i < L::SW; ++i) acc[i] = 0.0;
  val = 0.0;
  dl = 0.0;
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
      auto r = tt == MG_TERM_SPRING ? term_eval_diff<MG_TERM_SPRING, N>(t, e, d)
                                    : term_eval_diff<MG_TERM_EDGE_LENGTH, N>(t, e, d);
      val += r.v;
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] += r.g[i];
    } else {
      Vec<Dh<N, true>, N> d;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        d[c].v = xa[c] - xb[c];
#pragma unroll
        for (int i = 0; i < N; ++i) d[c].g[i] = (i == c) ? 1.0 : 0.0;
      }
      auto r = tt == MG_TERM_SPRING ? term_eval_diff<MG_TERM_SPRING, N>(t, e, d)
                                    : term_eval_diff<MG_TERM_EDGE_LENGTH, N>(t, e, d);
      double h[T];
#pragma unroll
      for (int i = 0; i < T; ++i) h[i] = 0.5 * (r.h[i] + r.h[i]);
      double sh = 0.0;
      if constexpr (PSD) {
        if (all_finite<N>(h)) {
          if (fa && fb) {
#pragma unroll
            for (int i = 0; i < T; ++i) h[i] = 2.0 * h[i];
            project_if_needed<N>(h, a.floor);
#pragma unroll
            for (int i = 0; i < T; ++i) h[i] = 0.5 * h[i];
            sh = 0.5 * a.floor;
          } else if (fa || fb) {
            project_if_needed<N>(h, a.floor);
          }
        }
      }
      val += r.v;
      if constexpr (MODE == MODE_HESS) {
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] += r.g[i];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) acc[N + tri(i, j)] += h[tri(i, j)] + (i == j ? sh : 0.0);
        dl += sh;
      } else {
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
          acc[i] += m + sh * ws[i];
          if constexpr (L::SW == 2 * N) acc[N + i] += -m + sh * ws[i];
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < L::SW; ++i) rec[i] = acc[i];
}

// HVP without PSD: forward-over-forward dual on d (exact path)
template <int N>
MG_DI void edge_dual_fof(const EvArgs& a, int64_t e, const double* xa, const double* xb, const double* wa,
                         const double* wb, bool fa, bool fb, double* rec) {
#pragma unroll
  for (int i = 0; i < N; ++i) rec[i] = 0.0;
  for (int ti = 0; ti < a.nterms; ++ti) {
    const TermDev& t = a.terms[ti];
    if (t.op != MG_OP_EV) continue;
    Vec<Df<N, true>, N> d;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      d[c].v = xa[c] - xb[c];
      d[c].vd = (fa ? wa[c] : 0.0) - (fb ? wb[c] : 0.0);
#pragma unroll
      for (int i = 0; i < N; ++i) d[c].g[i] = (i == c) ? 1.0 : 0.0;
    }
    auto r = t.type == MG_TERM_SPRING ? term_eval_diff<MG_TERM_SPRING, N>(t, e, d)
                                      : term_eval_diff<MG_TERM_EDGE_LENGTH, N>(t, e, d);
#pragma unroll
    for (int i = 0; i < N; ++i) rec[i] += r.gd[i];
  }
}


// phi, phi', phi'' of a radial term at r; the attribute value (spring: squared
// rest length) is preloaded. Closed forms of the reference callbacks:
//   spring  (apps/cloth.py:106-110): s = r/l2 - 1, phi = (s s)(c l2),
//           phi' = 2 c s, phi'' = 2 c / l2;   edge length (apps/smooth.py:27-28): phi = r.
// Returns false when a value is non-finite.
// NEEDV = false (HVP): the value is not formed and only the derivative
// factors are checked (an infinite value with finite derivatives leaves the
// reference's Hessian finite too)
template <int TT, bool NEEDV = true>
MG_DI bool radial_closed(const TermDev& t, double a0, double rr, double& pv, double& p1, double& p2) {
  if (TT == MG_TERM_SPRING) {
    const double c = t.c[0];
    const double u = rcp_fast(a0);
    const double sv = rr * u - 1.0;
    pv = NEEDV ? (sv * sv) * (c * a0) : 0.0;
    p1 = 2.0 * c * sv;
    p2 = 2.0 * c * u;
  } else {
    pv = rr;
    p1 = 1.0;
    p2 = 0.0;
  }
  return NEEDV ? isfinite(pv + p1 + p2) : isfinite(p1 + p2);
}

MG_DI bool radial_any(const TermDev& t, double a0, double rr, double& pv, double& p1, double& p2) {
  return t.type == MG_TERM_SPRING ? radial_closed<MG_TERM_SPRING>(t, a0, rr, pv, p1, p2)
                                  : radial_closed<MG_TERM_EDGE_LENGTH>(t, a0, rr, pv, p1, p2);
}


// Closed forms of the two builtin V terms (apps/cloth.py:102-104, 112-113) in
// the dual's operation order: inertia 0.5 m |x - t|^2 (gradient m d, Hessian
// m I exactly as 2 d_i * 0.5 m and 2 * 0.5 m round), gravity -h2 m x.g
// (structurally zero Hessian: floor I under a clamp, problem.py:463-464).
// The attribute loads of the first VPRE terms are issued early (vterms_load)
// so their latency overlaps the incidence gathers. Pinned rows' outputs are
// dropped by the caller, so no masking here; us is the masked direction.
constexpr int VPRE = 2;
template <int N>
struct VPreload {
  double m[VPRE], tg[VPRE][N];
};
template <int N, int MODE, class ST = double>
MG_DI VPreload<N> vterms_load(const EvArgs& a, int g) {
  VPreload<N> v;
#pragma unroll
  for (int j = 0; j < VPRE; ++j) {
    v.m[j] = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) v.tg[j][c] = 0.0;
    if (j < a.nvt) {
      const TermDev& t = a.terms[a.vt_idx[j]];
      v.m[j] = ldv<ST>(t.a[0], g);
      if (MODE != MODE_HVP && t.type == MG_TERM_INERTIA) {
#pragma unroll
        for (int c = 0; c < N; ++c) v.tg[j][c] = ldv<ST>(t.a[1], (int64_t)g * N + c);
      }
    }
  }
  return v;
}
template <int N, int MODE, bool PSD>
MG_DI void vterm_one(const EvArgs& a, const TermDev& t, double m, const double* tg, const double* xs, const double* us,
                     double& eacc, double* vec, double* dg) {
  double hd;  // the term's (clamped) diagonal Hessian entry
  if (t.type == MG_TERM_INERTIA) {
    if constexpr (MODE != MODE_HVP) {
      double d[N], r = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        d[c] = xs[c] - tg[c];
        r = d[c] * d[c] + r;
      }
      eacc += r * (0.5 * m);
#pragma unroll
      for (int c = 0; c < N; ++c) vec[c] += d[c] * m;
    }
    hd = PSD ? (m > a.floor ? m : a.floor) : m;
  } else {
    if constexpr (MODE != MODE_HVP) {
      double dot = xs[0] * t.c[1];
#pragma unroll
      for (int c = 1; c < N; ++c) dot = dot + xs[c] * t.c[1 + c];
      eacc += (dot * m) * (-t.c[0]);
#pragma unroll
      for (int c = 0; c < N; ++c) vec[c] += (t.c[1 + c] * m) * (-t.c[0]);
    }
    hd = PSD ? a.floor : 0.0;
  }
  if constexpr (MODE == MODE_HESS) {
#pragma unroll
    for (int c = 0; c < N; ++c) dg[tri(c, c)] += hd;
  } else if constexpr (MODE == MODE_HVP) {
#pragma unroll
    for (int c = 0; c < N; ++c) vec[c] += hd * us[c];
  }
}
template <int N, int MODE, bool PSD, class ST = double>
MG_DI void vterms_closed(const EvArgs& a, int g, const VPreload<N>& v, const double* xs, const double* us,
                         double& eacc, double* vec, double* dg) {
#pragma unroll
  for (int j = 0; j < VPRE; ++j)
    if (j < a.nvt) vterm_one<N, MODE, PSD>(a, a.terms[a.vt_idx[j]], v.m[j], v.tg[j], xs, us, eacc, vec, dg);
  for (int j = VPRE; j < a.nvt; ++j) {
    const TermDev& t = a.terms[a.vt_idx[j]];
    double tg[N];
#pragma unroll
    for (int c = 0; c < N; ++c)
      tg[c] = (MODE != MODE_HVP && t.type == MG_TERM_INERTIA) ? ldv<ST>(t.a[1], (int64_t)g * N + c) : 0.0;
    vterm_one<N, MODE, PSD>(a, t, ldv<ST>(t.a[0], g), tg, xs, us, eacc, vec, dg);
  }
}

// The builtin terms as a row-kernel policy (edge_rows.cuh): closed forms of
// the V terms with early attribute loads, and the radial closed forms of the
// EV terms; EVT fixes the single EV term's type at compile time (0: any mix,
// dispatched per incidence).
// The energy probe (MODE_ENERGY): every element value in the reference's own
// operations and order, unfused (numpy float64: ActiveVec.norm2 / dot left to
// right, division as a * (1 / b), active.py:180-211, 383-400), so each value
// — NaN / Inf included — is bitwise the reference's; only the sum's order differs.
MG_DI double ref_norm2(const double* d, int n) {
  double t = __dmul_rn(d[0], d[0]);
  for (int c = 1; c < n; ++c) t = __dadd_rn(t, __dmul_rn(d[c], d[c]));
  return t;
}

template <int EVT, class ST = double>
struct BuiltinRows {
  static constexpr bool kXFreeHvp = EVT == MG_TERM_EDGE_LENGTH;
  static constexpr bool kVertexOnly = EVT == MG_TERM_EDGE_LENGTH;
  using Store = ST;
  // energy of one edge at its first vertex (d = x_first - x_second, as the
  // reference's x[verts[0]] - x[verts[1]]): spring (apps/cloth.py:106-110,
  // coef * l2 * (s * s), s = |d|^2 / l2 - 1), edge length (apps/smooth.py:27-28)
  template <int N>
  MG_DI static double evalue(const EvArgs& a, double av, const double* d, uint32_t e) {
    if constexpr (EVT == MG_TERM_SPRING) {
      const double c = a.terms[a.ev_idx[0]].c[0];
      const double s = __dsub_rn(__dmul_rn(ref_norm2(d, N), __ddiv_rn(1.0, av)), 1.0);
      return __dmul_rn(__dmul_rn(c, av), __dmul_rn(s, s));
    } else if constexpr (EVT == MG_TERM_EDGE_LENGTH) {
      return ref_norm2(d, N);
    } else {
      double v = 0.0;
      for (int j = 0; j < a.nev; ++j) {
        const TermDev& t = a.terms[a.ev_idx[j]];
        double x;
        if (t.type == MG_TERM_SPRING) {
          const double l2 = (j == 0 && a.ev_a0) ? av : ldv<ST>(t.a[0], e);
          const double s = __dsub_rn(__dmul_rn(ref_norm2(d, N), __ddiv_rn(1.0, l2)), 1.0);
          x = __dmul_rn(__dmul_rn(t.c[0], l2), __dmul_rn(s, s));
        } else {
          x = ref_norm2(d, N);
        }
        v = j == 0 ? x : __dadd_rn(v, x);
      }
      return v;
    }
  }
  // energies of the row's V terms: inertia 0.5 m |x - t|^2 (apps/cloth.py:102-104),
  // gravity (-h2) (m x.g) (:112-113)
  template <int N>
  MG_DI static double venergy(const EvArgs& a, int g, const VPreload<N>& v, const double* xs) {
    double eacc = 0.0;
    for (int j = 0; j < a.nvt; ++j) {
      const TermDev& t = a.terms[a.vt_idx[j]];
      const double m = j < VPRE ? v.m[j] : ldv<ST>(t.a[0], g);
      double val;
      if (t.type == MG_TERM_INERTIA) {
        double d[N];
#pragma unroll
        for (int c = 0; c < N; ++c) d[c] = __dsub_rn(xs[c], j < VPRE ? v.tg[j][c] : ldv<ST>(t.a[1], (int64_t)g * N + c));
        val = __dmul_rn(__dmul_rn(0.5, m), ref_norm2(d, N));
      } else {
        double dot = __dmul_rn(xs[0], t.c[1]);
#pragma unroll
        for (int c = 1; c < N; ++c) dot = __dadd_rn(dot, __dmul_rn(xs[c], t.c[1 + c]));
        val = __dmul_rn(-t.c[0], __dmul_rn(m, dot));
      }
      eacc += val;
    }
    return eacc;
  }
  template <int N, int MODE>
  MG_DI static VPreload<N> vload(const EvArgs& a, int g) { return vterms_load<N, MODE, ST>(a, g); }
  template <int N, int MODE, bool PSD>
  MG_DI static void vterms(const EvArgs& a, int g, bool, const VPreload<N>& v, const double* xs, const double* us,
                           double& eacc, double* vec, double* dg, bool&) {
    vterms_closed<N, MODE, PSD, ST>(a, g, v, xs, us, eacc, vec, dg);
  }
  template <int MODE>
  MG_DI static double eload(const EvArgs& a, uint32_t e) { return a.ev_a0 ? ldv<ST>(a.ev_a0, e) : 0.0; }
  template <int MODE, bool NEEDV, class F>
  MG_DI static void eterms(const EvArgs& a, double av, double rr, uint32_t e, F&& one) {
    if constexpr (EVT != 0) {
      double pv, p1, p2;
      const bool ok = radial_closed<EVT, NEEDV>(a.terms[a.ev_idx[0]], av, rr, pv, p1, p2);
      one(ok, pv, p1, p2);
    } else {
      for (int j = 0; j < a.nev; ++j) {
        const TermDev& t = a.terms[a.ev_idx[j]];
        const double at = (j == 0 && a.ev_a0) ? av : (t.type == MG_TERM_SPRING ? ldv<ST>(t.a[0], e) : 0.0);
        double pv, p1, p2;
        const bool ok = radial_any(t, at, rr, pv, p1, p2);
        one(ok, pv, p1, p2);
      }
    }
  }
};

template <int N, int MODE, bool PSD, int EVT, class ST = double>
__global__ void __launch_bounds__(FastCfg<MODE, PSD>::BLOCK,
                                  (FastMinb<MODE, PSD, BuiltinRows<EVT>::kXFreeHvp>::v))
    k_rows_fast(const __grid_constant__ EvArgs a) {
  rows_fast_body<N, MODE, PSD, BuiltinRows<EVT, ST>>(a);
}

// Staged tile kernel, persistent and software-pipelined. Dispatched for the
// unclamped spring-family HVP (the cloth Newton-CG operator), where it beats
// the row kernel (0.251 vs 0.288 ms at 2048^2); the gradient and clamped-HVP
// branches are kept compiled-out (measured slower than the row kernel).
// Rows are cut into tiles of EV_TILE_ROWS (patch order); tile b owns a padded
// vertex table (its rows, then its halo) and edge table (every edge incident
// to one of its rows, once). A CTA walks tiles b, b + grid, ...; while it
// computes tile i, the gathers of tile i+1 (x, w, the edge attribute) are in
// flight as cp.async copies into the other shared-memory stage and the table
// entries of tile i+2 are in flight into registers, so a tile's dependent
// loads (table -> vertex data) never stall the SM. Per tile:
//   edges: each edge is evaluated ONCE into a per-edge record: the
//          contribution to its first vertex (the second gets the negation:
//          radial blocks are even in d) plus, under a PSD clamp, the
//          symmetric floor term;
//   rows:  V terms, then the incidences' records in their fixed order
//          (bitwise reproducible), one store per output row.
// The energy counts each edge in the tile of its first vertex.
#ifndef EV_TILE_MINB
#define EV_TILE_MINB 4
#endif
constexpr int TILE_IPT = 8;  // incidence slots per row in one 16-byte load

MG_DI void cp_async8(void* smem, const void* gmem, bool zero) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(zero ? 0 : 8) : "memory");
}

// one tile's share of the tables, held by each thread
struct TileRegs {
  int nv = 0, ne = 0;
  uint32_t tv[EV_TILE_VPT];
  uint64_t te[EV_TILE_EPT];
  uint4 sl4;
  uint32_t meta;
};

template <int N, int MODE, bool PSD, int EVT>
__global__ void __launch_bounds__(EV_TILE_ROWS, EV_TILE_MINB) k_tile_ev(const __grid_constant__ EvArgs a) {
  static_assert(MODE == MODE_GRAD || MODE == MODE_HVP, "tile kernel: gradient / HVP");
  constexpr int TB = EV_TILE_ROWS, VPT = EV_TILE_VPT, EPT = EV_TILE_EPT;
  constexpr int SW = (MODE == MODE_HVP && PSD) ? 2 * N : N;
  constexpr bool XFREE = MODE == MODE_HVP && !PSD && EVT == MG_TERM_EDGE_LENGTH;
  constexpr bool W = MODE == MODE_HVP;
  constexpr int XW = (XFREE ? 0 : N) + (W ? N : 0);  // doubles per vertex-table entry
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int MV = a.max_v, ME = a.max_e;
  const int64_t nt = (a.V + TB - 1) / TB;
  // stage layout (component-major): x (N, MV) | w (N, MV) | attribute (ME) | flags (MV bytes)
  const int stage_d = XW * MV + ME + (MV + 7) / 8;
  double* sr = sm + 2 * stage_d;  // (SW, ME) edge records
  auto sx = [&](int st) { return sm + st * stage_d; };
  auto sw = [&](int st) { return sm + st * stage_d + (XFREE ? 0 : N * MV); };
  auto sa0 = [&](int st) { return sm + st * stage_d + XW * MV; };
  auto sfl = [&](int st) { return reinterpret_cast<uint8_t*>(sm + st * stage_d + XW * MV + ME); };

  auto load_tables = [&](int64_t b, TileRegs& r) {
    const int2 c = a.tcnt[b];
    r.nv = c.x;
    r.ne = c.y;
#pragma unroll
    for (int k = 0; k < VPT; ++k) r.tv[k] = tid + k * TB < MV ? a.tv[b * MV + tid + k * TB] : 0u;
#pragma unroll
    for (int k = 0; k < EPT; ++k) r.te[k] = tid + k * TB < ME ? a.te[b * ME + tid + k * TB] : 0ull;
    const int64_t row = b * TB + tid;
    r.sl4 = row < a.V ? reinterpret_cast<const uint4*>(a.islot8)[row] : make_uint4(0, 0, 0, 0);
    r.meta = row < a.V ? a.rmeta[row] : 0u;
  };
  auto issue_gathers = [&](int64_t b, const TileRegs& r, int st) {
    double* x_ = sx(st);
    double* w_ = sw(st);
    uint8_t* f_ = sfl(st);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int i = tid + k * TB;
      if (i < r.nv) {
        const int64_t gv = r.tv[k] & 0x7fffffffu;
        const bool f = !(r.tv[k] >> 31);
#pragma unroll
        for (int c = 0; c < N; ++c) {
          if constexpr (!XFREE) cp_async8(x_ + c * MV + i, a.x + gv * N + c, false);
          if constexpr (W) cp_async8(w_ + c * MV + i, a.w + gv * N + c, !f);
        }
        f_[i] = f;
      }
    }
    if (a.ev_a0) {
      double* a_ = sa0(st);
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int j = tid + k * TB;
        if (j < r.ne) cp_async8(a_ + j, a.ev_a0 + (uint32_t)r.te[k], false);
      }
    }
    // the rows' V-term attributes (masses; the inertia target for the gradient) into L1
    const int64_t row = b * TB + tid;
    if (row < a.V) {
      const int64_t g = r.tv[0] & 0x7fffffffu;
      for (int j = 0; j < a.nvt; ++j) {
        const TermDev& t = a.terms[a.vt_idx[j]];
        asm volatile("prefetch.global.L1 [%0];" ::"l"(t.a[0] + g));
        if (MODE == MODE_GRAD && t.type == MG_TERM_INERTIA) asm volatile("prefetch.global.L1 [%0];" ::"l"(t.a[1] + g * N));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int64_t b = blockIdx.x;
  if (b >= nt) return;
  TileRegs cur, nxt;
  load_tables(b, cur);
  issue_gathers(b, cur, 0);
  if (b + gridDim.x < nt) load_tables(b + gridDim.x, nxt);
  bool finite = true;
  for (int it = 0; b < nt; ++it, b += gridDim.x) {
    const int st = it & 1;
    const int64_t bn = b + gridDim.x;
    if (bn < nt) issue_gathers(bn, nxt, st ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    TileRegs use = cur;
    cur = nxt;
    if (bn + gridDim.x < nt) load_tables(bn + gridDim.x, nxt);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    // ---- edges of tile b
    const double* x_ = sx(st);
    const double* w_ = sw(st);
    const double* a_ = sa0(st);
    const uint8_t* f_ = sfl(st);
    const int64_t rem = a.V - b * TB;
    const int nrows = rem < TB ? (int)rem : TB;
    double eacc = 0.0;
    auto edge = [&](int idx, uint64_t rec) {
      const uint32_t e = (uint32_t)rec;
      const int la = (int)((rec >> 32) & 0xffffu), lb = (int)(rec >> 48);
      const bool fa = f_[la], fb = f_[lb];
      const double av = a.ev_a0 ? a_[idx] : 0.0;
      double d[N], rr = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        d[c] = XFREE ? 0.0 : x_[c * MV + la] - x_[c * MV + lb];
        rr = d[c] * d[c] + rr;
      }
      double gam = 0.0, ci_s = 0.0, cd_s = 0.0, dl = 0.0, val = 0.0;
      auto one_term = [&](bool ok, double pv, double p1, double p2) {
        finite &= ok;
        val += pv;
        gam += 2.0 * p1;
        if constexpr (MODE == MODE_HVP) {
          double ci = 2.0 * p1, cd = 4.0 * p2, sh = 0.0;
          if constexpr (PSD) {
            if (fa && fb) {  // [[A,-A],[-A,A]]: clamp 2A, halve, shift floor/2
              ci *= 2.0; cd *= 2.0;
              radial_clamp_fast(ci, cd, rr, a.floor);
              ci *= 0.5; cd *= 0.5;
              sh = 0.5 * a.floor;
            } else if (fa || fb) {
              radial_clamp_fast(ci, cd, rr, a.floor);
            }
          }
          ci_s += ci;
          cd_s += cd;
          dl += sh;
        }
      };
      if constexpr (EVT != 0) {
        double pv, p1, p2;
        const bool ok = radial_closed<EVT, MODE != MODE_HVP>(a.terms[a.ev_idx[0]], av, rr, pv, p1, p2);
        one_term(ok, pv, p1, p2);
      } else {
        for (int j = 0; j < a.nev; ++j) {
          const TermDev& t = a.terms[a.ev_idx[j]];
          const double at = (j == 0 && a.ev_a0) ? av : (t.type == MG_TERM_SPRING ? t.a[0][e] : 0.0);
          double pv, p1, p2;
          const bool ok = radial_any(t, at, rr, pv, p1, p2);
          one_term(ok, pv, p1, p2);
        }
      }
      if constexpr (MODE == MODE_GRAD) {
        if (la < nrows) eacc += val;  // the edge's first vertex is a row of this tile
#pragma unroll
        for (int c = 0; c < N; ++c) sr[c * ME + idx] = gam * d[c];
      } else {
        double dw = 0.0, du[N];
#pragma unroll
        for (int c = 0; c < N; ++c) {
          du[c] = w_[c * MV + la] - w_[c * MV + lb];
          dw += d[c] * du[c];
        }
#pragma unroll
        for (int c = 0; c < N; ++c) sr[c * ME + idx] = ci_s * du[c] + cd_s * d[c] * dw;
        if constexpr (PSD) {
#pragma unroll
          for (int c = 0; c < N; ++c) sr[(N + c) * ME + idx] = dl * (w_[c * MV + la] + w_[c * MV + lb]);
        }
      }
    };
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (tid + k * TB < use.ne) edge(tid + k * TB, use.te[k]);
    __syncthreads();
    // ---- rows of tile b
    const int64_t row = b * TB + tid;
    if (tid < nrows) {
      const int g = (int)(use.tv[0] & 0x7fffffffu);
      const bool fr = f_[tid];
      double vec[N], xs[N], us[N];
#pragma unroll
      for (int c = 0; c < N; ++c) {
        vec[c] = 0.0;
        xs[c] = XFREE ? 0.0 : x_[c * MV + tid];
        us[c] = W ? w_[c * MV + tid] : 0.0;
      }
      double dgv[TriN<N>::value];
      vterms_closed<N, MODE, PSD>(a, g, vterms_load<N, MODE>(a, g), xs, us, eacc, vec, dgv);
      auto inc = [&](uint32_t s16) {
        const int sl = (int)(s16 & 0x7fff);
        const bool neg = (s16 >> 15) & 1;  // the row is the edge's second vertex
#pragma unroll
        for (int c = 0; c < N; ++c) {
          const double r = sr[c * ME + sl];
          double v = neg ? -r : r;
          if constexpr (MODE == MODE_HVP && PSD) v += sr[(N + c) * ME + sl];
          vec[c] += v;
        }
      };
      int cnt = (int)(use.meta & 0xff);
      if (cnt == 255) cnt = a.rinc_off[row + 1] - a.rinc_off[row];
      const uint32_t w4[4] = {use.sl4.x, use.sl4.y, use.sl4.z, use.sl4.w};
#pragma unroll
      for (int j = 0; j < TILE_IPT; ++j)
        if (j < cnt) inc((w4[j >> 1] >> (16 * (j & 1))) & 0xffffu);
      if (cnt > TILE_IPT) {
        const int k0 = a.rinc_off[row];
        for (int k = TILE_IPT; k < cnt; ++k) inc(a.islot[k0 + k]);
      }
      double* vout = MODE == MODE_HVP ? a.y : a.grad;
#pragma unroll
      for (int i = 0; i < N; ++i) vout[(int64_t)g * N + i] = fr ? vec[i] : 0.0;
    }
    if constexpr (MODE == MODE_GRAD) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(0xffffffffu, eacc, o);
      if ((tid & 31) == 0) a.partials[row >> 5] = eacc;
    }
    __syncthreads();  // stage st and the records are rewritten next
  }
  if (!finite) *a.redo = 1;
}

// EXACT = false: radial evaluation only; a non-finite lane raises *a.redo.
// EXACT = true : launched after it; returns at once unless *a.redo is set,
//                then recomputes every row with the exact K = n dual path.
template <int N, int MODE, bool PSD, bool EXACT>
__global__ void __launch_bounds__(PT) k_rows_ev(const __grid_constant__ EvArgs a) {
  using L = EvRec<N, MODE, PSD>;
  constexpr int T = L::T, SW = L::SW, NN = N * N;
  extern __shared__ __align__(16) double hbuf[];  // this CTA's rows in output layout
  if constexpr (EXACT) {
    if (*(volatile const int*)a.redo == 0) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.exact_runs, 1);
  }
  const int64_t nblk = (a.V + PT - 1) / PT;
  if constexpr (EXACT && MODE != MODE_HVP) {
    for (int64_t i = nblk * (PT / 32) + blockIdx.x * (int64_t)PT + threadIdx.x; i < a.np_total;
         i += (int64_t)gridDim.x * PT)
      a.partials[i] = 0.0;
  }
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
  const int64_t row = blk * PT + threadIdx.x;
  double eacc = 0.0;
  bool finite = true;
  if (row < a.V) {
    const int g = a.order ? a.order[row] : (int)row;
    const bool fr = !a.pfix[row];
    const int k0 = a.rinc_off[row], k1 = a.rinc_off[row + 1];
    int64_t ro = 0;
    int len = 0, dp = 255, ho = 0;
    if constexpr (MODE == MODE_HESS) {
      ro = a.prow_ro[row];
      len = a.prow_len[row];
      dp = a.prow_dp[row];
      ho = a.hoff[row];
    }
    double xs[N], wsv[N];
#pragma unroll
    for (int c = 0; c < N; ++c) {
      xs[c] = a.x[(int64_t)g * N + c];
      if constexpr (MODE == MODE_HVP) wsv[c] = a.w[(int64_t)g * N + c];
      else wsv[c] = 0.0;
    }
    double vec[N], dg[T];
#pragma unroll
    for (int i = 0; i < N; ++i) vec[i] = 0.0;
#pragma unroll
    for (int i = 0; i < T; ++i) dg[i] = 0.0;
    // V terms
    {
      const double* xr[1] = {xs};
      const double* wr[1] = {wsv};
      for (int ti = 0; ti < a.nterms; ++ti) {
        const TermDev& t = a.terms[ti];
        if (t.op != MG_OP_V) continue;
        if (t.type == MG_TERM_INERTIA) {
          ElemOut<MG_TERM_INERTIA, N, MODE, PSD> o;
          eval_element<MG_TERM_INERTIA, N, MODE, PSD>(t, g, &g, xr, wr, &fr, a.floor, o);
          eacc += o.val;
#pragma unroll
          for (int k = 0; k < N; ++k) vec[k] += o.g[k];
          if constexpr (MODE == MODE_HESS) {
            if (o.has_h)
#pragma unroll
              for (int k = 0; k < T; ++k) dg[k] += o.h[k];
          }
        } else if (t.type == MG_TERM_GRAVITY) {
          ElemOut<MG_TERM_GRAVITY, N, MODE, PSD> o;
          eval_element<MG_TERM_GRAVITY, N, MODE, PSD>(t, g, &g, xr, wr, &fr, a.floor, o);
          eacc += o.val;
#pragma unroll
          for (int k = 0; k < N; ++k) vec[k] += o.g[k];
          if constexpr (MODE == MODE_HESS) {
            if (o.has_h)
#pragma unroll
              for (int k = 0; k < T; ++k) dg[k] += o.h[k];
          }
        }
      }
    }
    // incident edges in column order; the diagonal block's position is where
    // the column passes g (free neighbours only own a block)
    double* hrow = hbuf + ho;
    int pos = 0;
    uint64_t nrc = k0 < k1 ? a.rrec[k0] : 0;
    for (int k = k0; k < k1; ++k) {
      const uint64_t rc = nrc;
      if (k + 1 < k1) nrc = a.rrec[k + 1];
      const uint32_t lo = (uint32_t)rc, hi = (uint32_t)(rc >> 32);
      const int64_t e = lo & 0x7fffffffu;
      const int q = (int)(lo >> 31);
      const int o = (int)(hi & 0x7fffffffu);
      const bool fo = !(hi >> 31);
      double xo[N], wo[N];
#pragma unroll
      for (int c = 0; c < N; ++c) {
        xo[c] = a.x[(int64_t)o * N + c];
        if constexpr (MODE == MODE_HVP) wo[c] = a.w[(int64_t)o * N + c];
        else wo[c] = 0.0;
      }
      // canonical orientation: slot 0 is the edge's first vertex (values
      // selected, not pointers, so everything stays in registers)
      double xa[N], xb[N], wa[N], wb[N];
#pragma unroll
      for (int c = 0; c < N; ++c) {
        xa[c] = q == 0 ? xs[c] : xo[c];
        xb[c] = q == 0 ? xo[c] : xs[c];
        wa[c] = q == 0 ? wsv[c] : wo[c];
        wb[c] = q == 0 ? wo[c] : wsv[c];
      }
      const bool fa = q == 0 ? fr : fo, fb = q == 0 ? fo : fr;
      double rec[SW], val, dl;
      if constexpr (EXACT) {
        if constexpr (MODE == MODE_HVP && !PSD) edge_dual_fof<N>(a, e, xa, xb, wa, wb, fa, fb, rec);
        else edge_dual<N, MODE, PSD>(a, e, xa, xb, wa, wb, fa, fb, val, rec, dl);
      } else {
        finite &= edge_radial<N, MODE, PSD>(a, e, xa, xb, wa, wb, fa, fb, val, rec, dl);
      }
      if constexpr (MODE != MODE_HVP) {
        if (q == 0) eacc += val;  // an edge's energy counts at its first vertex
      }
      if constexpr (MODE == MODE_HVP && PSD) {
#pragma unroll
        for (int i = 0; i < N; ++i) vec[i] += rec[q * N + i];
      } else {
        const double sg = q == 0 ? 1.0 : -1.0;
#pragma unroll
        for (int i = 0; i < N; ++i) vec[i] += sg * rec[i];
      }
      if constexpr (MODE == MODE_HESS) {
#pragma unroll
        for (int i = 0; i < T; ++i) dg[i] += rec[N + i];
        if (fr && fo) {
          if (dp != 255 && pos == dp) ++pos;  // leave the diagonal's slot
          double* dst = hrow + pos * NN;
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int c = 0; c < N; ++c) dst[i * N + c] = -rec[N + tri(i, c)] + (i == c ? 2.0 * dl : 0.0);
          ++pos;
        }
      }
    }
    double* vout = MODE == MODE_HVP ? a.y : a.grad;
#pragma unroll
    for (int i = 0; i < N; ++i) vout[(int64_t)g * N + i] = fr ? vec[i] : 0.0;
    if constexpr (MODE == MODE_HESS) {
      if (fr && dp != 255) {
        double* dst = hrow + dp * NN;
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int c = 0; c < N; ++c) dst[i * N + c] = dg[tri(i, c)];
      }
      // blocks written: off-diagonals, plus the diagonal if the walk never passed it
      const int len = (fr && dp != 255) ? (pos > dp + 1 ? pos : dp + 1) : pos;
      if (len > 0) {
        fence_proxy_async_smem();
        row_store_bulk(a.hess + ro * NN, hrow, len * NN);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
  }
  if constexpr (!EXACT) {
    if (!finite) *a.redo = 1;
  }
  if constexpr (MODE != MODE_HVP) {
    // fixed-order warp partial (no block barrier)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(0xffffffffu, eacc, o);
    if ((threadIdx.x & 31) == 0) a.partials[(blk * PT + threadIdx.x) >> 5] = eacc;
  }
  }  // row blocks
}

// MG_EDGE_TILES=0 selects the per-row kernel for gradient / HVP (A/B runs)
bool tiles_enabled() {
  static const bool on = [] {
    const char* e = getenv("MG_EDGE_TILES");
    return !(e && e[0] == '0');
  }();
  return on;
}

// MG_PERSISTENT=1: a persistent grid for the Hessian row kernel (measured
// slightly slower than one row block per CTA: the hardware block scheduler
// already overlaps a finishing CTA's stores with a starting CTA's loads)
bool persistent_enabled() {
  static const bool on = [] {
    const char* e = getenv("MG_PERSISTENT");
    return e && e[0] == '1';
  }();
  return on;
}

// grid of a gradient / HVP row kernel: one row block per CTA, or with
// EV_FLAT_PERSIST a persistent grid of resident CTAs
template <class K>
int64_t flat_grid(K kern, int64_t V, int block) {
  const int64_t nb = (V + block - 1) / block;
  if (!EV_FLAT_PERSIST && !EV_STAGED) return nb;
  int dev = 0, sms = 148, per_sm = 1;
  MG_CUDA(cudaGetDevice(&dev));
  MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, 0));
  const int64_t g = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  return g < nb ? g : nb;
}

template <int N, int MODE, bool PSD, int EVT, class ST>
void launch_rows_t(const Problem& p, const EvArgs& a, int hd_max, cudaStream_t st) {
  constexpr bool F32 = sizeof(ST) == 4;  // fp32 storage: no row buffers, no fp64-only variants
  const size_t sm = MODE == MODE_HESS ? (size_t)hd_max * 8 + 16 : 0;
  if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "row block does not fit in shared memory");
  const int64_t nb = (a.V + PT - 1) / PT;
  if (!nb) return;
  auto fast = k_rows_fast<N, MODE, PSD, EVT, ST>;
  // (the energy probe's values are the reference's own operations: no exact re-run)
  constexpr int XMODE = MODE == MODE_ENERGY ? MODE_GRAD : MODE;
  auto exact = k_rows_ev<N, XMODE, PSD, true>;
  if (sm) {
    MG_CUDA(cudaFuncSetAttribute(fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    MG_CUDA(cudaFuncSetAttribute(exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  }
  timing_begin(p, st);
  if constexpr (MODE == MODE_HVP && !PSD && EVT != MG_TERM_EDGE_LENGTH) {
    if (!F32 && p.tiles_ready && tiles_enabled()) {
      constexpr int SW = (MODE == MODE_HVP && PSD) ? 2 * N : N;
      constexpr bool XF = MODE == MODE_HVP && !PSD && EVT == MG_TERM_EDGE_LENGTH;
      constexpr int XW = (XF ? 0 : N) + (MODE == MODE_HVP ? N : 0);
      const size_t stage_d = (size_t)XW * a.max_v + a.max_e + (a.max_v + 7) / 8;
      const size_t ts = sizeof(double) * (2 * stage_d + (size_t)SW * a.max_e);
      auto tk = k_tile_ev<N, MODE, PSD, EVT>;
      if (ts > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "edge tile does not fit in shared memory");
      MG_CUDA(cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ts));
      int dev = 0, sms = 148, per_sm = 1;
      MG_CUDA(cudaGetDevice(&dev));
      MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tk, EV_TILE_ROWS, ts));
      const int64_t nt = (a.V + EV_TILE_ROWS - 1) / EV_TILE_ROWS;
      int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
      if (grid > nt) grid = nt;
      tk<<<(unsigned)grid, EV_TILE_ROWS, ts, st>>>(a);
      MG_LAUNCH_CHECK();
      timing_end(p, st);
    } else {
      constexpr int FB = FastCfg<MODE, PSD>::BLOCK;
      fast<<<(unsigned)flat_grid(fast, a.V, FB), FB, sm, st>>>(a);
      MG_LAUNCH_CHECK();
      timing_end(p, st);
    }
  } else {
    // Hessian: one row block per CTA (or, opt-in, a persistent grid whose
    // threads walk their rows with the next row's level-1 streams in flight)
    constexpr int FB = FastCfg<MODE, PSD>::BLOCK;
    const int64_t nfb = (a.V + FB - 1) / FB;
    int64_t grid = MODE == MODE_HESS ? nfb : flat_grid(fast, a.V, FB);
    if (MODE == MODE_HESS && (persistent_enabled() || EV_STAGED_HESS)) {
      int dev = 0, sms = 148, per_sm = 1;
      MG_CUDA(cudaGetDevice(&dev));
      MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fast, FB, sm));
      const int64_t g = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
      if (g < grid) grid = g;
    }
    fast<<<(unsigned)grid, FB, sm, st>>>(a);
    MG_LAUNCH_CHECK();
    timing_end(p, st);
  }
  // fp32 storage: the closed forms' own NaN / Inf propagation (the exact K = n
  // dual re-run is fp64)
  if constexpr (MODE == MODE_ENERGY || F32) return;
  // exact re-run only when a lane was non-finite (reads the flag and exits otherwise)
  int dev = 0, sms = 148;
  MG_CUDA(cudaGetDevice(&dev));
  MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t ge = nb < (int64_t)sms * 4 ? nb : (int64_t)sms * 4;
  exact<<<(unsigned)ge, PT, sm, st>>>(a);
  MG_LAUNCH_CHECK();
}

template <int N, int MODE, bool PSD>
void launch_rows(const Problem& p, const EvArgs& a, int hd_max, cudaStream_t st) {
  const int t0 = a.nev == 1 ? a.terms[a.ev_idx[0]].type : 0;
  if (p.store32) {
    if (t0 == MG_TERM_SPRING) launch_rows_t<N, MODE, PSD, MG_TERM_SPRING, float>(p, a, hd_max, st);
    else if (t0 == MG_TERM_EDGE_LENGTH) launch_rows_t<N, MODE, PSD, MG_TERM_EDGE_LENGTH, float>(p, a, hd_max, st);
    else launch_rows_t<N, MODE, PSD, 0, float>(p, a, hd_max, st);
    return;
  }
  if (t0 == MG_TERM_SPRING) launch_rows_t<N, MODE, PSD, MG_TERM_SPRING, double>(p, a, hd_max, st);
  else if (t0 == MG_TERM_EDGE_LENGTH) launch_rows_t<N, MODE, PSD, MG_TERM_EDGE_LENGTH, double>(p, a, hd_max, st);
  else launch_rows_t<N, MODE, PSD, 0, double>(p, a, hd_max, st);
}

template <int N>
void launch_rows_mode(const Problem& p, const EvArgs& a, int hd, Mode mode, bool psd, cudaStream_t st) {
  switch (mode) {
    case MODE_ENERGY: launch_rows<N, MODE_ENERGY, false>(p, a, hd, st); break;
    case MODE_GRAD: launch_rows<N, MODE_GRAD, false>(p, a, hd, st); break;
    case MODE_HESS:
      if (psd) launch_rows<N, MODE_HESS, true>(p, a, hd, st);
      else launch_rows<N, MODE_HESS, false>(p, a, hd, st);
      break;
    case MODE_HVP:
      if (psd) launch_rows<N, MODE_HVP, true>(p, a, hd, st);
      else launch_rows<N, MODE_HVP, false>(p, a, hd, st);
      break;
    default: throw Error(MG_ERR_UNSUPPORTED, "edge row kernel evaluates energy / grad / Hessian / HVP only");
  }
}

}  // namespace

namespace {

void fill_ev_args(const Problem& p, const LaunchCtx& c, int64_t partial_offset, EvArgs& a) {
  const Mesh& m = *p.mesh;
  if (p.terms.size() > MAXT) throw Error(MG_ERR_UNSUPPORTED, "at most 8 terms per problem on the patch path");
  std::memset(&a, 0, sizeof(a));
  a.nterms = (int)p.terms.size();
  a.V = m.Vr;
  a.order = (m.row_order_used == MG_ROW_IDENTITY && !m.owned.p) ? nullptr
            : (p.order_pad.n >= m.Vr && p.order_pad.p ? p.order_pad.p : m.patches.order.p);
  a.pfix = p.pfix.p;
  a.rmeta = p.rmeta.p;
  a.ell = p.ell.p;
  a.ell32 = p.ell32_ok ? p.ell32.p : nullptr;
  a.es = p.ell_stride ? p.ell_stride : m.Vr;
  a.rinc_off = p.rinc_off.p;
  a.rrec = p.rrec.p;
  a.prow_ro = p.prow_ro.p;
  a.prow_len = p.prow_len.p;
  a.prow_dp = p.prow_dp.p;
  a.hoff = p.hoff.p;
  a.x = c.x;
  a.w = c.w;
  a.grad = c.grad;
  a.hess = c.hess;
  a.y = c.y;
  a.partials = c.partials + partial_offset;
  a.redo = p.redo.p;
  a.exact_runs = p.exact_runs.p;
  a.floor = c.floor;
  for (int i = 0; i < a.nterms; ++i) a.terms[i] = p.terms[i].dev;
  a.nev = a.nvt = 0;
  a.ev_a0 = nullptr;
  a.tcnt = p.tcnt.p;
  a.tv = p.tv.p;
  a.te = p.te.p;
  a.islot = p.islot.p;
  a.islot8 = p.islot8.p;
  a.max_v = p.tile_max_v;
  a.max_e = p.tile_max_e;
  for (int i = 0; i < a.nterms; ++i) {
    if (p.terms[i].dev.op == MG_OP_EV) a.ev_idx[a.nev++] = i;
    else a.vt_idx[a.nvt++] = i;
  }
}

}  // namespace

int64_t launch_patch_ev(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  const Mesh& m = *p.mesh;
  EvArgs a;
  fill_ev_args(p, c, partial_offset, a);
  if (a.nev && p.terms[a.ev_idx[0]].dev.type == MG_TERM_SPRING) a.ev_a0 = p.terms[a.ev_idx[0]].dev.a[0];
  const int hd = mode == MODE_HESS ? p.max_patch_hdoubles : 0;
  // energy partials: one per warp of rows
  const int64_t np = mode == MODE_HVP ? 0 : (m.Vr + 31) / 32;
  a.np_total = np;
  if (p.n == 3) launch_rows_mode<3>(p, a, hd, mode, c.psd, c.stream);
  else launch_rows_mode<2>(p, a, hd, mode, c.psd, c.stream);
  return np;
}

// Traced terms with radial EV callbacks (jit_rows.cuh): the same row layout
// and kernel body, the problem's generated policy; the attribute streams of
// all its terms, in term order, in EvArgs::js. No exact re-run here: the
// caller launches the traced patch module gated on the redo flag.
bool rows_jit_supported(const Problem& p) {
  if (!p.row_module || p.terms.empty() || p.terms.size() > (size_t)MAXT) return false;
  if (p.n != 2 && p.n != 3) return false;
  size_t streams = 0;
  bool any_ev = false;
  for (auto& t : p.terms) {
    if (!t.jit || (t.dev.op != MG_OP_V && t.dev.op != MG_OP_EV)) return false;
    any_ev |= t.dev.op == MG_OP_EV;
    streams += t.jit_attrs.size();
  }
  return any_ev && streams <= (size_t)MAX_JS && p.mesh->E < (int64_t(1) << 31);
}

int64_t launch_rows_jit(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  const Mesh& m = *p.mesh;
  EvArgs a;
  fill_ev_args(p, c, partial_offset, a);
  int js = 0;
  for (auto& t : p.terms)
    for (auto* ptr : t.jit_attrs) {
      if (js >= MAX_JS) throw Error(MG_ERR_UNSUPPORTED, "row module: too many attribute streams");
      a.js[js++] = ptr;
    }
  const int64_t np = mode == MODE_HVP ? 0 : (m.Vr + 31) / 32;
  a.np_total = np;
  const size_t sm = mode == MODE_HESS ? (size_t)p.max_patch_hdoubles * 8 + 16 : 0;
  if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "row block does not fit in shared memory");
  const int B = mode == MODE_HESS ? FastCfg<MODE_HESS, false>::BLOCK
                : mode == MODE_GRAD ? FastCfg<MODE_GRAD, false>::BLOCK
                : c.psd ? FastCfg<MODE_HVP, true>::BLOCK : FastCfg<MODE_HVP, false>::BLOCK;
  const int64_t grid = (m.Vr + B - 1) / B;
  const bool persistent = mode == MODE_HESS ? EV_STAGED_HESS : EV_STAGED;
  timing_begin(p, c.stream);
  jit_rows_launch(p, mode, c.psd, &a, grid, B, sm, c.stream, persistent);
  timing_end(p, c.stream);
  return np;
}

}  // namespace mg
