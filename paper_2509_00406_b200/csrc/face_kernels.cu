// Face row kernel: the patch-owner assembly specialised to the symmetric
// Dirichlet distortion energy (apps/param.py:170-177), BASELINE config 3.
//
// The energy of a face depends on its six UV variables only through the 2x2
// Jacobian J = [x1 - x0, x2 - x0] R (R = rest_inv), a linear map J = B x with
// B = I_2 (x) W, W[k][q] the constant weights of vertex q (W 1 = 0). So:
//   * value, gradient and Hessian come from a K = 4 second-order dual on the
//     entries of J (10 Hessian entries instead of the K = 6 dual's 21), then
//     g_x = B^T g_J and H_x = B^T H_J B (chain rule; the reference's K = 6 dual
//     gives the same values to rounding);
//   * the PSD clamp of the 6x6 block (active.py:490-504) reduces to a 4x4
//     eigenproblem: with Q_W an orthonormal basis of 1-perp, W = L_W Q_W^T and
//     P_f(H_x) = (I (x) Q_W) P_f(M) (I (x) Q_W)^T + f (I (x) 1 1^T / 3),
//     M = (I (x) L_W)^T H_J (I (x) L_W) — the two translation modes sit at
//     eigenvalue 0 and clamp to the floor exactly as the reference's eigh does.
// One thread per owned row (Morton patch order, as the edge row kernel): it
// walks the row's incident faces (ELL / CSR incidence records built at
// setup), evaluates each face, accumulates gradient / HVP and the diagonal
// block in registers and the off-diagonal blocks in its shared-memory row
// buffer (output layout), and streams the finished row to HBM with one bulk
// copy. Each face is evaluated by each of its (up to three) owner rows:
// recompute instead of communicate; the FP64 work per face is small.
// Faces with non-finite values, or pinned corners under a PSD clamp, raise the
// redo flag: the generic patch kernel then recomputes the whole call exactly.
#include "elem_eval.cuh"
#include "mg_internal.cuh"
#include "psd.cuh"

namespace mg {

namespace {

constexpr int PT = EV_ROW_BLOCK;
constexpr int KF = EV_ELL_K;  // face incidences per row in the ELL part
constexpr double INV_SQRT2 = 0.70710678118654752440;
constexpr double INV_SQRT6 = 0.40824829046386301637;

struct FvArgs {
  int64_t V;
  const int32_t* order;
  const uint32_t* rmeta;     // incidence count (sat. 255) | pinned << 8 | diagonal position << 16
  const uint64_t* ell;       // (KF, V) slot-major incidence records
  const int32_t* rinc_off;   // (V+1) CSR of all incidences
  const uint64_t* rrec;
  const int64_t* prow_ro;
  const int32_t* hoff;
  const int32_t* faces;      // (F,3)
  const double* x;
  const double* w;
  double* grad;
  double* hess;
  double* y;
  double* partials;
  int* redo;
  double floor;
  TermDev t;                 // the SymDirichlet term: a[0] rest_inv (F,4), a[1] areas (F)
};

MG_DI void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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

// f(J) of the symmetric Dirichlet term on a K = 4 dual over the entries of J
// (same operation order as terms.cuh / apps/param.py:170-177)
MG_DI Dh<4, false> dirichlet_J(const double* J, double area) {
  Dh<4, true> j[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    j[a].v = J[a];
#pragma unroll
    for (int b = 0; b < 4; ++b) j[a].g[b] = a == b ? 1.0 : 0.0;
  }
  auto det = positive_guard(j[0] * j[3] - j[1] * j[2]);
  auto fro = j[0] * j[0] + 0.0;
  fro = j[1] * j[1] + fro;
  fro = j[2] * j[2] + fro;
  fro = j[3] * j[3] + fro;
  return (fro + fro / (det * det)) * area;
}

template <int MODE, bool PSD>
__global__ void __launch_bounds__(PT) k_rows_dirichlet(const __grid_constant__ FvArgs a) {
  constexpr int N = 2, NN = 4;
  extern __shared__ __align__(16) double hbuf[];
  const int64_t row = (int64_t)blockIdx.x * PT + threadIdx.x;
  double eacc = 0.0;
  bool ok = true;
  if (row < a.V) {
    const int g = a.order[row];
    const uint32_t meta = a.rmeta[row];
    int64_t ro = 0;
    int ho = 0;
    if constexpr (MODE == MODE_HESS) {
      ro = a.prow_ro[row];
      ho = a.hoff[row];
    }
    uint64_t rc[KF];
#pragma unroll
    for (int j = 0; j < KF; ++j) rc[j] = a.ell[(int64_t)j * a.V + row];
    const bool fr = !((meta >> 8) & 1);
    const int dp = (int)(meta >> 16) & 0xff;
    const int cnt = (meta & 0xff) < 255 ? (int)(meta & 0xff) : a.rinc_off[row + 1] - a.rinc_off[row];
    double* hrow = hbuf + ho;
    int nblk = 0;
    if constexpr (MODE == MODE_HESS) {
      // the row's blocks: off-diagonals accumulate (two faces per edge), so clear first
      nblk = (int)(((meta >> 24) & 0xff));
      for (int k = 0; k < nblk * NN; ++k) hrow[k] = 0.0;
    }
    double vec[N] = {0.0, 0.0}, dg[3] = {0.0, 0.0, 0.0};
    const double* R_all = a.t.a[0];
    const double* A_all = a.t.a[1];
    auto incidence = [&](uint64_t r64) {
      const uint32_t lo = (uint32_t)r64, hi = (uint32_t)(r64 >> 32);
      const int64_t f = lo & 0x3fffffffu;
      const int s = (int)(lo >> 30);
      const int pos1 = (int)(hi & 0xff), pos2 = (int)((hi >> 8) & 0xff);
      const int pins = (int)((hi >> 16) & 7);
      const int v0 = a.faces[3 * f], v1 = a.faces[3 * f + 1], v2 = a.faces[3 * f + 2];
      double X[3][2], U[3][2];
      const int vv[3] = {v0, v1, v2};
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          X[q][c] = a.x[(int64_t)vv[q] * 2 + c];
          if constexpr (MODE == MODE_HVP) U[q][c] = ((pins >> q) & 1) ? 0.0 : a.w[(int64_t)vv[q] * 2 + c];
          else U[q][c] = 0.0;
        }
      const double* R = R_all + 4 * f;
      const double R0 = R[0], R1 = R[1], R2 = R[2], R3 = R[3];
      const double area = A_all[f];
      // J = [d1 d2] R, entries (c,k) -> 2c + k
      double J[4];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double d1 = X[1][c] - X[0][c], d2 = X[2][c] - X[0][c];
        J[2 * c] = d1 * R0 + d2 * R2;
        J[2 * c + 1] = d1 * R1 + d2 * R3;
      }
      // weights W[k][q]: vertex q's coefficient on J[., k]
      const double W[2][3] = {{-(R0 + R2), R0, R2}, {-(R1 + R3), R1, R3}};
      if constexpr (MODE == MODE_GRAD) {
        Dg<4> j[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          j[q].v = J[q];
#pragma unroll
          for (int b = 0; b < 4; ++b) j[q].g[b] = q == b ? 1.0 : 0.0;
        }
        auto det = positive_guard(j[0] * j[3] - j[1] * j[2]);
        auto fro = j[0] * j[0] + 0.0;
        fro = j[1] * j[1] + fro;
        fro = j[2] * j[2] + fro;
        fro = j[3] * j[3] + fro;
        auto E = (fro + fro / (det * det)) * area;
        ok &= isfinite(E.v + E.g[0] + E.g[1] + E.g[2] + E.g[3]);
        if (s == 0) eacc += E.v;
#pragma unroll
        for (int c = 0; c < 2; ++c) vec[c] += W[0][s] * E.g[2 * c] + W[1][s] * E.g[2 * c + 1];
        return;
      } else {
        const auto E = dirichlet_J(J, area);
        bool fin = isfinite(E.v);
#pragma unroll
        for (int i = 0; i < 4; ++i) fin &= isfinite(E.g[i]);
#pragma unroll
        for (int i = 0; i < 10; ++i) fin &= isfinite(E.h[i]);
        if constexpr (PSD) fin &= pins == 0;  // the reference clamps the pinned-masked block: exact path
        ok &= fin;
        if (MODE == MODE_HESS && s == 0) eacc += E.v;
        if constexpr (MODE == MODE_HESS) {
#pragma unroll
          for (int c = 0; c < 2; ++c) vec[c] += W[0][s] * E.g[2 * c] + W[1][s] * E.g[2 * c + 1];
        }
        // block(s, t)[c][c'] of the (possibly clamped) 6x6 Hessian
        double P[4][4];  // PSD: clamped M; otherwise H_J (full 4x4)
        double Lw[2][2];
        if constexpr (PSD) {
          // Q_W columns u1 = (1,-1,0)/sqrt2, u2 = (1,1,-2)/sqrt6; L_W = W Q_W
          const double Q[3][2] = {{INV_SQRT2, INV_SQRT6}, {-INV_SQRT2, INV_SQRT6}, {0.0, -2.0 * INV_SQRT6}};
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int b = 0; b < 2; ++b) Lw[k][b] = W[k][0] * Q[0][b] + W[k][1] * Q[1][b] + W[k][2] * Q[2][b];
          double M[10];
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int aa = 0; aa < 2; ++aa)
#pragma unroll
              for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
                for (int bb = 0; bb < 2; ++bb) {
                  const int I = 2 * c + aa, Jx = 2 * c2 + bb;
                  if (Jx > I) continue;
                  double acc = 0.0;
#pragma unroll
                  for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) acc += Lw[k][aa] * E.h[tri(2 * c + k, 2 * c2 + k2)] * Lw[k2][bb];
                  M[tri(I, Jx)] = acc;
                }
          project_if_needed<4>(M, a.floor);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) P[i][j] = M[tri(i, j)];
          // block(s,t)[c][c'] = sum_{a,b} Q[s][a] Q[t][b] P[(c,a),(c',b)] + f delta_cc' / 3,
          // evaluated as 0.5 (X(s,t,c,c') + X(t,s,c',c)) so the row kernel's
          // (r,j) and (j,r) blocks are bitwise transposes
          auto X = [&](int s_, int t_, int c, int c2) {
            double acc = 0.0;
#pragma unroll
            for (int aa = 0; aa < 2; ++aa)
#pragma unroll
              for (int bb = 0; bb < 2; ++bb) acc += Q[s_][aa] * Q[t_][bb] * P[2 * c + aa][2 * c2 + bb];
            return acc;
          };
          auto blk = [&](int t, double* out) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int c2 = 0; c2 < 2; ++c2)
                out[2 * c + c2] = 0.5 * (X(s, t, c, c2) + X(t, s, c2, c)) + (c == c2 ? a.floor * (1.0 / 3.0) : 0.0);
          };
          if constexpr (MODE == MODE_HESS) {
            double b[4];
            blk(s, b);
            dg[0] += b[0];
            dg[1] += b[1];
            dg[2] += b[3];
            if (pos1 != 255) {
              blk((s + 1) % 3, b);
              double* dst = hrow + pos1 * NN;
#pragma unroll
              for (int k = 0; k < 4; ++k) dst[k] += b[k];
            }
            if (pos2 != 255) {
              blk((s + 2) % 3, b);
              double* dst = hrow + pos2 * NN;
#pragma unroll
              for (int k = 0; k < 4; ++k) dst[k] += b[k];
            }
          } else {  // HVP with clamp: y_s = sum_t block(s,t) u_t
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              double b[4];
              blk(t, b);
#pragma unroll
              for (int c = 0; c < 2; ++c) vec[c] += b[2 * c] * U[t][0] + b[2 * c + 1] * U[t][1];
            }
          }
        } else {
          // unclamped: block(s,t)[c][c'] = sum_{k,k'} W[k][s] W[k'][t] H_J[(c,k),(c',k')],
          // symmetrised like the reference's 0.5 (h + h^T) (problem.py:466), which
          // also makes the (r,j) and (j,r) blocks bitwise transposes
          auto X = [&](int s_, int t_, int c, int c2) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
              for (int k2 = 0; k2 < 2; ++k2) acc += W[k][s_] * W[k2][t_] * E.h[tri(2 * c + k, 2 * c2 + k2)];
            return acc;
          };
          auto blk = [&](int t, double* out) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int c2 = 0; c2 < 2; ++c2) out[2 * c + c2] = 0.5 * (X(s, t, c, c2) + X(t, s, c2, c));
          };
          if constexpr (MODE == MODE_HESS) {
            double b[4];
            blk(s, b);
            dg[0] += b[0];
            dg[1] += b[1];
            dg[2] += b[3];
            if (pos1 != 255) {
              blk((s + 1) % 3, b);
              double* dst = hrow + pos1 * NN;
#pragma unroll
              for (int k = 0; k < 4; ++k) dst[k] += b[k];
            }
            if (pos2 != 255) {
              blk((s + 2) % 3, b);
              double* dst = hrow + pos2 * NN;
#pragma unroll
              for (int k = 0; k < 4; ++k) dst[k] += b[k];
            }
          } else {  // HVP: y_s = B_s^T H_J (B u)
            double bu[4];
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int k = 0; k < 2; ++k) bu[2 * c + k] = W[k][0] * U[0][c] + W[k][1] * U[1][c] + W[k][2] * U[2][c];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              double acc = 0.0;
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                double hb = 0.0;
#pragma unroll
                for (int jx = 0; jx < 4; ++jx) hb += E.h[tri(2 * c + k, jx)] * bu[jx];
                acc += W[k][s] * hb;
              }
              vec[c] += acc;
            }
          }
        }
      }
    };
    const int ne = cnt < KF ? cnt : KF;
#pragma unroll
    for (int j = 0; j < KF; ++j)
      if (j < ne) incidence(rc[j]);
    for (int k = KF; k < cnt; ++k) incidence(a.rrec[a.rinc_off[row] + k]);
    double* vout = MODE == MODE_HVP ? a.y : a.grad;
#pragma unroll
    for (int i = 0; i < N; ++i) vout[(int64_t)g * N + i] = fr ? vec[i] : 0.0;
    if constexpr (MODE == MODE_HESS) {
      if (fr && dp != 255) {
        double* dst = hrow + dp * NN;
        dst[0] = dg[0];
        dst[1] = dg[1];
        dst[2] = dg[1];
        dst[3] = dg[2];
      }
      if (nblk > 0) {
        fence_proxy_async_smem();
        row_store_bulk(a.hess + ro * NN, hrow, nblk * NN);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (!ok) *a.redo = 1;
  if constexpr (MODE != MODE_HVP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(0xffffffffu, eacc, o);
    if ((threadIdx.x & 31) == 0) a.partials[row >> 5] = eacc;
  }
  if constexpr (MODE == MODE_HESS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int MODE, bool PSD>
void launch_fv(const Problem& p, const FvArgs& a, int hd_max, cudaStream_t st) {
  const size_t sm = MODE == MODE_HESS ? (size_t)hd_max * 8 + 16 : 0;
  if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "row block does not fit in shared memory");
  const int64_t nb = (a.V + PT - 1) / PT;
  if (!nb) return;
  auto kern = k_rows_dirichlet<MODE, PSD>;
  if (sm) MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  timing_begin(p, st);
  kern<<<(unsigned)nb, PT, sm, st>>>(a);
  MG_LAUNCH_CHECK();
  timing_end(p, st);
}

}  // namespace

int64_t launch_patch_fv(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  const Mesh& m = *p.mesh;
  FvArgs a;
  a.V = m.Vr;
  a.order = m.patches.order.p;
  a.rmeta = p.rmeta.p;
  a.ell = p.ell.p;
  a.rinc_off = p.rinc_off.p;
  a.rrec = p.rrec.p;
  a.prow_ro = p.prow_ro.p;
  a.hoff = p.hoff.p;
  a.faces = m.faces.p;
  a.x = c.x;
  a.w = c.w;
  a.grad = c.grad;
  a.hess = c.hess;
  a.y = c.y;
  a.partials = c.partials + partial_offset;
  a.redo = p.redo.p;
  a.floor = c.floor;
  a.t = p.terms[0].dev;
  const int hd = mode == MODE_HESS ? p.max_patch_hdoubles : 0;
  switch (mode) {
    case MODE_GRAD: launch_fv<MODE_GRAD, false>(p, a, hd, c.stream); break;
    case MODE_HESS:
      if (c.psd) launch_fv<MODE_HESS, true>(p, a, hd, c.stream);
      else launch_fv<MODE_HESS, false>(p, a, hd, c.stream);
      break;
    case MODE_HVP:
      if (c.psd) launch_fv<MODE_HVP, true>(p, a, hd, c.stream);
      else launch_fv<MODE_HVP, false>(p, a, hd, c.stream);
      break;
    default: throw Error(MG_ERR_UNSUPPORTED, "face row kernel assembles grad / Hessian / HVP only");
  }
  return mode == MODE_HVP ? 0 : (m.Vr + 31) / 32;
}

}  // namespace mg
