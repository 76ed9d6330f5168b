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
#include "stage.cuh"

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
  const uint64_t* ellv;      // (KF, V) the incidence's other two corners (s+1, s+2)
  int64_t es;                // slot stride of ell / ellv (V padded to whole row blocks)
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
  double* vscr;              // sphere: per-vertex retraction (p, pdot), (V, 6)
  int64_t nv;                // vertices of the (shard) mesh
  double* fpsd;              // PSD clamp: per face P_f(M), packed 4x4 (F, 10)
  double* fpsd6;             // faces with a pinned corner: the clamped masked 6x6, packed (F, 21)
  const uint8_t* fixed;      // (nv) pinned vertices, or null
  int64_t nf;                // faces of the (shard) mesh
  // CTA face lists (k_cta_dirichlet): per 64-row block its distinct incident
  // faces (face | corner-0-row-in-block << 31), and per incidence the face's
  // slot in its block's list (ELL slot-major for the first KF, then CSR)
  const int32_t* cf_off;     // (blocks + 1)
  const int4* cf_face;       // {face | own0 << 31, corner 0, 1, 2}
  const uint16_t* eslot;     // (KF, V) slot | corner << 14
  const uint16_t* rslot;     // (incidences) parallel to rrec, same packing
  int cf_max;                // max faces of one block (shared-memory records)
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

MG_DI double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
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

// Closed form of the same function and its J-derivatives (F = |J|^2, D = det J,
// cof = dD/dJ, C2 = d2D/dJ2):
//   g = 2a [(1 + D^-2) J - F D^-3 cof]
//   H = 2a [(1 + D^-2) I - 2 D^-3 (J cof^T + cof J^T) + 3 F D^-4 cof cof^T - F D^-3 C2]
// Returns false unless D > 0 and all values are finite (positive_guard NaNs the
// reference's value there; the exact kernel then reproduces its NaN pattern).
template <bool HESS>
MG_DI bool dirichlet_closed(const double* J, double area, double& val, double* g, double* h) {
  const double F = J[0] * J[0] + J[1] * J[1] + J[2] * J[2] + J[3] * J[3];
  const double D = J[0] * J[3] - J[1] * J[2];
  const double iD = rcp_fast(D), q = iD * iD, r = q * iD;
  const double cof[4] = {J[3], -J[2], -J[1], J[0]};
  val = (F + F * q) * area;
  const double a2 = 2.0 * area, s1 = 1.0 + q, sF = F * r;
#pragma unroll
  for (int i = 0; i < 4; ++i) g[i] = a2 * (s1 * J[i] - sF * cof[i]);
  double chk = val + g[0] + g[1] + g[2] + g[3];
  if constexpr (HESS) {
    const double t2 = 2.0 * r, t3 = 3.0 * F * q * q;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        double v = -t2 * (J[i] * cof[j] + cof[i] * J[j]) + t3 * cof[i] * cof[j];
        if (i == j) v += s1;
        if ((i == 3 && j == 0)) v -= sF;   // C2[0][3] = 1
        if ((i == 2 && j == 1)) v += sF;   // C2[1][2] = -1
        h[tri(i, j)] = a2 * v;
        chk += h[tri(i, j)];
      }
  }
  return D > 0.0 && isfinite(chk);
}

// The reduced PSD clamp of one face (see the header): M = (I (x) L_W)^T H_J
// (I (x) L_W), then P_f(M) in place — Cholesky test, else the certified
// rank-one update from the twist direction, else round-robin Jacobi.
// Non-finite faces (fin false) are left unclamped (the caller raises redo).
MG_DI void face_psd_reduce(const double* J, double R0, double R1, double R2, double R3, const double* h,
                           double floor_, bool fin, double* M) {
  const double Wa0 = -(R0 + R2), Wa1 = -(R1 + R3);
  // Q_W rows (corners): (1/sqrt2, 1/sqrt6), (-1/sqrt2, 1/sqrt6), (0, -2/sqrt6); L_W = W Q_W
  const double Lw00 = (Wa0 - R0) * INV_SQRT2, Lw01 = (Wa0 + R0 - 2.0 * R2) * INV_SQRT6;
  const double Lw10 = (Wa1 - R1) * INV_SQRT2, Lw11 = (Wa1 + R1 - 2.0 * R3) * INV_SQRT6;
  const double Lw[2][2] = {{Lw00, Lw01}, {Lw10, Lw11}};
#pragma unroll
  for (int I = 0; I < 4; ++I)
#pragma unroll
    for (int Jx = 0; Jx <= I; ++Jx) {
      const int c = I >> 1, aa = I & 1, c2 = Jx >> 1, bb = Jx & 1;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) acc += Lw[k][aa] * h[tri(2 * c + k, 2 * c2 + k2)] * Lw[k2][bb];
      M[tri(I, Jx)] = acc;
    }
  // non-finite faces: the row kernel takes the exact path
  if (fin && !shifted_pd<4>(M, floor_)) {
    // only the twist mode of the isotropic energy can be negative: start the
    // eigen-iteration from J's twist direction [[q, -p], [p, q]] (p = tr-like,
    // q = skew part of J) mapped through the reduced basis (M = C^T H_J C,
    // C = I (x) L_W: v0 = C^-1 u_T)
    const double p = J[0] + J[3], q = J[1] - J[2];
    const double uT[4] = {q, -p, p, q};
    const double dl = Lw00 * Lw11 - Lw01 * Lw10;
    double v0[4];
    if (dl != 0.0) {
      const double idl = 1.0 / dl;
#pragma unroll
      for (int c = 0; c < 2; ++c) {  // solve sum_a Lw[k][a] y_a = uT[2c+k]
        const double u0 = uT[2 * c], u1 = uT[2 * c + 1];
        v0[2 * c] = (Lw11 * u0 - Lw01 * u1) * idl;
        v0[2 * c + 1] = (-Lw10 * u0 + Lw00 * u1) * idl;
      }
    }
    if (dl == 0.0 || !psd_rank1_update<4>(M, floor_, v0)) jacobi_project_rr<4>(M, floor_);
  }
}

// Per-face PSD clamp of the reduced 4x4 matrix M = (I (x) L_W)^T H_J (I (x) L_W)
// (see the header), once per face: the three owner rows of a face then read
// P_f(M) instead of each recomputing the eigen-decomposition.
__global__ void __launch_bounds__(128) k_face_psd(const __grid_constant__ FvArgs a) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= a.nf) return;
  const int v0 = a.faces[3 * f], v1 = a.faces[3 * f + 1], v2 = a.faces[3 * f + 2];
  double X[3][2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    X[0][c] = a.x[(int64_t)v0 * 2 + c];
    X[1][c] = a.x[(int64_t)v1 * 2 + c];
    X[2][c] = a.x[(int64_t)v2 * 2 + c];
  }
  const double* Rp = a.t.a[0] + 4 * f;
  const double R0 = Rp[0], R1 = Rp[1], R2 = Rp[2], R3 = Rp[3];
  const double area = a.t.a[1][f];
  double J[4];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double d1 = X[1][c] - X[0][c], d2 = X[2][c] - X[0][c];
    J[2 * c] = d1 * R0 + d2 * R2;
    J[2 * c + 1] = d1 * R1 + d2 * R3;
  }
  double v, g[4], h[10];
  const bool fin = dirichlet_closed<true>(J, area, v, g, h);
  double M[10];
  face_psd_reduce(J, R0, R1, R2, R3, h, a.floor, fin, M);
  double2* out = reinterpret_cast<double2*>(a.fpsd + f * 10);
#pragma unroll
  for (int k = 0; k < 5; ++k) out[k] = make_double2(M[2 * k], M[2 * k + 1]);
}

// Faces with a pinned corner under a clamp: the masked 6x6 (pinned corners'
// rows / columns zero), clamped in full, packed (rows 2q + c).
MG_DI void face_psd6(double R0, double R1, double R2, double R3, const double* h, const bool* pq, double floor_,
                     bool fin, double* H6) {
  const double W[3][2] = {{-(R0 + R2), -(R1 + R3)}, {R0, R1}, {R2, R3}};
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int q2 = 0; q2 <= q; ++q2)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          const int R = 2 * q + c, C = 2 * q2 + c2;
          if (C > R) continue;
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int k2 = 0; k2 < 2; ++k2) acc += W[q][k] * h[tri(2 * c + k, 2 * c2 + k2)] * W[q2][k2];
          H6[tri(R, C)] = (pq[q] || pq[q2]) ? 0.0 : acc;
        }
  if (fin) project_if_needed<6>(H6, floor_);  // non-finite faces: the row kernel takes the exact path
}

// Faces with a pinned corner under a clamp (launched only when the problem
// has pinned vertices): the reference clamps the masked 6x6 (pinned corners'
// rows / columns zero, problem.py:420-438 + active.py:490-504), which has no
// translation symmetry left to reduce by, so the full block (packed, rows
// 2q + c) is clamped and stored for the row kernel.
__global__ void __launch_bounds__(128) k_face_psd_pinned(const __grid_constant__ FvArgs a) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= a.nf) return;
  const int v0 = a.faces[3 * f], v1 = a.faces[3 * f + 1], v2 = a.faces[3 * f + 2];
  const bool p0 = a.fixed[v0], p1 = a.fixed[v1], p2 = a.fixed[v2];
  if (!(p0 || p1 || p2)) return;
  double X[3][2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    X[0][c] = a.x[(int64_t)v0 * 2 + c];
    X[1][c] = a.x[(int64_t)v1 * 2 + c];
    X[2][c] = a.x[(int64_t)v2 * 2 + c];
  }
  const double* Rp = a.t.a[0] + 4 * f;
  const double R0 = Rp[0], R1 = Rp[1], R2 = Rp[2], R3 = Rp[3];
  const double area = a.t.a[1][f];
  double J[4];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double d1 = X[1][c] - X[0][c], d2 = X[2][c] - X[0][c];
    J[2 * c] = d1 * R0 + d2 * R2;
    J[2 * c + 1] = d1 * R1 + d2 * R3;
  }
  double v, g[4], h[10];
  const bool fin = dirichlet_closed<true>(J, area, v, g, h);
  const bool pq[3] = {p0, p1, p2};
  double H6[21];
  face_psd6(R0, R1, R2, R3, h, pq, a.floor, fin, H6);
#pragma unroll
  for (int k = 0; k < 21; ++k) a.fpsd6[f * 21 + k] = H6[k];
}

// H_J V of the same function without forming H_J (the HVP's directional
// derivative of the closed-form gradient along V):
//   dF = 2 J.V, dD = cof.V,
//   H_J V = 2a [(1 + D^-2) V - 2 D^-3 dD J - (dF D^-3 - 3 F D^-4 dD) cof - F D^-3 cof(V)]
// Returns false unless D > 0 and the result is finite.
MG_DI bool dirichlet_hv_closed(const double* J, const double* V, double area, double* out) {
  const double F = J[0] * J[0] + J[1] * J[1] + J[2] * J[2] + J[3] * J[3];
  const double D = J[0] * J[3] - J[1] * J[2];
  const double iD = rcp_fast(D), q = iD * iD, r = q * iD;
  const double cof[4] = {J[3], -J[2], -J[1], J[0]};
  const double cofV[4] = {V[3], -V[2], -V[1], V[0]};
  const double dF = 2.0 * (J[0] * V[0] + J[1] * V[1] + J[2] * V[2] + J[3] * V[3]);
  const double dD = cof[0] * V[0] + cof[1] * V[1] + cof[2] * V[2] + cof[3] * V[3];
  const double a2 = 2.0 * area, s1 = 1.0 + q, tJ = 2.0 * r * dD, tc = dF * r - 3.0 * F * q * q * dD, tv = F * r;
  double chk = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[i] = a2 * (s1 * V[i] - tJ * J[i] - tc * cof[i] - tv * cofV[i]);
    chk += out[i];
  }
  return D > 0.0 && isfinite(chk);
}

#ifndef FV_MINB
#define FV_MINB 6
#endif
#ifndef FV_STAGES
#define FV_STAGES 1  // staged level-1 ring of the per-row face kernels (1: Dirichlet grad+H 1.934 -> 1.893 ms vs 2)
#endif
// CTAs per SM to fit: the clamped Hessian path carries the per-face P_f(M)
// of two incidences in flight and gets more registers
template <int MODE, bool PSD> struct FvMinb {
  static constexpr int v = (PSD && MODE == MODE_HESS) ? 4 : FV_MINB;
};
template <int MODE, bool PSD, bool PIN = false>
__global__ void __launch_bounds__(PT, FvMinb<MODE, PSD>::v) k_rows_dirichlet(const __grid_constant__ FvArgs a) {
  constexpr int N = 2, NN = 4;
  extern __shared__ __align__(16) double hbuf[];
  bool ok = true;
  // Persistent CTAs walk row blocks grid-stride; each block's level-1 streams
  // (ELL records and other-corner records, meta words, row order, row starts,
  // row-buffer offsets) arrive by TMA FV_STAGES blocks ahead (stage.cuh)
  constexpr bool HS = MODE == MODE_HESS;
  constexpr int S_RC = 0, S_OV = KF * PT * 8, S_ME = 2 * KF * PT * 8, S_OR = S_ME + PT * 4, S_RO = S_OR + PT * 4,
                S_HO = S_RO + PT * 8, S_BYTES = HS ? S_HO + PT * 4 : S_RO;
  __shared__ __align__(128) unsigned char stg[FV_STAGES][S_BYTES];
  __shared__ __align__(8) uint64_t sbar[FV_STAGES];
  const int64_t nblocks = (a.V + PT - 1) / PT;
  auto stage_issue = [&](int st, int64_t b) {  // one thread
    mbar_expect_tx(&sbar[st], 2 * KF * PT * 8 + PT * 4 + (a.order ? PT * 4 : 0) + (HS ? PT * 12 : 0));
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      bulk_g2s(stg[st] + S_RC + j * PT * 8, a.ell + (int64_t)j * a.es + b * PT, PT * 8, &sbar[st]);
      bulk_g2s(stg[st] + S_OV + j * PT * 8, a.ellv + (int64_t)j * a.es + b * PT, PT * 8, &sbar[st]);
    }
    bulk_g2s(stg[st] + S_ME, a.rmeta + b * PT, PT * 4, &sbar[st]);
    if (a.order) bulk_g2s(stg[st] + S_OR, a.order + b * PT, PT * 4, &sbar[st]);
    if constexpr (HS) {
      bulk_g2s(stg[st] + S_RO, a.prow_ro + b * PT, PT * 8, &sbar[st]);
      bulk_g2s(stg[st] + S_HO, a.hoff + b * PT, PT * 4, &sbar[st]);
    }
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < FV_STAGES; ++st) mbar_init(&sbar[st], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int st = 0; st < FV_STAGES; ++st)
      if (blockIdx.x + (int64_t)st * gridDim.x < nblocks) stage_issue(st, blockIdx.x + (int64_t)st * gridDim.x);
  int it = 0;
  for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x, ++it) {
  const int64_t row = blk * PT + threadIdx.x;
  double eacc = 0.0;
  const int stn = it % FV_STAGES;
  mbar_wait(&sbar[stn], (uint32_t)(it / FV_STAGES) & 1u);
  const unsigned char* sp = stg[stn];
  const int g = a.order ? reinterpret_cast<const int32_t*>(sp + S_OR)[threadIdx.x] : (int)row;
  const uint32_t meta = reinterpret_cast<const uint32_t*>(sp + S_ME)[threadIdx.x];
  int64_t ro = 0;
  int ho = 0;
  if constexpr (HS) {
    ro = reinterpret_cast<const int64_t*>(sp + S_RO)[threadIdx.x];
    ho = reinterpret_cast<const int32_t*>(sp + S_HO)[threadIdx.x];
  }
  uint64_t rc[KF], ov[KF];
#pragma unroll
  for (int j = 0; j < KF; ++j) {
    rc[j] = reinterpret_cast<const uint64_t*>(sp + S_RC)[j * PT + threadIdx.x];
    ov[j] = reinterpret_cast<const uint64_t*>(sp + S_OV)[j * PT + threadIdx.x];
  }
  __syncthreads();  // every thread has read the stage: refill it
  if (threadIdx.x == 0 && blk + (int64_t)FV_STAGES * gridDim.x < nblocks) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    stage_issue(stn, blk + (int64_t)FV_STAGES * gridDim.x);
  }
  // the previous block's bulk row stores must have read the row buffers
  if constexpr (HS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  if (row < a.V) {
    const bool fr = !((meta >> 8) & 1);
    const int dp = (int)(meta >> 16) & 0xff;
    const int cnt = (meta & 0xff) < 255 ? (int)(meta & 0xff) : a.rinc_off[row + 1] - a.rinc_off[row];
    double* hrow = hbuf + ho;
    int nblk = 0;
    // fan rows (incidences in rotation order around the vertex, setup): each
    // off-diagonal block's two face contributions meet in registers and the
    // block is written once; other rows accumulate in the cleared row buffer
    const bool fan = (meta >> 9) & 1;
    double carry[4] = {0.0, 0.0, 0.0, 0.0}, first[4] = {0.0, 0.0, 0.0, 0.0};
    int first_pos = 255, last_pos2 = 255;
    if constexpr (MODE == MODE_HESS) {
      nblk = (int)(((meta >> 24) & 0xff));
      if (!fan)
        for (int k = 0; k < nblk * NN; ++k) hrow[k] = 0.0;
    }
    double vec[N] = {0.0, 0.0}, dg[3] = {0.0, 0.0, 0.0};
    const double* R_all = a.t.a[0];
    const double* A_all = a.t.a[1];
    // one incidence: face f (record), its corners' x (and w), rest_inv, area
    struct FaceIn {
      double X[3][2], U[3][2], R[4], area;
      double M[PSD ? 10 : 1];
    };
    auto load_face = [&](uint64_t r64, const int* v) {
      FaceIn d;
      const int64_t f = (uint32_t)r64 & 0x3fffffffu;
      const int pins = (int)((r64 >> 48) & 7);
      if constexpr (PSD) {
        const double2* m2 = reinterpret_cast<const double2*>(a.fpsd + f * 10);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double2 t = m2[k];
          d.M[2 * k] = t.x;
          d.M[2 * k + 1] = t.y;
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          d.X[q][c] = a.x[(int64_t)v[q] * 2 + c];
          if constexpr (MODE == MODE_HVP) d.U[q][c] = ((pins >> q) & 1) ? 0.0 : a.w[(int64_t)v[q] * 2 + c];
          else d.U[q][c] = 0.0;
        }
#pragma unroll
      for (int k = 0; k < 4; ++k) d.R[k] = R_all[4 * f + k];
      d.area = A_all[f];
      return d;
    };
    auto sel3 = [](int i, double p0, double p1, double p2) { return i == 0 ? p0 : (i == 1 ? p1 : p2); };
    auto incidence = [&](uint64_t r64, const FaceIn& d, int jidx) {
      const uint32_t lo = (uint32_t)r64, hi = (uint32_t)(r64 >> 32);
      const int s = (int)(lo >> 30);
      const int pos1 = (int)(hi & 0xff), pos2 = (int)((hi >> 8) & 0xff);
      const int pins = (int)((hi >> 16) & 7);
      const double R0 = d.R[0], R1 = d.R[1], R2 = d.R[2], R3 = d.R[3];
      // J = [d1 d2] R, entries (c,k) -> 2c + k
      double J[4];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double d1 = d.X[1][c] - d.X[0][c], d2 = d.X[2][c] - d.X[0][c];
        J[2 * c] = d1 * R0 + d2 * R2;
        J[2 * c + 1] = d1 * R1 + d2 * R3;
      }
      // weights of corner q on J[., k]: W[k] = (-(R0k + R1k), R0k, R1k); the
      // row's corner s and the next two, selected into registers
      const double Wa0 = -(R0 + R2), Wa1 = -(R1 + R3);
      double ws[2], w1[2], w2[2];
      ws[0] = sel3(s, Wa0, R0, R2);
      ws[1] = sel3(s, Wa1, R1, R3);
      const int s1 = s == 2 ? 0 : s + 1, s2 = s == 0 ? 2 : s - 1;
      w1[0] = sel3(s1, Wa0, R0, R2);
      w1[1] = sel3(s1, Wa1, R1, R3);
      w2[0] = sel3(s2, Wa0, R0, R2);
      w2[1] = sel3(s2, Wa1, R1, R3);
      if constexpr (MODE == MODE_GRAD) {
        double val, gJ[4];
        ok &= dirichlet_closed<false>(J, d.area, val, gJ, nullptr);
        if (s == 0) eacc += val;
#pragma unroll
        for (int c = 0; c < 2; ++c) vec[c] += ws[0] * gJ[2 * c] + ws[1] * gJ[2 * c + 1];
      } else {
        // G[(c,k),(c2,b)]: the 4x4 matrix whose (s,t) block contraction gives the
        // 6x6 Hessian block: unclamped G = H_J with weights W; clamped G = P_f(M)
        // (k_face_psd, once per face) with weights Q_W (orthonormal basis of
        // 1-perp) plus the floor on 1 1^T / 3
        double G[4][4];
        double as[2], a1[2], a2[2];
        // faces with a pinned corner under a clamp: blocks straight from the
        // clamped masked 6x6 of the pre-pass
        // (PIN: compiled in only for problems with pinned vertices)
        const double* P6 = (PSD && PIN && pins != 0) ? a.fpsd6 + ((int64_t)((uint32_t)lo & 0x3fffffffu)) * 21 : nullptr;
        if constexpr (PSD) {
          double val, gJ[4];
          bool fin = dirichlet_closed<false>(J, d.area, val, gJ, nullptr);
          double chk = 0.0;
#pragma unroll
          for (int k = 0; k < 10; ++k) chk += d.M[k];
          if (P6) {
            chk = 0.0;
#pragma unroll
            for (int k = 0; k < 21; ++k) chk += P6[k];
          }
          ok &= fin && isfinite(chk);
          if (MODE == MODE_HESS && s == 0) eacc += val;
          if constexpr (MODE == MODE_HESS) {
#pragma unroll
            for (int c = 0; c < 2; ++c) vec[c] += ws[0] * gJ[2 * c] + ws[1] * gJ[2 * c + 1];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) G[i][j] = d.M[tri(i, j)];
          as[0] = sel3(s, INV_SQRT2, -INV_SQRT2, 0.0);
          as[1] = sel3(s, INV_SQRT6, INV_SQRT6, -2.0 * INV_SQRT6);
          a1[0] = sel3(s1, INV_SQRT2, -INV_SQRT2, 0.0);
          a1[1] = sel3(s1, INV_SQRT6, INV_SQRT6, -2.0 * INV_SQRT6);
          a2[0] = sel3(s2, INV_SQRT2, -INV_SQRT2, 0.0);
          a2[1] = sel3(s2, INV_SQRT6, INV_SQRT6, -2.0 * INV_SQRT6);
        } else if constexpr (MODE == MODE_HVP) {
          // unclamped HVP: only H_J dJ is needed (G unused below)
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            as[k] = ws[k];
            a1[k] = w1[k];
            a2[k] = w2[k];
          }
        } else {
          struct {
            double v, g[4], h[10];
          } E;
          ok &= dirichlet_closed<true>(J, d.area, E.v, E.g, E.h);
          if (MODE == MODE_HESS && s == 0) eacc += E.v;
          if constexpr (MODE == MODE_HESS) {
#pragma unroll
            for (int c = 0; c < 2; ++c) vec[c] += ws[0] * E.g[2 * c] + ws[1] * E.g[2 * c + 1];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) G[i][j] = E.h[tri(i, j)];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            as[k] = ws[k];
            a1[k] = w1[k];
            a2[k] = w2[k];
          }
        }
        const double fl3 = PSD ? a.floor * (1.0 / 3.0) : 0.0;
        // block(u,v)[c][c2] = 0.5 (X(u,v,c,c2) + X(v,u,c2,c)), X = sum_{k,k2} u[k] v[k2] G[(c,k),(c2,k2)]:
        // the reference's symmetrisation, and the (r,j) / (j,r) blocks come out bitwise transposed
        auto X = [&](const double* u, const double* v, int c, int c2) {
          return u[0] * (G[2 * c][2 * c2] * v[0] + G[2 * c][2 * c2 + 1] * v[1]) +
                 u[1] * (G[2 * c + 1][2 * c2] * v[0] + G[2 * c + 1][2 * c2 + 1] * v[1]);
        };
        auto blk = [&](const double* u, const double* v, bool diag, double* out) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2)
              out[2 * c + c2] = 0.5 * (X(u, v, c, c2) + X(v, u, c2, c)) + (diag && c == c2 ? fl3 : 0.0) +
                                (!diag && c == c2 ? fl3 : 0.0);
        };
        // off-diagonal block (s, t) evaluated once in the canonical slot order:
        // the row at the lower slot computes X(w_lo, w_hi), the other row the
        // same expression transposed — the two blocks come out bitwise
        // transposed with half the work of the averaged form
        auto blk_pair = [&](int st, const double* wt, double* out) {
          const bool lo = s < st;
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2)
              out[2 * c + c2] = (lo ? X(as, wt, c, c2) : X(wt, as, c2, c)) + (c == c2 ? fl3 : 0.0);
        };
        // block (s, t) of the pinned face's clamped 6x6
        auto p6blk = [&](int t, double* out) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) out[2 * c + c2] = P6[tri(2 * s + c, 2 * t + c2)];
        };
        if constexpr (MODE == MODE_HESS) {
          double b[4];
          if (P6) p6blk(s, b);
          else blk(as, as, true, b);
          dg[0] += b[0];
          dg[1] += b[1];
          dg[2] += b[3];
          if (fan) {
            // face j's first other corner is face j-1's second: finish that block
            double b1[4], b2[4];
            if (P6) {
              p6blk(s1, b1);
              p6blk(s2, b2);
            } else {
              blk_pair(s1, a1, b1);
              blk_pair(s2, a2, b2);
            }
            if (jidx == 0) {
#pragma unroll
              for (int k = 0; k < 4; ++k) first[k] = b1[k];
              first_pos = pos1;
            } else if (pos1 != 255) {
              double* dst = hrow + pos1 * NN;
#pragma unroll
              for (int k = 0; k < 4; ++k) dst[k] = carry[k] + b1[k];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) carry[k] = b2[k];
            last_pos2 = pos2;
          } else {
            if (pos1 != 255) {
              if (P6) p6blk(s1, b);
              else blk_pair(s1, a1, b);
              double* dst = hrow + pos1 * NN;
#pragma unroll
              for (int k = 0; k < 4; ++k) dst[k] += b[k];
            }
            if (pos2 != 255) {
              if (P6) p6blk(s2, b);
              else blk_pair(s2, a2, b);
              double* dst = hrow + pos2 * NN;
#pragma unroll
              for (int k = 0; k < 4; ++k) dst[k] += b[k];
            }
          }
        } else {
          // HVP: y_s = sum_t block(s,t) u_t = (I (x) w_s)^T G dJ with dJ = sum_t (w_t (x) u_t)
          // the face's masked direction in J space (the blocks' symmetrisation is
          // exact here: G is symmetric), plus the floor term f/3 sum_t u_t under a clamp
          double wq[3][2];
          if constexpr (PSD) {
            wq[0][0] = INV_SQRT2; wq[0][1] = INV_SQRT6;
            wq[1][0] = -INV_SQRT2; wq[1][1] = INV_SQRT6;
            wq[2][0] = 0.0; wq[2][1] = -2.0 * INV_SQRT6;
          } else {
            wq[0][0] = -(d.R[0] + d.R[2]); wq[0][1] = -(d.R[1] + d.R[3]);
            wq[1][0] = d.R[0]; wq[1][1] = d.R[1];
            wq[2][0] = d.R[2]; wq[2][1] = d.R[3];
          }
          double dv[4];
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int k = 0; k < 2; ++k)
              dv[2 * c + k] = wq[0][k] * d.U[0][c] + wq[1][k] * d.U[1][c] + wq[2][k] * d.U[2][c];
          double gv[4];
          if constexpr (PSD) {
#pragma unroll
            for (int i = 0; i < 4; ++i) gv[i] = G[i][0] * dv[0] + G[i][1] * dv[1] + G[i][2] * dv[2] + G[i][3] * dv[3];
          } else {
            ok &= dirichlet_hv_closed(J, dv, d.area, gv);
          }
          if (P6) {  // y_s = sum_t P6(s, t) u_t (u masked)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              double y = 0.0;
#pragma unroll
              for (int t = 0; t < 3; ++t)
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2) y += P6[tri(2 * s + c, 2 * t + c2)] * d.U[t][c2];
              vec[c] += y;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              double y = as[0] * gv[2 * c] + as[1] * gv[2 * c + 1];
              if constexpr (PSD) y += fl3 * (d.U[0][c] + d.U[1][c] + d.U[2][c]);
              vec[c] += y;
            }
          }
        }
      }
    };
    // face corner ids of the ELL incidences (one batched level), then the
    // corners' data streamed one incidence ahead of the compute
    // (the other two corners come from the ELL other-corner records, so no
    // dependent faces[] lookup; the row's own vertex is corner s)
    const int ne = cnt < KF ? cnt : KF;
    int fv[KF][3];
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      const int s = (int)((uint32_t)rc[j] >> 30);
      const int o1 = (int)(uint32_t)ov[j], o2 = (int)(ov[j] >> 32);
      fv[j][0] = s == 0 ? g : (s == 1 ? o2 : o1);
      fv[j][1] = s == 0 ? o1 : (s == 1 ? g : o2);
      fv[j][2] = s == 0 ? o2 : (s == 1 ? o1 : g);
    }
    FaceIn cur;
    if (ne > 0) cur = load_face(rc[0], fv[0]);
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      if (j < ne) {
        FaceIn nxt;
        if (j + 1 < ne) nxt = load_face(rc[j + 1], fv[j + 1]);
        incidence(rc[j], cur, j);
        cur = nxt;
      }
    }
    for (int k = KF; k < cnt; ++k) {
      const uint64_t r64 = a.rrec[a.rinc_off[row] + k];
      const int64_t f = (uint32_t)r64 & 0x3fffffffu;
      const int v3[3] = {a.faces[3 * f], a.faces[3 * f + 1], a.faces[3 * f + 2]};
      incidence(r64, load_face(r64, v3), k);
    }
    if constexpr (MODE == MODE_HESS) {
      if (fan && cnt > 0) {  // close the fan: the first block meets the last carry, or both stand alone
        if (last_pos2 == first_pos) {
          if (first_pos != 255) {
            double* dst = hrow + first_pos * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = carry[k] + first[k];
          }
        } else {
          if (first_pos != 255) {
            double* dst = hrow + first_pos * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = first[k];
          }
          if (last_pos2 != 255) {
            double* dst = hrow + last_pos2 * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = carry[k];
          }
        }
      }
    }
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
  if constexpr (MODE != MODE_HVP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(0xffffffffu, eacc, o);
    if ((threadIdx.x & 31) == 0) a.partials[row >> 5] = eacc;
  }
  }  // row blocks
  if (!ok) *a.redo = 1;
  if constexpr (MODE == MODE_HESS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// CTA face-list variant (default): each face is evaluated ONCE per 64-row
// block instead of once per owner row. Phase A: the block's threads walk its
// distinct incident faces (setup: cf_off / cf_face; Morton rows put ~177
// faces behind 64 rows, against 384 row incidences) and write per corner q
// what its row needs into a shared-memory record: the gradient (HVP: H u)
// part, and for the Hessian the diagonal block (3 unique entries) and the
// off-diagonal block (q, q+1 mod 3) (its transpose is block (q+1, q), so the
// two come out bitwise transposed). The PSD clamp runs here too, once per
// face, in registers (no P_f(M) round trip through HBM). Phase B: one thread
// per row sums its incidences' records in the same fixed incidence order as
// the per-row kernel, builds its row in the shared-memory row buffer and
// streams it out with one bulk copy. The energy counts each face in the block
// that owns its first corner's row.
template <int MODE> struct CfRec { static constexpr int S = MODE == MODE_HESS ? 27 : 6; };
#ifndef CF_STAGES
#define CF_STAGES 2  // staged row blocks (face lists + row streams) in flight per CTA
#endif
#ifndef CF_PERSIST_HESS
#define CF_PERSIST_HESS 0
#endif
#ifndef CF_HESS_MINB
#define CF_HESS_MINB 4
#endif
#ifndef CF_FLAT_MINB
#define CF_FLAT_MINB 6  // HVP 0.772 -> 0.699 ms at 8 -> 6 (128 registers spilled 56 bytes); 5: 0.695, 4: 0.694
#endif
#ifndef CF_NB
#define CF_NB 3  // faces per thread with their loads in flight together (unclamped; HVP 0.866 -> 0.848 ms with MINB 8)
#endif

// one face's inputs (phase A loads them for two faces before computing)
struct CfIn {
  double X[3][2], U[3][2], R[4], area;
  bool pq[3];
};
template <int MODE, bool PSD>
MG_DI void cf_load(const FvArgs& a, const int4& fe, CfIn& d) {
  const int64_t f = (uint32_t)fe.x & 0x7fffffffu;
  const int v[3] = {fe.y, fe.z, fe.w};
#pragma unroll
  for (int q = 0; q < 3; ++q) d.pq[q] = (MODE == MODE_HVP || PSD) && a.fixed && a.fixed[v[q]];
  // (caller buffers: 8-byte alignment only, scalar loads)
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    d.X[q][0] = a.x[(int64_t)v[q] * 2];
    d.X[q][1] = a.x[(int64_t)v[q] * 2 + 1];
    if constexpr (MODE == MODE_HVP) {
      d.U[q][0] = a.w[(int64_t)v[q] * 2];
      d.U[q][1] = a.w[(int64_t)v[q] * 2 + 1];
    }
  }
  const double* Rp = a.t.a[0] + 4 * f;
#pragma unroll
  for (int k = 0; k < 4; ++k) d.R[k] = Rp[k];
  d.area = a.t.a[1][f];
}

template <int MODE, bool PSD, bool PIN>
MG_DI void cf_face(const FvArgs& a, const CfIn& d, double* out, double& val, bool& ok) {
  double X[3][2], U[3][2];
  bool pq[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    pq[q] = d.pq[q];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      X[q][c] = d.X[q][c];
      U[q][c] = (MODE == MODE_HVP && !pq[q]) ? d.U[q][c] : 0.0;
    }
  }
  const double R0 = d.R[0], R1 = d.R[1], R2 = d.R[2], R3 = d.R[3];
  const double area = d.area;
  double J[4];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double d1 = X[1][c] - X[0][c], d2 = X[2][c] - X[0][c];
    J[2 * c] = d1 * R0 + d2 * R2;
    J[2 * c + 1] = d1 * R1 + d2 * R3;
  }
  // corner weights on J's columns: J[2c + k] = sum_q W[q][k] X[q][c]
  const double W[3][2] = {{-(R0 + R2), -(R1 + R3)}, {R0, R1}, {R2, R3}};
  // Q_W (orthonormal basis of 1-perp) rows: the clamped blocks' weights
  const double QW[3][2] = {{INV_SQRT2, INV_SQRT6}, {-INV_SQRT2, INV_SQRT6}, {0.0, -2.0 * INV_SQRT6}};
  const bool pinned_face = PSD && PIN && (pq[0] || pq[1] || pq[2]);
  val = 0.0;
  if constexpr (MODE == MODE_GRAD) {
    double gJ[4];
    ok &= dirichlet_closed<false>(J, area, val, gJ, nullptr);
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c) out[2 * q + c] = W[q][0] * gJ[2 * c] + W[q][1] * gJ[2 * c + 1];
    return;
  }
  double gJ[4], h[10];
  bool fin;
  if constexpr (MODE == MODE_HESS || PSD) {
    fin = dirichlet_closed<true>(J, area, val, gJ, h);
  }
  // G (4x4, J space) and the corner weights its blocks contract with
  double G[10], M6[PIN ? 21 : 1];
  const double(*wt)[2] = W;
  const double fl3 = PSD ? a.floor * (1.0 / 3.0) : 0.0;
  if constexpr (PSD) {
    if (pinned_face) {
      if constexpr (PIN) {
        face_psd6(R0, R1, R2, R3, h, pq, a.floor, fin, M6);
        double chk = 0.0;
#pragma unroll
        for (int k = 0; k < 21; ++k) chk += M6[k];
        fin = fin && isfinite(chk);
      }
    } else {
      face_psd_reduce(J, R0, R1, R2, R3, h, a.floor, fin, G);
      double chk = 0.0;
#pragma unroll
      for (int k = 0; k < 10; ++k) chk += G[k];
      fin = fin && isfinite(chk);
    }
    wt = QW;
    ok &= fin;
  } else if constexpr (MODE == MODE_HESS) {
#pragma unroll
    for (int k = 0; k < 10; ++k) G[k] = h[k];
    ok &= fin;
  }
  // X(u, v, c, c2) = sum_{k,k2} u[k] G[(c,k),(c2,k2)] v[k2]
  auto Xf = [&](const double* u, const double* w2, int c, int c2) {
    return u[0] * (G[tri(2 * c, 2 * c2)] * w2[0] + G[tri(2 * c, 2 * c2 + 1)] * w2[1]) +
           u[1] * (G[tri(2 * c + 1, 2 * c2)] * w2[0] + G[tri(2 * c + 1, 2 * c2 + 1)] * w2[1]);
  };
  if constexpr (MODE == MODE_HESS) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
      for (int c = 0; c < 2; ++c) out[2 * q + c] = W[q][0] * gJ[2 * c] + W[q][1] * gJ[2 * c + 1];
      const int q1 = q == 2 ? 0 : q + 1;
      double* dq = out + 6 + 3 * q;
      double* oq = out + 15 + 4 * q;
      if (PIN && pinned_face) {
        dq[0] = M6[tri(2 * q, 2 * q)];
        dq[1] = M6[tri(2 * q, 2 * q + 1)];
        dq[2] = M6[tri(2 * q + 1, 2 * q + 1)];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) oq[2 * c + c2] = M6[tri(2 * q + c, 2 * q1 + c2)];
      } else {
        // the reference's symmetrisation on the diagonal block
        dq[0] = Xf(wt[q], wt[q], 0, 0) + fl3;
        dq[1] = 0.5 * (Xf(wt[q], wt[q], 0, 1) + Xf(wt[q], wt[q], 1, 0));
        dq[2] = Xf(wt[q], wt[q], 1, 1) + fl3;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) oq[2 * c + c2] = Xf(wt[q], wt[q1], c, c2) + (c == c2 ? fl3 : 0.0);
      }
    }
  } else {  // HVP: y_q = block row q . u
    if (PIN && pinned_face) {
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          double y = 0.0;
#pragma unroll
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) y += M6[tri(2 * q + c, 2 * t + c2)] * U[t][c2];
          out[2 * q + c] = y;
        }
      return;
    }
    double dv[4], gv[4];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int k = 0; k < 2; ++k) dv[2 * c + k] = wt[0][k] * U[0][c] + wt[1][k] * U[1][c] + wt[2][k] * U[2][c];
    if constexpr (PSD) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc += G[tri(i, j)] * dv[j];
        gv[i] = acc;
      }
    } else {
      ok &= dirichlet_hv_closed(J, dv, area, gv);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double y = wt[q][0] * gv[2 * c] + wt[q][1] * gv[2 * c + 1];
        if constexpr (PSD) y += fl3 * (U[0][c] + U[1][c] + U[2][c]);
        out[2 * q + c] = y;
      }
  }
}

// threads per CTA (64 rows): the Hessian's larger records allow fewer CTAs
// per SM, so its CTAs bring two threads per row to phase A
// (problems with pinned vertices under a clamp compile the masked 6x6 clamp
// in: fewer CTAs per SM, more registers)
template <int MODE, bool PSD, bool PIN = false> struct CfCfg {
  static constexpr int NT = MODE == MODE_HESS ? 128 : 64;
  static constexpr int MINB = (PSD && PIN) ? (MODE == MODE_HESS ? 2 : 4)
                                           : (MODE == MODE_HESS ? CF_HESS_MINB : CF_FLAT_MINB);
};
// shared-memory stage of one row block (k_cta_dirichlet): its face-list
// entries, the rows' slot ids (slot | corner << 14), meta words, row order,
// and for the Hessian the incidence records, row starts and row count
template <int MODE> struct CfStage {
  static constexpr int SL = 0, ME = KF * PT * 2, OR = ME + PT * 4, RC = OR + PT * 4,
                       RO = RC + (MODE == MODE_HESS ? KF * PT * 8 : 0), CF = RO + (MODE == MODE_HESS ? PT * 8 : 0);
  __host__ __device__ static size_t bytes(int cf_max) { return (size_t)CF + (size_t)cf_max * 16; }
};

template <int MODE, bool PSD, bool PIN>
__global__ void __launch_bounds__(CfCfg<MODE, PSD>::NT, (CfCfg<MODE, PSD, PIN>::MINB))
    k_cta_dirichlet(const __grid_constant__ FvArgs a) {
  constexpr int NT = CfCfg<MODE, PSD>::NT;
  constexpr int S = CfRec<MODE>::S, NN = 4;
  using STG = CfStage<MODE>;
  // the clamped Hessian reads its streams with plain loads, one row block per
  // CTA (staged: 3.4-3.6 ms vs 3.12 at icosphere(10); its 27-double records
  // already bound residency)
  constexpr bool STAGED = MODE != MODE_HESS;
  constexpr int NSTG = STAGED ? CF_STAGES : 1;
  // persistent CTAs walk row blocks grid-stride; a block's stage (face list,
  // row streams) arrives by TMA NSTG blocks ahead, so phase A starts
  // with its gathers instead of a DRAM round trip for the list
  extern __shared__ __align__(128) unsigned char cf_smem[];
  const size_t sbytes = (STG::bytes(a.cf_max) + 127) & ~(size_t)127;
  double* rec = reinterpret_cast<double*>(cf_smem + (STAGED ? NSTG * sbytes : 0));
  __shared__ __align__(8) uint64_t sbar[NSTG];
  __shared__ int snf[NSTG];
  __shared__ double wsum[NT / 32];
  const int64_t nblocks = (a.V + PT - 1) / PT;
  auto stage_issue = [&](int st, int64_t b) {  // one thread
    unsigned char* sp = cf_smem + st * sbytes;
    const int i0 = a.cf_off[b], nf = a.cf_off[b + 1] - i0;
    snf[st] = nf;
    uint32_t bytes = KF * PT * 2 + PT * 4 + (a.order ? PT * 4 : 0) + (uint32_t)nf * 16;
    if constexpr (MODE == MODE_HESS) bytes += KF * PT * 8 + PT * 8;
    mbar_expect_tx(&sbar[st], bytes);
#pragma unroll
    for (int j = 0; j < KF; ++j) bulk_g2s(sp + STG::SL + j * PT * 2, a.eslot + (int64_t)j * a.es + b * PT, PT * 2, &sbar[st]);
    bulk_g2s(sp + STG::ME, a.rmeta + b * PT, PT * 4, &sbar[st]);
    if (a.order) bulk_g2s(sp + STG::OR, a.order + b * PT, PT * 4, &sbar[st]);
    if constexpr (MODE == MODE_HESS) {
#pragma unroll
      for (int j = 0; j < KF; ++j) bulk_g2s(sp + STG::RC + j * PT * 8, a.ell + (int64_t)j * a.es + b * PT, PT * 8, &sbar[st]);
      bulk_g2s(sp + STG::RO, a.prow_ro + b * PT, PT * 8, &sbar[st]);
    }
    if (nf) bulk_g2s(sp + STG::CF, a.cf_face + i0, (uint32_t)nf * 16, &sbar[st]);
  };
  if constexpr (STAGED) {
    if (threadIdx.x == 0) {
      for (int st = 0; st < NSTG; ++st) mbar_init(&sbar[st], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int st = 0; st < NSTG; ++st)
        if (blockIdx.x + (int64_t)st * gridDim.x < nblocks) stage_issue(st, blockIdx.x + (int64_t)st * gridDim.x);
  }
  bool ok = true;
  int it = 0;
  for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x, ++it) {
  const int64_t row = blk * PT + threadIdx.x;
  const int stn = it % NSTG;
  const unsigned char* sp = cf_smem + stn * sbytes;
  int nfc;
  const int4* cfl;
  if constexpr (STAGED) {
    mbar_wait(&sbar[stn], (uint32_t)(it / NSTG) & 1u);
    nfc = snf[stn];
    cfl = reinterpret_cast<const int4*>(sp + STG::CF);
  } else {
    const int i0 = a.cf_off[blk];
    nfc = a.cf_off[blk + 1] - i0;
    cfl = a.cf_face + i0;
  }
  // phase B's row streams, from the stage into registers
  int g = 0;
  uint32_t meta = 0;
  int64_t ro = 0;
  uint64_t rc[KF];
  int sl[KF];
  const bool has_row = threadIdx.x < PT && row < a.V;
  if (has_row && STAGED) {
    g = a.order ? reinterpret_cast<const int32_t*>(sp + STG::OR)[threadIdx.x] : (int)row;
    meta = reinterpret_cast<const uint32_t*>(sp + STG::ME)[threadIdx.x];
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      rc[j] = 0;
      sl[j] = reinterpret_cast<const uint16_t*>(sp + STG::SL)[j * PT + threadIdx.x];
    }
  } else if (has_row) {  // plain loads (their latency overlaps phase A)
    g = a.order ? a.order[row] : (int)row;
    meta = a.rmeta[row];
    if constexpr (MODE == MODE_HESS) ro = a.prow_ro[row];
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      rc[j] = MODE == MODE_HESS ? a.ell[(int64_t)j * a.es + row] : 0;
      sl[j] = a.eslot[(int64_t)j * a.es + row];
    }
  }
  // phase A: the block's faces, once each
  double eacc = 0.0;
  // two / three faces' loads in flight (one under a clamp: register pressure)
  constexpr int NB = PSD ? 1 : CF_NB;
  for (int i = threadIdx.x; i < nfc; i += NB * NT) {
    int4 fe[NB];
    CfIn d[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int ib = i + b * NT;
      fe[b] = cfl[ib < nfc ? ib : i];
      cf_load<MODE, PSD>(a, fe[b], d[b]);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int ib = i + b * NT;
      if (ib < nfc) {
        double val;
        cf_face<MODE, PSD, PIN>(a, d[b], rec + (size_t)ib * S, val, ok);
        if (MODE != MODE_HVP && ((uint32_t)fe[b].x >> 31)) eacc += val;
      }
    }
  }
  __syncthreads();  // records complete; the stage is read: refill it
  if (STAGED && threadIdx.x == 0 && blk + (int64_t)NSTG * gridDim.x < nblocks) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    stage_issue(stn, blk + (int64_t)NSTG * gridDim.x);
  }
  // phase B: rows sum their incidences' records in incidence order; Hessian
  // blocks go straight to the output row (each 32-byte block is one sector;
  // fan rows write every block once; other rows are cleared, then accumulated)
  if (has_row) {
    const bool fr = !((meta >> 8) & 1);
    const int dp = (int)(meta >> 16) & 0xff;
    const int cnt = (meta & 0xff) < 255 ? (int)(meta & 0xff) : a.rinc_off[row + 1] - a.rinc_off[row];
    const bool fan = (meta >> 9) & 1;
    double* hrow = MODE == MODE_HESS ? a.hess + ro * NN : nullptr;
    if constexpr (MODE == MODE_HESS) {
      const int nblk = (int)((meta >> 24) & 0xff);
      if (!fan)
        for (int k = 0; k < nblk * NN; ++k) hrow[k] = 0.0;
    }
    double vec[2] = {0.0, 0.0}, dg[3] = {0.0, 0.0, 0.0};
    double carry[4] = {0.0, 0.0, 0.0, 0.0}, first[4] = {0.0, 0.0, 0.0, 0.0};
    int first_pos = 255, last_pos2 = 255;
    auto incidence = [&](uint64_t r64, int spk, int jidx) {
      const uint32_t hi = (uint32_t)(r64 >> 32);
      const int s = spk >> 14, slot = spk & 0x3fff;
      const double* r = rec + (size_t)slot * S;
      vec[0] += r[2 * s];
      vec[1] += r[2 * s + 1];
      if constexpr (MODE == MODE_HESS) {
        const int pos1 = (int)(hi & 0xff), pos2 = (int)((hi >> 8) & 0xff);
        const int s2 = s == 0 ? 2 : s - 1;
        const double* dq = r + 6 + 3 * s;
        dg[0] += dq[0];
        dg[1] += dq[1];
        dg[2] += dq[2];
        const double* o1 = r + 15 + 4 * s;   // block (s, s+1)
        const double* o2 = r + 15 + 4 * s2;  // block (s-1, s): block (s, s-1) is its transpose
        const double b1[4] = {o1[0], o1[1], o1[2], o1[3]};
        const double b2[4] = {o2[0], o2[2], o2[1], o2[3]};
        if (fan) {
          if (jidx == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) first[k] = b1[k];
            first_pos = pos1;
          } else if (pos1 != 255) {
            double* dst = hrow + pos1 * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = carry[k] + b1[k];
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) carry[k] = b2[k];
          last_pos2 = pos2;
        } else {
          if (pos1 != 255) {
            double* dst = hrow + pos1 * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] += b1[k];
          }
          if (pos2 != 255) {
            double* dst = hrow + pos2 * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] += b2[k];
          }
        }
      }
    };
#pragma unroll
    for (int j = 0; j < KF; ++j)
      if (j < cnt) incidence(rc[j], sl[j], j);
    for (int k = KF; k < cnt; ++k) {
      const int64_t q = a.rinc_off[row] + k;
      incidence(a.rrec[q], a.rslot[q], k);
    }
    if constexpr (MODE == MODE_HESS) {
      if (fan && cnt > 0) {  // close the fan: the first block meets the last carry, or both stand alone
        if (last_pos2 == first_pos) {
          if (first_pos != 255) {
            double* dst = hrow + first_pos * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = carry[k] + first[k];
          }
        } else {
          if (first_pos != 255) {
            double* dst = hrow + first_pos * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = first[k];
          }
          if (last_pos2 != 255) {
            double* dst = hrow + last_pos2 * NN;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = carry[k];
          }
        }
      }
    }
    double* vout = MODE == MODE_HVP ? a.y : a.grad;
    vout[(int64_t)g * 2] = fr ? vec[0] : 0.0;
    vout[(int64_t)g * 2 + 1] = fr ? vec[1] : 0.0;
    if constexpr (MODE == MODE_HESS) {
      if (fr && dp != 255) {
        double* dst = hrow + dp * NN;
        dst[0] = dg[0];
        dst[1] = dg[1];
        dst[2] = dg[1];
        dst[3] = dg[2];
      }
    }
  }
  if constexpr (MODE != MODE_HVP) {
    // the block's face energies (spread over all its threads by phase A) in
    // fixed order into its first warp's partial; its other row warp's slot is zero
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(0xffffffffu, eacc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = eacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = wsum[0];
#pragma unroll
      for (int w = 1; w < NT / 32; ++w) t += wsum[w];
      a.partials[(blk * PT) >> 5] = t;
    } else if (threadIdx.x == 32 && blk * PT + 32 < a.V) {
      a.partials[(blk * PT + 32) >> 5] = 0.0;
    }
  }
  __syncthreads();  // phase B has read the records (and thread 0 the sums) before the next block's phase A
  }  // row blocks
  if (!ok) *a.redo = 1;
}

// ---------------------------------------------------------------------------
// Sphere barrier + stretch (apps/sphere.py:71-99), BASELINE config 4: gradient
// and matrix-free HVP in closed form through the per-vertex retraction
// p = r / |r|, r = s + x0 b1 + x1 b2 (J = dp/dx = (I - p p^T) B / rho, B = [b1 b2]):
//   face energy  E = -log det[p0 p1 p2] + sum_{a<b} |p_a - p_b|^2  on p-space,
//   c_s = d det / d p_s (cross products), g_s = -c_s / det + 2 (2 p_s - p_s1 - p_s2),
//   (grad^2 E pdot)_s = -cdot_s / det + c_s detdot / det^2 + 2 (2 pdot_s - pdot_s1 - pdot_s2),
//   row: grad_x = J^T sum g_s;  (H u)_x = J^T sum (grad^2 E pdot)_s + (dJ/de)^T sum g_s,
//   dJ/de = [-(pdot p^T + p pdot^T)/rho - (I - p p^T) rhodot / rho^2] B,  pdot = J u.
// Faces are recomputed by each corner row (no communication); non-finite
// faces raise the redo flag (the generic patch kernel then reproduces the
// reference's NaN placement).
struct Retract {
  double p[3], pd[3], rho, rhod;  // p, pdot = J u, |r|, d|r|/de
};

// Reference-order, unfused primal of the retraction and of the barrier's
// determinant. At BASELINE size (icosphere(10), edge ~1.1e-3) det[p0 p1 p2]
// ~1e-6 is a difference of O(1) products, so its rounding (~1e-10 relative)
// moves every face gradient by as much, and the six faces around a vertex
// cancel to a gradient ~25x smaller. Computing p and det with exactly the
// reference's operations (apps/sphere.py:69-71: r = (x0 b1 + x1 b2) + s,
// p = r * (1/sqrt(r.r)); active.py:445-453 cofactor expansion in face
// order; numpy never fuses a multiply-add) makes both bitwise equal to the
// reference's, leaving only well-conditioned differences.
MG_DI double rmul(double a, double b) { return __dmul_rn(a, b); }
MG_DI double radd(double a, double b) { return __dadd_rn(a, b); }
MG_DI double rsub(double a, double b) { return __dsub_rn(a, b); }

MG_DI double retract_ref(const double* s, const double* b1, const double* b2, double x0, double x1, double* r,
                         double* p) {
#pragma unroll
  for (int c = 0; c < 3; ++c) r[c] = radd(radd(rmul(x0, b1[c]), rmul(x1, b2[c])), s[c]);
  const double rho = ::sqrt(radd(radd(rmul(r[0], r[0]), rmul(r[1], r[1])), rmul(r[2], r[2])));
  const double ir = 1.0 / rho;
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = rmul(r[c], ir);
  return rho;
}

// SmallMatrix.from_columns(p0, p1, p2).det() (m_ij = p_j[i])
MG_DI double det_ref(const double* p0, const double* p1, const double* p2) {
  return radd(rsub(rmul(p0[0], rsub(rmul(p1[1], p2[2]), rmul(p2[1], p1[2]))),
                   rmul(p1[0], rsub(rmul(p0[1], p2[2]), rmul(p2[1], p0[2])))),
              rmul(p2[0], rsub(rmul(p0[1], p1[2]), rmul(p1[1], p0[2]))));
}

MG_DI Retract retract(const double* s, const double* b1, const double* b2, double x0, double x1, double u0, double u1) {
  Retract R;
  double r[3], rd[3];
  R.rho = retract_ref(s, b1, b2, x0, x1, r, R.p);
  const double ir = 1.0 / R.rho;
#pragma unroll
  for (int c = 0; c < 3; ++c) rd[c] = u0 * b1[c] + u1 * b2[c];
  const double prd = R.p[0] * rd[0] + R.p[1] * rd[1] + R.p[2] * rd[2];
  R.rhod = prd;
#pragma unroll
  for (int c = 0; c < 3; ++c) R.pd[c] = (rd[c] - R.p[c] * prd) * ir;
  return R;
}

MG_DI void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// per-vertex retraction once per call: p and pdot = J u (u free-masked)
template <int MODE>
__global__ void k_sphere_retract(const __grid_constant__ FvArgs a, const uint8_t* fixed) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= a.nv) return;
  const bool pinned = fixed && fixed[v];
  double u0 = 0.0, u1 = 0.0;
  if (MODE == MODE_HVP && !pinned) {
    u0 = a.w[v * 2];
    u1 = a.w[v * 2 + 1];
  }
  const Retract R = retract(a.t.a[0] + 3 * v, a.t.a[1] + 3 * v, a.t.a[2] + 3 * v, a.x[v * 2], a.x[v * 2 + 1], u0, u1);
  double* o = a.vscr + 6 * v;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    o[c] = R.p[c];
    if constexpr (MODE == MODE_HVP) o[3 + c] = R.pd[c];
  }
}

template <int MODE>
#ifndef SPH_MINB
#define SPH_MINB 1  // 118 registers, 8 CTAs/SM; 9 / 10 / 12 CTAs (spills): HVP 1.686 / 1.686 / 1.931 vs 1.542 ms at icosphere(10)
#endif
__global__ void __launch_bounds__(PT, SPH_MINB) k_rows_sphere(const __grid_constant__ FvArgs a) {
  const int64_t row = (int64_t)blockIdx.x * PT + threadIdx.x;
  double eacc = 0.0;
  bool ok = true;
  if (row < a.V) {
    const int g = a.order ? a.order[row] : (int)row;
    const uint32_t meta = a.rmeta[row];
    uint64_t rc[KF];
#pragma unroll
    for (int j = 0; j < KF; ++j) rc[j] = a.ell[(int64_t)j * a.es + row];
    const bool fr = !((meta >> 8) & 1);
    const int cnt = (meta & 0xff) < 255 ? (int)(meta & 0xff) : a.rinc_off[row + 1] - a.rinc_off[row];
    const bool barrier = a.t.c[0] != 0.0, stretch = a.t.c[1] != 0.0;
    const double* S = a.t.a[0];
    const double* B1 = a.t.a[1];
    const double* B2 = a.t.a[2];
    double A[3] = {0.0, 0.0, 0.0}, Bs[3] = {0.0, 0.0, 0.0};  // sum (grad^2 E pdot)_s, sum g_s
    auto corner = [&](int v, bool pinned) {
      const double x0 = a.x[(int64_t)v * 2], x1 = a.x[(int64_t)v * 2 + 1];
      double u0 = 0.0, u1 = 0.0;
      if (MODE == MODE_HVP && !pinned) {
        u0 = a.w[(int64_t)v * 2];
        u1 = a.w[(int64_t)v * 2 + 1];
      }
      return retract(S + 3 * (int64_t)v, B1 + 3 * (int64_t)v, B2 + 3 * (int64_t)v, x0, x1, u0, u1);
    };
    // the row's own retraction (p, pdot) once; the other two corners' per incidence
    double ps[3], ds[3];
    {
      const double* o = a.vscr + 6 * (int64_t)g;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ps[c] = o[c];
        ds[c] = MODE == MODE_HVP ? o[3 + c] : 0.0;
      }
    }
    struct Other {
      double p1[3], p2[3], d1[3], d2[3];
    };
    auto load_other = [&](int o1, int o2) {
      Other r;
      const double* q1 = a.vscr + 6 * (int64_t)o1;
      const double* q2 = a.vscr + 6 * (int64_t)o2;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        r.p1[c] = q1[c];
        r.p2[c] = q2[c];
        r.d1[c] = MODE == MODE_HVP ? q1[3 + c] : 0.0;
        r.d2[c] = MODE == MODE_HVP ? q2[3 + c] : 0.0;
      }
      return r;
    };
    auto incidence = [&](uint64_t r64, const Other& O) {
      const uint32_t lo = (uint32_t)r64;
      const int s = (int)(lo >> 30);
      const double* p1 = O.p1;
      const double* p2 = O.p2;
      const double* d1 = O.d1;
      const double* d2 = O.d2;
      double val = 0.0, gs[3] = {0.0, 0.0, 0.0}, hs[3] = {0.0, 0.0, 0.0};
      if (barrier) {
        // det[p0 p1 p2] = ps . (p1 x p2) for the cyclic order (s, s1, s2)
        double cs[3], c1[3], c2[3];
        cross3(p1, p2, cs);
        cross3(p2, ps, c1);
        cross3(ps, p1, c2);
        // the determinant in the face's own corner order (slot s is this row)
        double f0[3], f1[3], f2[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          f0[c] = s == 0 ? ps[c] : (s == 1 ? p2[c] : p1[c]);
          f1[c] = s == 0 ? p1[c] : (s == 1 ? ps[c] : p2[c]);
          f2[c] = s == 0 ? p2[c] : (s == 1 ? p1[c] : ps[c]);
        }
        const double det = det_ref(f0, f1, f2);
        const double id = rcp_fast(det);  // non-finite / zero det -> non-finite, the exact path takes over
        // the value only feeds the gradient call's energy; the HVP needs the
        // derivative factors (finite for any det != 0, like the reference's dual)
        if constexpr (MODE == MODE_GRAD) val += -::log(det);
#pragma unroll
        for (int c = 0; c < 3; ++c) gs[c] += -cs[c] * id;
        if constexpr (MODE == MODE_HVP) {
          double t1[3], t2[3];
          cross3(d1, p2, t1);
          cross3(p1, d2, t2);
          const double detd = cs[0] * ds[0] + cs[1] * ds[1] + cs[2] * ds[2] + c1[0] * d1[0] + c1[1] * d1[1] +
                              c1[2] * d1[2] + c2[0] * d2[0] + c2[1] * d2[1] + c2[2] * d2[2];
#pragma unroll
          for (int c = 0; c < 3; ++c) hs[c] += -(t1[c] + t2[c]) * id + cs[c] * detd * id * id;
        }
      }
      if (stretch) {
        double e01 = 0.0, e12 = 0.0, e20 = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double a01 = ps[c] - p1[c], a12 = p1[c] - p2[c], a20 = p2[c] - ps[c];
          e01 += a01 * a01;
          e12 += a12 * a12;
          e20 += a20 * a20;
          gs[c] += 2.0 * (2.0 * ps[c] - p1[c] - p2[c]);
          if constexpr (MODE == MODE_HVP) hs[c] += 2.0 * (2.0 * ds[c] - d1[c] - d2[c]);
        }
        val += e01 + e12 + e20;
      }
      ok &= isfinite(val + gs[0] + gs[1] + gs[2] + hs[0] + hs[1] + hs[2]);
      if (MODE == MODE_GRAD && s == 0) eacc += val;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        Bs[c] += gs[c];
        A[c] += hs[c];
      }
    };
    const int ne = cnt < KF ? cnt : KF;
    uint64_t ov[KF];
#pragma unroll
    for (int j = 0; j < KF; ++j) ov[j] = a.ellv[(int64_t)j * a.es + row];
    // corners streamed one incidence ahead of the compute
    Other cur;
    if (ne > 0) cur = load_other((int)(uint32_t)ov[0], (int)(ov[0] >> 32));
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      if (j < ne) {
        Other nxt;
        if (j + 1 < ne) nxt = load_other((int)(uint32_t)ov[j + 1], (int)(ov[j + 1] >> 32));
        incidence(rc[j], cur);
        cur = nxt;
      }
    }
    for (int k = KF; k < cnt; ++k) {
      const uint64_t r64 = a.rrec[a.rinc_off[row] + k];
      const int64_t f = (uint32_t)r64 & 0x3fffffffu;
      const int s = (int)((uint32_t)r64 >> 30);
      incidence(r64, load_other(a.faces[3 * f + (s + 1) % 3], a.faces[3 * f + (s + 2) % 3]));
    }
    // the row's own retraction: J, dJ
    const Retract R = corner(g, !fr);
    const double* b1 = B1 + 3 * (int64_t)g;
    const double* b2 = B2 + 3 * (int64_t)g;
    const double ir = 1.0 / R.rho;
    // (I - p p^T) v / rho
    auto proj = [&](const double* v, double* o) {
      const double pv = R.p[0] * v[0] + R.p[1] * v[1] + R.p[2] * v[2];
#pragma unroll
      for (int c = 0; c < 3; ++c) o[c] = (v[c] - R.p[c] * pv) * ir;
    };
    double out[2];
    double q[3];
    if constexpr (MODE == MODE_GRAD) {
      proj(Bs, q);  // J^T Bs = B^T (I - p p^T) Bs / rho
      out[0] = q[0] * b1[0] + q[1] * b1[1] + q[2] * b1[2];
      out[1] = q[0] * b2[0] + q[1] * b2[1] + q[2] * b2[2];
    } else {
      double qa[3];
      proj(A, qa);
      // dJ^T Bs = B^T [-(p pdot^T + pdot p^T) Bs / rho - (I - p p^T) Bs rhodot / rho^2]
      const double pB = R.p[0] * Bs[0] + R.p[1] * Bs[1] + R.p[2] * Bs[2];
      const double dB = R.pd[0] * Bs[0] + R.pd[1] * Bs[1] + R.pd[2] * Bs[2];
      double qb[3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        qb[c] = -(R.p[c] * dB + R.pd[c] * pB) * ir - (Bs[c] - R.p[c] * pB) * R.rhod * ir * ir;
#pragma unroll
      for (int c = 0; c < 3; ++c) q[c] = qa[c] + qb[c];
      out[0] = q[0] * b1[0] + q[1] * b1[1] + q[2] * b1[2];
      out[1] = q[0] * b2[0] + q[1] * b2[1] + q[2] * b2[2];
    }
    double* vout = MODE == MODE_HVP ? a.y : a.grad;
    vout[(int64_t)g * 2] = fr ? out[0] : 0.0;
    vout[(int64_t)g * 2 + 1] = fr ? out[1] : 0.0;
  }
  if (!ok) *a.redo = 1;
  if constexpr (MODE != MODE_HVP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(0xffffffffu, eacc, o);
    if ((threadIdx.x & 31) == 0) a.partials[row >> 5] = eacc;
  }
}


// Sphere HVP under a PSD clamp (the Newton-CG probe, solvers.py:274-277):
// face-parallel pass + fixed-order row gather. Per face, the 6x6 Hessian in
// x comes in closed form from the retraction p = r / |r| (J_q = dp_q/dx_q):
//   H[q][q'] = J_q^T Hp[q][q'] J_q' + delta_qq' T_q,   T_q[i][j] = g_q . d2p_q/dx_i dx_j,
//   Hp = -D2 / det + c c^T / det^2  (barrier; c_q = d det / d p_q, D2 = d2 det, cross-product blocks)
//        + 2 L (x) I_3              (stretch; L the triangle's graph Laplacian),
// pinned corners' rows / columns zeroed (the reference's masked lift), then
// clamped (active.py:490-504) and applied to the masked direction; the face's
// three 2-vectors go to scratch and each owned row sums its faces' entries in
// its fixed incidence order. Non-finite faces raise the redo flag.
__global__ void __launch_bounds__(128) k_sphere_face_hvp_psd(const __grid_constant__ FvArgs a, const uint8_t* fixed,
                                                            double* yscr) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= a.nf) return;
  int v[3];
  bool pin[3];
  double p[3][3], J[3][3][2], B[3][3][2], rho[3], u[3][2];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    v[q] = a.faces[3 * f + q];
    pin[q] = fixed && fixed[v[q]];
    const double* S = a.t.a[0] + 3 * (int64_t)v[q];
    const double* b1 = a.t.a[1] + 3 * (int64_t)v[q];
    const double* b2 = a.t.a[2] + 3 * (int64_t)v[q];
    const double x0 = a.x[(int64_t)v[q] * 2], x1 = a.x[(int64_t)v[q] * 2 + 1];
    u[q][0] = pin[q] ? 0.0 : a.w[(int64_t)v[q] * 2];
    u[q][1] = pin[q] ? 0.0 : a.w[(int64_t)v[q] * 2 + 1];
    double r[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      B[q][c][0] = b1[c];
      B[q][c][1] = b2[c];
    }
    const double ir = 1.0 / retract_ref(S, b1, b2, x0, x1, r, p[q]);
    rho[q] = ir;  // 1 / |r| (only the inverse is used below)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double pb = p[q][0] * B[q][0][j] + p[q][1] * B[q][1][j] + p[q][2] * B[q][2][j];
#pragma unroll
      for (int c = 0; c < 3; ++c) J[q][c][j] = (B[q][c][j] - p[q][c] * pb) * ir;
    }
  }
  const bool barrier = a.t.c[0] != 0.0, stretch = a.t.c[1] != 0.0;
  // p-space gradient; the Hessian enters only through its x-space blocks
  //   barrier: Hp = c c^T / det^2 + (1/det) E, E[q][q+1] = [p_{q+2}]x, E[q][q+2] = -[p_{q+1}]x
  //   stretch: Hp[q][q] = 4 I, Hp[q][q'] = -2 I
  double g[3][3], jc[3][2];
  double id = 0.0, chk = 0.0;
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int c = 0; c < 3; ++c) g[q][c] = 0.0;
  if (barrier) {
    double cc[3][3];
    cross3(p[1], p[2], cc[0]);
    cross3(p[2], p[0], cc[1]);
    cross3(p[0], p[1], cc[2]);
    const double det = det_ref(p[0], p[1], p[2]);
    id = 1.0 / det;
    chk += ::log(det);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
      for (int c = 0; c < 3; ++c) g[q][c] -= cc[q][c] * id;
#pragma unroll
      for (int i = 0; i < 2; ++i) jc[q][i] = (J[q][0][i] * cc[q][0] + J[q][1][i] * cc[q][1] + J[q][2][i] * cc[q][2]) * id;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 3; ++q) jc[q][0] = jc[q][1] = 0.0;
  }
  if (stretch) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int qa = q == 2 ? 0 : q + 1, qb = q == 0 ? 2 : q - 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) g[q][c] += 2.0 * (2.0 * p[q][c] - p[qa][c] - p[qb][c]);
    }
  }
  // x-space packed 6x6 (rows / columns 2q + i), blocks q2 <= q
  double H[21];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int q2 = 0; q2 <= q; ++q2)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int R = 2 * q + i, C = 2 * q2 + j;
          if (C > R) continue;
          double acc = jc[q][i] * jc[q2][j];
          const double jj = J[q][0][i] * J[q2][0][j] + J[q][1][i] * J[q2][1][j] + J[q][2][i] * J[q2][2][j];
          if (stretch) acc += (q == q2 ? 4.0 : -2.0) * jj;
          if (barrier && q != q2) {
            // q2 = q + 1 (mod 3): + [p_{q+2}]x ; q2 = q + 2: - [p_{q+1}]x
            const int qa = q == 2 ? 0 : q + 1, qb = q == 0 ? 2 : q - 1;
            const bool next = q2 == qa;
            const double* pk = next ? p[qb] : p[qa];
            double cx[3];
            const double v3[3] = {J[q2][0][j], J[q2][1][j], J[q2][2][j]};
            cross3(pk, v3, cx);
            const double e = J[q][0][i] * cx[0] + J[q][1][i] * cx[1] + J[q][2][i] * cx[2];
            acc += next ? id * e : -id * e;
          }
          if (q == q2) {  // T_q[i][j] = g_q . d2 p_q / dx_i dx_j (symmetrised)
            auto tij = [&](int ii, int jj2) {
              const double pbi = p[q][0] * B[q][0][ii] + p[q][1] * B[q][1][ii] + p[q][2] * B[q][2][ii];
              const double rdj = p[q][0] * B[q][0][jj2] + p[q][1] * B[q][1][jj2] + p[q][2] * B[q][2][jj2];
              double gp = 0.0, gpd = 0.0, pdb = 0.0, gb = 0.0;
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                gp += g[q][c] * p[q][c];
                gpd += g[q][c] * J[q][c][jj2];
                pdb += J[q][c][jj2] * B[q][c][ii];
                gb += g[q][c] * B[q][c][ii];
              }
              const double ir = rho[q];
              return -(gpd * pbi + gp * pdb) * ir - (gb - gp * pbi) * rdj * ir * ir;
            };
            acc += 0.5 * (tij(i, j) + tij(j, i));
          }
          H[tri(R, C)] = (pin[q] || pin[q2]) ? 0.0 : acc;
          chk += H[tri(R, C)];
        }
  if (!isfinite(chk)) {
    *a.redo = 1;
    return;
  }
  {
    // the face Hessian's one eigenvalue below the floor (every face at the
    // benchmark state: -0.85 of the spectral radius, next eigenvalue > 0) is
    // the barrier's twist mode, the in-plane rotation about the centroid
    // (measured overlap 0.994): start the certified rank-one update from its
    // tangent coordinates B^T (n x (p_q - c)); anything else (no eigenvalue
    // below the floor, several, pinned corners) falls through to the general
    // clamp
    double z[6], cen[3], e1[3], e2[3], nrm[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      cen[c] = (p[0][c] + p[1][c] + p[2][c]) * (1.0 / 3.0);
      e1[c] = p[1][c] - p[0][c];
      e2[c] = p[2][c] - p[0][c];
    }
    cross3(e1, e2, nrm);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double d[3], t[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = p[q][c] - cen[c];
      cross3(nrm, d, t);
#pragma unroll
      for (int j = 0; j < 2; ++j) z[2 * q + j] = B[q][0][j] * t[0] + B[q][1][j] * t[1] + B[q][2][j] * t[2];
    }
    if (!psd_rank1_update<6>(H, a.floor, z)) project_if_needed<6>(H, a.floor);
  }
  const double uu[6] = {u[0][0], u[0][1], u[1][0], u[1][1], u[2][0], u[2][1]};
  double2* out = reinterpret_cast<double2*>(yscr + f * 6);
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    double yy[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < 6; ++l) acc += H[tri(2 * q + i, l)] * uu[l];
      yy[i] = acc;
    }
    out[q] = make_double2(yy[0], yy[1]);
  }
}

// y_row = sum over the row's faces (fixed incidence order) of the face's entry
__global__ void __launch_bounds__(PT) k_rows_face_gather(const __grid_constant__ FvArgs a, const double* yscr) {
  const int64_t row = (int64_t)blockIdx.x * PT + threadIdx.x;
  if (row >= a.V) return;
  const int g = a.order ? a.order[row] : (int)row;
  const uint32_t meta = a.rmeta[row];
  const bool fr = !((meta >> 8) & 1);
  const int cnt = (meta & 0xff) < 255 ? (int)(meta & 0xff) : a.rinc_off[row + 1] - a.rinc_off[row];
  uint64_t rc[KF];
#pragma unroll
  for (int j = 0; j < KF; ++j) rc[j] = a.ell[(int64_t)j * a.es + row];
  double2 yv[KF];
#pragma unroll
  for (int j = 0; j < KF; ++j) {
    const uint32_t lo = (uint32_t)rc[j];
    yv[j] = j < cnt ? reinterpret_cast<const double2*>(yscr + (int64_t)(lo & 0x3fffffffu) * 6)[lo >> 30]
                    : make_double2(0.0, 0.0);
  }
  double y0 = 0.0, y1 = 0.0;
#pragma unroll
  for (int j = 0; j < KF; ++j) {
    y0 += yv[j].x;
    y1 += yv[j].y;
  }
  for (int k = KF; k < cnt; ++k) {
    const uint32_t lo = (uint32_t)a.rrec[a.rinc_off[row] + k];
    const double2 t = reinterpret_cast<const double2*>(yscr + (int64_t)(lo & 0x3fffffffu) * 6)[lo >> 30];
    y0 += t.x;
    y1 += t.y;
  }
  a.y[(int64_t)g * 2] = fr ? y0 : 0.0;
  a.y[(int64_t)g * 2 + 1] = fr ? y1 : 0.0;
}

// (a CTA face-list variant of the sphere kernels, each face once per 64-row
// block like k_cta_dirichlet, measured slower at icosphere(10): gradient
// 1.23 vs 1.105 ms, HVP 2.07 vs 1.54 — the per-incidence work is light once
// the retraction is per vertex, so the records' round trip does not pay)
template <int MODE>
void launch_sphere(const Problem& p, const FvArgs& a, cudaStream_t st) {
  const int64_t nb = (a.V + PT - 1) / PT;
  if (!nb) return;
  timing_begin(p, st);
  k_sphere_retract<MODE><<<(unsigned)((a.nv + 255) / 256), 256, 0, st>>>(a, p.any_fixed ? p.fixed.p : nullptr);
  MG_LAUNCH_CHECK();
  k_rows_sphere<MODE><<<(unsigned)nb, PT, 0, st>>>(a);
  MG_LAUNCH_CHECK();
  timing_end(p, st);
}

// MG_FV_CTA=0: the per-row kernel (each face evaluated by each owner row)
// with the per-face PSD pre-pass (A/B runs)
bool fv_cta_enabled() {
  static const bool on = [] {
    const char* e = getenv("MG_FV_CTA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CF_HESS_CTA 0: the unclamped Hessian keeps the per-row kernel (icosphere(10):
// per-row 2.05 ms, CTA lists 2.53 with direct block stores / 2.80 with the row
// buffers; under the clamp the CTA lists win, 3.32 vs 3.87 ms)
#ifndef CF_HESS_CTA
#define CF_HESS_CTA 0
#endif
// shared memory of the CTA face-list kernel: CF_STAGES stages, then the face records
size_t cta_smem(int mode, int cf_max, int) {
  const size_t S = mode == MODE_HESS ? CfRec<MODE_HESS>::S : CfRec<MODE_GRAD>::S;
  const size_t sb = mode == MODE_HESS ? CfStage<MODE_HESS>::bytes(cf_max) : CfStage<MODE_GRAD>::bytes(cf_max);
  return (mode == MODE_HESS ? 1 : CF_STAGES) * ((sb + 127) & ~(size_t)127) * (mode == MODE_HESS ? 0 : 1) +
         (size_t)cf_max * S * 8;
}
bool fv_use_cta(const Problem& p, int mode, bool psd) {
  const int hd = mode == MODE_HESS ? p.max_patch_hdoubles : 0;
  return (mode != MODE_HESS || psd || CF_HESS_CTA) && p.cf_max > 0 && cta_smem(mode, p.cf_max, hd) <= 227 * 1024 &&
         fv_cta_enabled();
}

template <int MODE, bool PSD>
void launch_fv(const Problem& p, const FvArgs& a, int hd_max, cudaStream_t st) {
  const size_t sm = MODE == MODE_HESS ? (size_t)hd_max * 8 + 16 : 0;
  if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "row block does not fit in shared memory");
  const int64_t nb = (a.V + PT - 1) / PT;
  if (!nb) return;
  const size_t smc = cta_smem(MODE, a.cf_max, hd_max);
  if (fv_use_cta(p, MODE, PSD)) {
    auto kc = (PSD && a.fixed) ? k_cta_dirichlet<MODE, PSD, true> : k_cta_dirichlet<MODE, PSD, false>;
    MG_CUDA(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc));
    int64_t grid = nb;  // persistent CTAs: as many as are resident (the clamped Hessian: one block per CTA,
    if (MODE != MODE_HESS || CF_PERSIST_HESS) {  // measured 3.12 vs 3.42 ms persistent at icosphere(10))
      int dev = 0, sms = 148, per_sm = 1;
      MG_CUDA(cudaGetDevice(&dev));
      MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kc, CfCfg<MODE, PSD>::NT, smc));
      if ((int64_t)sms * (per_sm > 0 ? per_sm : 1) < grid) grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    }
    timing_begin(p, st);
    kc<<<(unsigned)grid, CfCfg<MODE, PSD>::NT, smc, st>>>(a);
    MG_LAUNCH_CHECK();
    timing_end(p, st);
    return;
  }
  auto kern = (PSD && a.fpsd6) ? k_rows_dirichlet<MODE, PSD, true> : k_rows_dirichlet<MODE, PSD, false>;
  if (sm) MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  // persistent CTAs (the staged level-1 ring): as many as are resident
  int64_t grid = nb;
  {
    int dev = 0, sms = 148, per_sm = 1;
    MG_CUDA(cudaGetDevice(&dev));
    MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PT, sm));
    if ((int64_t)sms * (per_sm > 0 ? per_sm : 1) < grid) grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  }
  timing_begin(p, st);
  if constexpr (PSD) {
    if (a.nf) k_face_psd<<<(unsigned)((a.nf + 127) / 128), 128, 0, st>>>(a);
    MG_LAUNCH_CHECK();
    if (a.nf && a.fpsd6) k_face_psd_pinned<<<(unsigned)((a.nf + 127) / 128), 128, 0, st>>>(a);
    MG_LAUNCH_CHECK();
  }
  kern<<<(unsigned)grid, PT, sm, st>>>(a);
  MG_LAUNCH_CHECK();
  timing_end(p, st);
}

}  // namespace

int64_t launch_patch_fv(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  const Mesh& m = *p.mesh;
  FvArgs a;
  a.V = m.Vr;
  a.order = (m.row_order_used == MG_ROW_IDENTITY && !m.owned.p) ? nullptr
            : (p.order_pad.n >= m.Vr && p.order_pad.p ? p.order_pad.p : m.patches.order.p);
  a.rmeta = p.rmeta.p;
  a.ell = p.ell.p;
  a.rinc_off = p.rinc_off.p;
  a.rrec = p.rrec.p;
  a.prow_ro = p.prow_ro.p;
  a.hoff = p.hoff.p;
  a.faces = m.faces.p;
  a.ellv = p.ellv.p;
  a.es = p.ell_stride ? p.ell_stride : m.Vr;
  a.x = c.x;
  a.w = c.w;
  a.grad = c.grad;
  a.hess = c.hess;
  a.y = c.y;
  a.partials = c.partials + partial_offset;
  a.redo = p.redo.p;
  a.floor = c.floor;
  a.t = p.terms[0].dev;
  a.nv = m.V;
  a.vscr = nullptr;
  a.nf = m.F;
  a.fpsd = nullptr;
  a.fpsd6 = nullptr;
  a.fixed = p.any_fixed ? p.fixed.p : nullptr;
  a.cf_off = p.cf_off.p;
  a.cf_face = p.cf_face.p;
  a.eslot = p.eslot.p;
  a.rslot = p.rslot.p;
  a.cf_max = p.cf_max;
  if (c.psd && mode != MODE_GRAD && a.t.type != MG_TERM_SPHERE && !fv_use_cta(p, mode, true)) {
    if (p.fpsd.n < 10 * m.F) p.fpsd.alloc(10 * m.F > 0 ? 10 * m.F : 2);
    a.fpsd = p.fpsd.p;
    if (p.any_fixed) {
      if (p.fpsd6.n < 21 * m.F) p.fpsd6.alloc(21 * m.F > 0 ? 21 * m.F : 2);
      a.fpsd6 = p.fpsd6.p;
    }
  }
  const int hd = mode == MODE_HESS ? p.max_patch_hdoubles : 0;
  if (a.t.type == MG_TERM_SPHERE) {
    if (p.vscr.n < 6 * m.V) p.vscr.alloc(6 * m.V > 0 ? 6 * m.V : 1);
    a.vscr = p.vscr.p;
    if (mode == MODE_GRAD) launch_sphere<MODE_GRAD>(p, a, c.stream);
    else if (mode == MODE_HVP && !c.psd) launch_sphere<MODE_HVP>(p, a, c.stream);
    else if (mode == MODE_HVP) {
      if (p.fpsd.n < 6 * m.F) p.fpsd.alloc(6 * m.F > 0 ? 6 * m.F : 2);
      timing_begin(p, c.stream);
      if (m.F)
        k_sphere_face_hvp_psd<<<(unsigned)((m.F + 127) / 128), 128, 0, c.stream>>>(a, p.any_fixed ? p.fixed.p : nullptr,
                                                                                 p.fpsd.p);
      MG_LAUNCH_CHECK();
      if (m.Vr) k_rows_face_gather<<<(unsigned)((m.Vr + PT - 1) / PT), PT, 0, c.stream>>>(a, p.fpsd.p);
      MG_LAUNCH_CHECK();
      timing_end(p, c.stream);
    } else throw Error(MG_ERR_UNSUPPORTED, "sphere face kernels: gradient and HVP only");
    return mode == MODE_HVP ? 0 : (m.Vr + 31) / 32;
  }
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
