// Per-element eigenvalue clamp, in registers.
//
// Reference: project_psd (meshgrad/active.py:490-504): w, Q = eigh(H);
// w = max(w, floor); out = Q diag(w) Q^T; out = 0.5 (out + out^T).
// `_extract` (problem.py:454-476) symmetrises first and only projects lanes
// whose Hessian is entirely finite.
//
// The spectral projector is unique even when eigenvectors are not, so any
// accurate symmetric eigensolver reproduces the reference to rounding
// (cyclic Jacobi matched eigh to <= 1e-14 relative).
//
// Paths:
//  * a Cholesky test of A - floor*I: already above the floor -> unchanged;
//  * 2x2 / 3x3: non-iterative deflation solver (psd_small.h);
//  * cyclic Jacobi on the packed K x K matrix (generic, K <= 12);
//  * a two-point shortcut: when H == [[A,-A],[-A,A]] bitwise (every
//    translation-invariant edge term: springs, edge lengths), the spectrum is
//    {2 eig(A)} U {0,0,0}, so P(H) = 1/2 [[P2, -P2],[-P2, P2]] + f/2 [[I, I],[I, I]]
//    with P2 = Q max(2 Lambda, f) Q^T from an n x n Jacobi. Exact same
//    projector, a fraction of the flops. The test is a runtime bitwise check,
//    so any other Hessian silently takes the generic path.
#pragma once
#include "dual.cuh"
#include "psd_small.h"

namespace mg {

// In-place: A (packed K x K, symmetric) -> Q max(Lambda, floor) Q^T.
template <int K>
MG_DI void jacobi_project(double* A, double floor) {
  constexpr int T = TriN<K>::value;
  double Q[K][K];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) Q[i][j] = (i == j) ? 1.0 : 0.0;

  double fro2 = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) fro2 += (i == j ? 1.0 : 2.0) * A[tri(i, j)] * A[tri(i, j)];
  const double tol2 = fro2 * 1e-30;  // off-diagonal mass ~1e-15 relative: below eigh-level error, far below the 1e-10 bar

  for (int sweep = 0; sweep < 12; ++sweep) {
    double off = 0.0;
#pragma unroll
    for (int i = 1; i < K; ++i)
#pragma unroll
      for (int j = 0; j < i; ++j) off += A[tri(i, j)] * A[tri(i, j)];
    if (!(off > tol2)) break;
#pragma unroll
    for (int p = 0; p < K - 1; ++p) {
#pragma unroll
      for (int q = p + 1; q < K; ++q) {
        const double apq = A[tri(q, p)];
        if (apq != 0.0) {
          const double app = A[tri(p, p)], aqq = A[tri(q, q)];
          const double theta = (aqq - app) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + ::sqrt(theta * theta + 1.0));
          const double c = 1.0 / ::sqrt(t * t + 1.0), s = t * c;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (k != p && k != q) {
              const double akp = A[tri(k, p)], akq = A[tri(k, q)];
              A[tri(k, p)] = c * akp - s * akq;
              A[tri(k, q)] = s * akp + c * akq;
            }
          }
          A[tri(p, p)] = app - t * apq;
          A[tri(q, q)] = aqq + t * apq;
          A[tri(q, p)] = 0.0;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const double qkp = Q[k][p], qkq = Q[k][q];
            Q[k][p] = c * qkp - s * qkq;
            Q[k][q] = s * qkp + c * qkq;
          }
        }
      }
    }
  }
  double w[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double l = A[tri(j, j)];
    w[j] = l > floor ? l : floor;  // np.maximum (NaN-free here: lanes are finite)
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) acc += Q[i][j] * w[j] * Q[k][j];
      A[tri(i, k)] = acc;
    }
  (void)T;
}

// 1/x: hardware estimate + two Newton steps (full fp64 precision for finite,
// non-zero x; the callers only pass such values)
MG_DI double psd_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Jacobi rotation zeroing a_pq: t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)),
// theta = (a_qq - a_pp) / (2 a_pq), written without divisions
MG_DI void jacobi_angle(double app, double aqq, double apq, double& c, double& s, double& t) {
  const double d = aqq - app, b = 2.0 * apq;
  const double h = ::sqrt(d * d + b * b);
  const double sg = ((d >= 0.0) == (b >= 0.0)) ? 1.0 : -1.0;
  t = sg * fabs(b) * psd_rcp(fabs(d) + h);
  c = rsqrt(fma(t, t, 1.0));
  s = t * c;
}

// round-robin (circle method) orderings: K/2 disjoint pairs per step, K-1
// steps per sweep; the pairs of a step are independent, so their angles and
// updates interleave (instruction-level parallelism on the rotation chain)
template <int K> struct RoundRobin;
// pair k of step st: 4-bit fields of a packed code, (0,1),(2,3) / (0,2),(1,3) / ...
template <> struct RoundRobin<4> {
  static constexpr int S = 3, PP = 2;
  static constexpr unsigned long long PC = 0x101020ull, QC = 0x233231ull;
};
template <> struct RoundRobin<6> {
  static constexpr int S = 5, PP = 3;
  static constexpr unsigned long long PC = 0x210130120410320ull, QC = 0x345254543532451ull;
};
MG_DI constexpr int rr_field(unsigned long long code, int i) { return (int)((code >> (4 * i)) & 0xF); }

// In-place: A (packed K x K, symmetric) -> Q max(Lambda, floor) Q^T, parallel
// ordering (K = 4, 6)
template <int K>
MG_DI void jacobi_project_rr(double* A, double floor) {
  using RR = RoundRobin<K>;
  double Q[K][K];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) Q[i][j] = (i == j) ? 1.0 : 0.0;
  double fro2 = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) fro2 += (i == j ? 1.0 : 2.0) * A[tri(i, j)] * A[tri(i, j)];
  // stop at off-diagonal mass 1e-12 of the Frobenius norm: the clamp max(l, f)
  // is Lipschitz, and a pair mixed by the residual rotation is either both
  // clamped (no effect) or separated by at least f - l_min, so the projector's
  // error stays at the residual's level, two orders under the 1e-10 bar
  const double tol2 = fro2 * 1e-24;
  for (int sweep = 0; sweep < 12; ++sweep) {
    double off = 0.0;
#pragma unroll
    for (int i = 1; i < K; ++i)
#pragma unroll
      for (int j = 0; j < i; ++j) off += A[tri(i, j)] * A[tri(i, j)];
    if (!(off > tol2)) break;
#pragma unroll
    for (int st = 0; st < RR::S; ++st) {
      double c[RR::PP], sn[RR::PP], t[RR::PP];
#pragma unroll
      for (int k = 0; k < RR::PP; ++k) {
        const int p = rr_field(RR::PC, st * RR::PP + k), q = rr_field(RR::QC, st * RR::PP + k);
        const double apq = A[tri(q, p)];
        if (apq != 0.0) {
          jacobi_angle(A[tri(p, p)], A[tri(q, q)], apq, c[k], sn[k], t[k]);
        } else {
          c[k] = 1.0;
          sn[k] = 0.0;
          t[k] = 0.0;
        }
      }
#pragma unroll
      for (int k = 0; k < RR::PP; ++k) {
        const int p = rr_field(RR::PC, st * RR::PP + k), q = rr_field(RR::QC, st * RR::PP + k);
        const double apq = A[tri(q, p)];
#pragma unroll
        for (int m = 0; m < K; ++m) {
          if (m != p && m != q) {
            const double amp = A[tri(m, p)], amq = A[tri(m, q)];
            A[tri(m, p)] = c[k] * amp - sn[k] * amq;
            A[tri(m, q)] = sn[k] * amp + c[k] * amq;
          }
        }
        A[tri(p, p)] -= t[k] * apq;
        A[tri(q, q)] += t[k] * apq;
        A[tri(q, p)] = 0.0;
#pragma unroll
        for (int m = 0; m < K; ++m) {
          const double qmp = Q[m][p], qmq = Q[m][q];
          Q[m][p] = c[k] * qmp - sn[k] * qmq;
          Q[m][q] = sn[k] * qmp + c[k] * qmq;
        }
      }
    }
  }
  double w[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double l = A[tri(j, j)];
    w[j] = l > floor ? l : floor;
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) acc += Q[i][j] * w[j] * Q[k][j];
      A[tri(i, k)] = acc;
    }
}

// Is A - floor*I positive definite? (Cholesky in registers.) When it is,
// max(Lambda, floor) == Lambda and the projector is A itself up to rounding
// (a misclassification can only happen when an eigenvalue is within rounding
// of the floor, where clamping changes nothing measurable).
template <int K>
MG_DI bool shifted_pd(const double* A, double floor) {
  double L[TriN<K>::value];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double d = A[tri(j, j)] - floor;
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[tri(j, k)] * L[tri(j, k)];
    ok &= d > 0.0;
    const double r = d > 0.0 ? rsqrt(d) : 0.0;
    L[tri(j, j)] = d * r;
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double v = A[tri(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[tri(i, k)] * L[tri(j, k)];
      L[tri(i, j)] = v * r;
    }
  }
  return ok;
}

// One eigenvalue below the floor, from a start vector v0 with a non-positive
// shifted Rayleigh quotient: the start is refined by Rayleigh-Ritz on
// span{v0, A v0} (the smaller Ritz pair of the 2 x 2 projection), then
// Rayleigh-quotient iteration for (lambda, v), and
// P_f(A) = A + (f - lambda) v v^T. The error of this update is bounded by the
// eigenvector residual times |f - lambda| / gap <= 1 (the gap to the next
// eigenvalue is at least f - lambda), so it is as accurate as the full
// eigendecomposition. The shifted solves are LDL^T without pivoting (A - rho I
// is nearly semi-definite once rho approaches the lowest eigenvalue; a pivot
// that vanishes — rho an eigenvalue to working precision — is replaced by
// 2^-52 |A|_F, so the solve still returns the eigenvector to full precision).
// Convergence is judged on the true residual |A v - rho v|, so the solver's
// conditioning never reaches the result. Returns false (A untouched) unless
// the iteration converged below the floor and A + (s - lambda) v v^T - f I is
// positive definite for a large s, i.e. no other eigenvalue sits below the
// floor; the caller then falls back to Jacobi.
template <int K>
MG_DI bool psd_rank1_update(double* A, double floor, const double* v0) {
  double v[K], nrm = 0.0, fro2 = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) nrm += v0[i] * v0[i];
  if (!(nrm > 0.0) || !isfinite(nrm)) return false;
  nrm = rsqrt(nrm);
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = v0[i] * nrm;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) fro2 += (i == j ? 1.0 : 2.0) * A[tri(i, j)] * A[tri(i, j)];
  const double scale = ::sqrt(fro2);
  const double tiny = 0x1p-52 * scale;
  auto matvec = [&](const double* x, double* y) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) acc += A[i >= j ? tri(i, j) : tri(j, i)] * x[j];
      y[i] = acc;
    }
  };
  {  // Rayleigh-Ritz on span{v, A v}
    double w[K], u[K], au[K], a = 0.0, nu = 0.0;
    matvec(v, w);
#pragma unroll
    for (int i = 0; i < K; ++i) a += v[i] * w[i];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      u[i] = w[i] - a * v[i];
      nu += u[i] * u[i];
    }
    if (nu > 1e-28 * fro2) {
      const double inu = rsqrt(nu);
      nu *= inu;
#pragma unroll
      for (int i = 0; i < K; ++i) u[i] *= inu;
      matvec(u, au);
      double c = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) c += u[i] * au[i];
      const double h = 0.5 * (a - c);
      const double mu = 0.5 * (a + c) - ::sqrt(h * h + nu * nu);
      double n2 = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        v[i] = nu * v[i] + (mu - a) * u[i];
        n2 += v[i] * v[i];
      }
      if (!(n2 > 0.0)) return false;
      n2 = rsqrt(n2);
#pragma unroll
      for (int i = 0; i < K; ++i) v[i] *= n2;
    }
  }
  double rho = 0.0;
  bool conv = false;
  for (int it = 0; it < 8; ++it) {
    double w[K];
    matvec(v, w);
    rho = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) rho += v[i] * w[i];
    double res = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) res += (w[i] - rho * v[i]) * (w[i] - rho * v[i]);
    if (res <= 1e-28 * fro2) {
      conv = true;
      break;
    }
    // (A - rho I) y = v: LDL^T without pivoting
    double L[TriN<K>::value], D[K], y[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double d = A[tri(j, j)] - rho;
#pragma unroll
      for (int k = 0; k < j; ++k) d -= L[tri(j, k)] * L[tri(j, k)] * D[k];
      if (fabs(d) < tiny) d = d < 0.0 ? -tiny : tiny;
      D[j] = d;
      const double id = psd_rcp(d);
#pragma unroll
      for (int i = j + 1; i < K; ++i) {
        double t = A[tri(i, j)];
#pragma unroll
        for (int k = 0; k < j; ++k) t -= L[tri(i, k)] * L[tri(j, k)] * D[k];
        L[tri(i, j)] = t * id;
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double t = v[i];
#pragma unroll
      for (int k = 0; k < i; ++k) t -= L[tri(i, k)] * y[k];
      y[i] = t;
    }
#pragma unroll
    for (int i = 0; i < K; ++i) y[i] *= psd_rcp(D[i]);
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      double t = y[i];
#pragma unroll
      for (int k = i + 1; k < K; ++k) t -= L[tri(k, i)] * y[k];
      y[i] = t;
    }
    double yn = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) yn += y[i] * y[i];
    if (!(yn > 0.0) || !isfinite(yn)) return false;
    yn = rsqrt(yn);
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] = y[i] * yn;
  }
  if (!conv || !(rho < floor)) return false;
  // no other eigenvalue below the floor: lift v's eigenvalue out of the way and test
  double T[TriN<K>::value];
  const double lift = scale + floor - rho;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) T[tri(i, j)] = A[tri(i, j)] + lift * v[i] * v[j];
  if (!shifted_pd<K>(T, floor)) return false;
  const double d = floor - rho;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) A[tri(i, j)] += d * v[i] * v[j];
  return true;
}

// shifted_pd, and when A - floor*I is not positive definite a direction z of
// non-positive curvature: at the first failing pivot j, with the leading j x j
// block M = L L^T and column b above the pivot, z = [-M^{-1} b; 1; 0...] gives
// z^T (A - floor I) z = the Schur pivot <= 0 (M^{-1} b = L^{-T} l_j, l_j the
// factor's row j)
template <int K>
MG_DI bool shifted_pd_dir(const double* A, double floor, double* z) {
  double L[TriN<K>::value];
  int fail = -1;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double d = A[tri(j, j)] - floor;
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[tri(j, k)] * L[tri(j, k)];
    if (fail < 0 && !(d > 0.0)) fail = j;
    const double r = d > 0.0 ? rsqrt(d) : 0.0;
    L[tri(j, j)] = d * r;
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double v = A[tri(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[tri(i, k)] * L[tri(j, k)];
      L[tri(i, j)] = v * r;
    }
  }
  if (fail < 0) return true;
  double y[K];  // L11^T y = l_fail (back substitution over the leading fail x fail block)
#pragma unroll
  for (int i = K - 1; i >= 0; --i) {
    double rhs = 0.0;
#pragma unroll
    for (int c = i + 1; c < K; ++c)
      if (c == fail) rhs = L[tri(c, i)];
#pragma unroll
    for (int k = i + 1; k < K; ++k)
      if (k < fail) rhs -= L[tri(k, i)] * y[k];
    y[i] = i < fail ? rhs * psd_rcp(L[tri(i, i)]) : 0.0;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) z[i] = i < fail ? -y[i] : (i == fail ? 1.0 : 0.0);
  return false;
}

// project in place unless already above the floor; 2x2 / 3x3 blocks (vertex
// terms, two-point edge terms) use the non-iterative solver of psd_small.h.
// 4x4 / 6x6: one eigenvalue below the floor is the common case (e.g. the
// sphere face Hessian's one strongly negative mode, every face at the
// benchmark state): Rayleigh-quotient iteration from the Cholesky test's
// negative-curvature direction and a certified rank-one update; Jacobi when
// that fails (several eigenvalues below the floor, or no convergence)
template <int K>
MG_DI void project_if_needed(double* A, double floor) {
  if constexpr (K == 4 || K == 6) {
    double z[K];
    if (shifted_pd_dir<K>(A, floor, z)) return;
    if (!psd_rank1_update<K>(A, floor, z)) jacobi_project_rr<K>(A, floor);
    return;
  }
  if (shifted_pd<K>(A, floor)) return;
  if constexpr (K == 2) psd_small::project2(A, floor);
  else if constexpr (K == 3) psd_small::project3(A, floor);
  else jacobi_project<K>(A, floor);
}

template <int K>
MG_DI bool all_finite(const double* A) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < TriN<K>::value; ++i) ok &= isfinite(A[i]);
  return ok;
}

// `_extract` epilogue for a packed Hessian: symmetrise (identity on packed
// storage except for overflow, mirrored anyway) then clamp finite lanes.
// N: per-vertex block dim; P: vertices per element (K = P*N).
template <int P, int N>
MG_DI void extract_psd(double* H, double floor) {
  constexpr int K = P * N;
#pragma unroll
  for (int i = 0; i < TriN<K>::value; ++i) H[i] = 0.5 * (H[i] + H[i]);
  if (!all_finite<K>(H)) return;
  {
    // diagonal block (vertex terms such as inertia m I, or a structural-zero
    // Hessian): the eigenvalues are the diagonal entries on the coordinate
    // axes, so the clamp is elementwise and exact
    bool diag = true;
#pragma unroll
    for (int i = 1; i < K; ++i)
#pragma unroll
      for (int j = 0; j < i; ++j) diag &= H[tri(i, j)] == 0.0;
    if (diag) {
#pragma unroll
      for (int i = 0; i < K; ++i) H[tri(i, i)] = H[tri(i, i)] > floor ? H[tri(i, i)] : floor;
      return;
    }
  }
  if constexpr (P == 2) {
    // bitwise two-point structure test
    bool two = true;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        two &= H[tri(N + i, N + j)] == H[tri(i, j)];
        two &= H[tri(N + i, j)] == -H[tri(i, j)];
        if (i != j) two &= H[tri(N + j, i)] == -H[tri(i, j)];
      }
    if (two) {
      double A2[TriN<N>::value];
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) A2[tri(i, j)] = 2.0 * H[tri(i, j)];
      project_if_needed<N>(A2, floor);
      const double hf = 0.5 * floor;
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double p = 0.5 * A2[tri(i, j)];
          const double d = (i == j) ? hf : 0.0;
          if (j <= i) {
            H[tri(i, j)] = p + d;
            H[tri(N + i, N + j)] = p + d;
          }
          H[tri(N + i, j)] = -p + d;
        }
      return;
    }
  }
  project_if_needed<K>(H, floor);
}

}  // namespace mg
