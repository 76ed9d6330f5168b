// Closed-form-seeded spectral clamp for symmetric 2x2 and 3x3 matrices
// (host + device; the host build is exercised by tests/test_psd_small.py).
//
// project_psd (meshgrad/active.py:490-504) needs P = Q max(L, floor) Q^T.
// The projector is unique, so any accurate eigen-decomposition reproduces
// the reference; here it is built without iteration:
//
//  3x3: 1. fp32 trigonometric estimate of the most isolated extreme eigenvalue, polished by
//          one fp64 Newton step on det(A - l I) (simple roots -> full fp64);
//       2. its eigenvector = the largest column of adj(A - l I) (a cross
//          product of two rows), normalised; the isolated eigenvalue's gap is
//          >= half the spectral spread, so this vector is accurate;
//       3. an orthonormal completion (v1, v2) and the 2x2 block
//          B = [v1 v2]^T A [v1 v2], diagonalised exactly by one rotation.
//     The remaining pair may be clustered or degenerate; the exact 2x2
//     rotation handles that, and the neglected coupling u^T A v_k is
//     O(eps |A|), so the projector error stays O(eps |A|).
//  2x2: one exact rotation.
//
// Packed lower storage, index tri(i, j) = i (i + 1) / 2 + j for i >= j:
//   3x3: [a00, a10, a11, a20, a21, a22];  2x2: [a00, a10, a11].
#pragma once
#include <cmath>

#if defined(__CUDACC__)
#define PSD_HD __host__ __device__ __forceinline__
#else
#define PSD_HD inline
#endif

namespace mg {
namespace psd_small {

PSD_HD double dmax(double a, double b) { return a > b ? a : b; }

// exact 2x2 symmetric eigen-decomposition by one Jacobi rotation:
// returns (l1, l2) and rotation (c, s) with w1 = (c, -s), w2 = (s, c)
PSD_HD void eig2(double a, double b, double d, double& l1, double& l2, double& c, double& s) {
  if (b == 0.0) {
    l1 = a; l2 = d; c = 1.0; s = 0.0;
    return;
  }
  const double theta = (d - a) / (2.0 * b);
  const double t = (theta >= 0.0 ? 1.0 : -1.0) / (::fabs(theta) + ::sqrt(theta * theta + 1.0));
  c = 1.0 / ::sqrt(t * t + 1.0);
  s = t * c;
  l1 = a - t * b;
  l2 = d + t * b;
}

// 2x2: A (packed) -> Q max(L, f) Q^T in place
PSD_HD void project2(double* A, double f) {
  double l1, l2, c, s;
  eig2(A[0], A[1], A[2], l1, l2, c, s);
  l1 = dmax(l1, f);
  l2 = dmax(l2, f);
  // w1 = (c, -s), w2 = (s, c)
  A[0] = l1 * c * c + l2 * s * s;
  A[1] = -l1 * c * s + l2 * s * c;
  A[2] = l1 * s * s + l2 * c * c;
}

// 3x3: A (packed) -> Q max(L, f) Q^T in place. Caller guarantees finite A.
PSD_HD void project3(double* A, double f) {
  const double a00 = A[0], a10 = A[1], a11 = A[2], a20 = A[3], a21 = A[4], a22 = A[5];
  const double off2 = a10 * a10 + a20 * a20 + a21 * a21;
  const double q = (a00 + a11 + a22) / 3.0;
  const double d0 = a00 - q, d1 = a11 - q, d2 = a22 - q;
  const double p2 = d0 * d0 + d1 * d1 + d2 * d2 + 2.0 * off2;
  if (!(p2 > 0.0)) {  // A == q I
    const double m = dmax(q, f);
    A[0] = m; A[1] = 0.0; A[2] = m; A[3] = 0.0; A[4] = 0.0; A[5] = m;
    return;
  }
  const double pp = ::sqrt(p2 / 6.0);
  // r = det((A - qI)/p) / 2
  const double detB = d0 * (d1 * d2 - a21 * a21) - a10 * (a10 * d2 - a21 * a20) + a20 * (a10 * a21 - d1 * a20);
  double r = detB / (2.0 * pp * pp * pp);
  r = r < -1.0 ? -1.0 : (r > 1.0 ? 1.0 : r);
  const float phi = ::acosf((float)r) / 3.0f;
  // deflate with the more isolated extreme eigenvalue (its gap is at least
  // half the spread, so the adjugate vector below is well conditioned)
  const double ltop = q + 2.0 * pp * (double)::cosf(phi);
  const double lbot = q + 2.0 * pp * (double)::cosf(phi + 2.0943951023931953f);
  const double lmid = 3.0 * q - ltop - lbot;
  double lam = (ltop - lmid >= lmid - lbot) ? ltop : lbot;
  // one Newton step on the characteristic polynomial  g(l) = det(A - l I)
  {
    const double x0 = a00 - lam, x1 = a11 - lam, x2 = a22 - lam;
    const double g = x0 * (x1 * x2 - a21 * a21) - a10 * (a10 * x2 - a21 * a20) + a20 * (a10 * a21 - x1 * a20);
    const double dg = -((x1 * x2 - a21 * a21) + (x0 * x2 - a20 * a20) + (x0 * x1 - a10 * a10));
    if (dg != 0.0) {
      const double step = g / dg;
      if (::fabs(step) < 0.5 * pp) lam -= step;
    }
  }
  // top eigenvector: largest column of adj(A - lam I)
  const double x0 = a00 - lam, x1 = a11 - lam, x2 = a22 - lam;
  // rows: r0 = (x0, a10, a20), r1 = (a10, x1, a21), r2 = (a20, a21, x2)
  double c0x = a10 * a21 - a20 * x1, c0y = a20 * a10 - x0 * a21, c0z = x0 * x1 - a10 * a10;  // r0 x r1
  double c1x = a10 * x2 - a20 * a21, c1y = a20 * a20 - x0 * x2, c1z = x0 * a21 - a10 * a20;  // r0 x r2
  double c2x = x1 * x2 - a21 * a21, c2y = a21 * a20 - a10 * x2, c2z = a10 * a21 - x1 * a20;  // r1 x r2
  const double n0 = c0x * c0x + c0y * c0y + c0z * c0z;
  const double n1 = c1x * c1x + c1y * c1y + c1z * c1z;
  const double n2 = c2x * c2x + c2y * c2y + c2z * c2z;
  double ux, uy, uz, nn;
  if (n0 >= n1 && n0 >= n2) { ux = c0x; uy = c0y; uz = c0z; nn = n0; }
  else if (n1 >= n2) { ux = c1x; uy = c1y; uz = c1z; nn = n1; }
  else { ux = c2x; uy = c2y; uz = c2z; nn = n2; }
  if (!(nn > 0.0)) {  // lam hit an exact multiple root everywhere: any basis works
    ux = 1.0; uy = 0.0; uz = 0.0; nn = 1.0;
  }
  {
    const double inv = 1.0 / ::sqrt(nn);
    ux *= inv; uy *= inv; uz *= inv;
  }
  // orthonormal completion: v1 from the axis least aligned with u
  double v1x, v1y, v1z;
  {
    const double ax = ::fabs(ux), ay = ::fabs(uy), az = ::fabs(uz);
    if (ax <= ay && ax <= az) { v1x = 1.0 - ux * ux; v1y = -ux * uy; v1z = -ux * uz; }
    else if (ay <= az) { v1x = -uy * ux; v1y = 1.0 - uy * uy; v1z = -uy * uz; }
    else { v1x = -uz * ux; v1y = -uz * uy; v1z = 1.0 - uz * uz; }
    const double inv = 1.0 / ::sqrt(v1x * v1x + v1y * v1y + v1z * v1z);
    v1x *= inv; v1y *= inv; v1z *= inv;
  }
  const double v2x = uy * v1z - uz * v1y, v2y = uz * v1x - ux * v1z, v2z = ux * v1y - uy * v1x;
  // A v1, A v2, A u
  const double av1x = a00 * v1x + a10 * v1y + a20 * v1z, av1y = a10 * v1x + a11 * v1y + a21 * v1z,
               av1z = a20 * v1x + a21 * v1y + a22 * v1z;
  const double av2x = a00 * v2x + a10 * v2y + a20 * v2z, av2y = a10 * v2x + a11 * v2y + a21 * v2z,
               av2z = a20 * v2x + a21 * v2y + a22 * v2z;
  const double aux = a00 * ux + a10 * uy + a20 * uz, auy = a10 * ux + a11 * uy + a21 * uz,
               auz = a20 * ux + a21 * uy + a22 * uz;
  const double b11 = v1x * av1x + v1y * av1y + v1z * av1z;
  const double b12 = v1x * av2x + v1y * av2y + v1z * av2z;
  const double b22 = v2x * av2x + v2y * av2y + v2z * av2z;
  const double l3 = ux * aux + uy * auy + uz * auz;
  double l1, l2, c, s;
  eig2(b11, b12, b22, l1, l2, c, s);
  // w1 = c v1 - s v2, w2 = s v1 + c v2
  const double w1x = c * v1x - s * v2x, w1y = c * v1y - s * v2y, w1z = c * v1z - s * v2z;
  const double w2x = s * v1x + c * v2x, w2y = s * v1y + c * v2y, w2z = s * v1z + c * v2z;
  const double m1 = dmax(l1, f), m2 = dmax(l2, f), m3 = dmax(l3, f);
  A[0] = m1 * w1x * w1x + m2 * w2x * w2x + m3 * ux * ux;
  A[1] = m1 * w1y * w1x + m2 * w2y * w2x + m3 * uy * ux;
  A[2] = m1 * w1y * w1y + m2 * w2y * w2y + m3 * uy * uy;
  A[3] = m1 * w1z * w1x + m2 * w2z * w2x + m3 * uz * ux;
  A[4] = m1 * w1z * w1y + m2 * w2z * w2y + m3 * uz * uy;
  A[5] = m1 * w1z * w1z + m2 * w2z * w2z + m3 * uz * uz;
}

}  // namespace psd_small
}  // namespace mg
