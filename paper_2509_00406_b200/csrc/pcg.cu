// Truncated, block-Jacobi preconditioned CG on the device, the inner solver of
// the device Newton drivers (reference solvers.py:142-175 cg_linear_solve,
// used by newton_solve (:244-263) on the assembled Hessian and newton_cg_solve
// (:266-287) on Hessian-vector products).
//
// The reference's decisions (curvature sign, alpha, convergence, beta) read
// scalars; here every scalar stays on the device: each iteration is a fixed
// sequence of launches (operator apply with the p.Ap partials, a one-CTA
// reduction that decides, the x / r / z update with the r.r and r.z partials,
// a one-CTA reduction that decides, the p update), every launch after a
// decision reads a device status word and returns at once once the solve has
// stopped. The host waits once per CHECK_EVERY iterations instead of three
// times per iteration. Dot products are fixed-order (a fixed grid of
// grid-stride blocks, then one CTA): bitwise reproducible.
#include <functional>

#include "mg_internal.cuh"

namespace mg {
namespace {

constexpr int VB = 256;           // threads per vector block
constexpr int VG = 4 * 148;       // vector blocks (fixed: the reduction order does not depend on the device)
constexpr int CHECK_EVERY = 8;    // iterations between host checks of the status word
// (an 8-lanes-per-row SpMV with coalesced block reads measured 2x slower than
// one thread per row: 1.65 vs 0.80 ms per iteration on the 2048^2 cloth)
enum { RUN = 0, CONVERGED = 1, NEGATIVE = 2, MAXITER = 3 };

struct PcgState {
  double bnorm;      // |b|
  double rz, pap, alpha, beta, rr;
  int status, it, progressed, pad;
};

__device__ __forceinline__ double block_reduce(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < VB / 32; ++i) r += sh[i];
  __syncthreads();
  return r;
}

// r = b, z = M r, p = z, x = 0; partials of b.b and r.z
__global__ void __launch_bounds__(VB) k_pcg_init(const double* b, const double* inv, int n, int64_t V, double* x,
                                                 double* r, double* z, double* p, double* part) {
  __shared__ double sh[VB / 32];
  double bb = 0.0, rz = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)VB + threadIdx.x; v < V; v += (int64_t)VG * VB) {
    for (int i = 0; i < n; ++i) {
      const double bi = b[v * n + i];
      r[v * n + i] = bi;
      x[v * n + i] = 0.0;
      bb += bi * bi;
    }
    for (int i = 0; i < n; ++i) {
      double zi = b[v * n + i];
      if (inv) {
        zi = 0.0;
        for (int j = 0; j < n; ++j) zi += inv[(v * n + i) * n + j] * b[v * n + j];
      }
      z[v * n + i] = zi;
      p[v * n + i] = zi;
      rz += b[v * n + i] * zi;
    }
  }
  const double s0 = block_reduce(bb, sh), s1 = block_reduce(rz, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[VG + blockIdx.x] = s1;
  }
}

__device__ __forceinline__ double sum_parts(const double* part, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < VG; i += VB) v += part[i];  // fixed per-thread order
  return block_reduce(v, sh);
}

__global__ void __launch_bounds__(VB) k_pcg_start(const double* part, PcgState* st, int max_iters) {
  __shared__ double sh[VB / 32];
  const double bb = sum_parts(part, sh), rz = sum_parts(part + VG, sh);
  if (threadIdx.x == 0) {
    st->bnorm = ::sqrt(bb);
    st->rz = rz;
    st->it = 0;
    st->progressed = 0;
    st->status = (bb == 0.0) ? CONVERGED : (max_iters < 1 ? MAXITER : RUN);
  }
}

// y = H p (assembled BSR) with the partials of p.y
template <int N>
__global__ void __launch_bounds__(VB) k_pcg_spmv(const int64_t* ro, const int32_t* col, const double* H,
                                                 const double* p, double* y, int64_t V, double* part,
                                                 const PcgState* st) {
  __shared__ double sh[VB / 32];
  if (st->status != RUN) return;
  double acc_dot = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VB + threadIdx.x; i < V; i += (int64_t)VG * VB) {
    double acc[N];
#pragma unroll
    for (int r = 0; r < N; ++r) acc[r] = 0.0;
    for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
      const double* b = H + k * N * N;
      const double* vv = p + (int64_t)col[k] * N;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) acc[r] += b[r * N + c] * vv[c];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      y[i * N + r] = acc[r];
      acc_dot += p[i * N + r] * acc[r];
    }
  }
  const double s = block_reduce(acc_dot, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// partials of p.y (matrix-free operator: y came from the HVP kernels)
__global__ void __launch_bounds__(VB) k_pcg_dot(const double* p, const double* y, int64_t nd, double* part,
                                                const PcgState* st) {
  __shared__ double sh[VB / 32];
  if (st->status != RUN) return;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VB + threadIdx.x; i < nd; i += (int64_t)VG * VB) acc += p[i] * y[i];
  const double s = block_reduce(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// pap; non-positive curvature stops the solve (solvers.py:158-161), else alpha
__global__ void __launch_bounds__(VB) k_pcg_curv(const double* part, PcgState* st) {
  __shared__ double sh[VB / 32];
  if (st->status != RUN) return;
  const double pap = sum_parts(part, sh);
  if (threadIdx.x == 0) {
    st->it += 1;
    st->pap = pap;
    if (pap <= 0.0) {
      st->status = NEGATIVE;
    } else {
      st->alpha = st->rz / pap;
      if (st->alpha != 0.0) st->progressed = 1;
    }
  }
}

// x += alpha p, r -= alpha y, z = M r; partials of r.r and r.z
__global__ void __launch_bounds__(VB) k_pcg_update(const double* p, const double* y, const double* inv, int n,
                                                   int64_t V, double* x, double* r, double* z, double* part,
                                                   const PcgState* st) {
  __shared__ double sh[VB / 32];
  if (st->status != RUN) return;
  const double alpha = st->alpha;
  double rr = 0.0, rz = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)VB + threadIdx.x; v < V; v += (int64_t)VG * VB) {
    double rv[8];
    for (int i = 0; i < n; ++i) {
      const int64_t k = v * n + i;
      x[k] += alpha * p[k];
      const double ri = r[k] - alpha * y[k];
      r[k] = ri;
      if (i < 8) rv[i] = ri;
      rr += ri * ri;
    }
    for (int i = 0; i < n; ++i) {
      const int64_t k = v * n + i;
      double zi = i < 8 ? rv[i] : r[k];
      if (inv) {
        zi = 0.0;
        for (int j = 0; j < n; ++j) zi += inv[(v * n + i) * n + j] * (j < 8 ? rv[j] : r[v * n + j]);
      }
      z[k] = zi;
      rz += (i < 8 ? rv[i] : r[k]) * zi;
    }
  }
  const double s0 = block_reduce(rr, sh), s1 = block_reduce(rz, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[VG + blockIdx.x] = s1;
  }
}

// |r| <= tol |b| stops the solve (solvers.py:166-167); else beta = rz'/rz
__global__ void __launch_bounds__(VB) k_pcg_conv(const double* part, PcgState* st, double tol, int max_iters) {
  __shared__ double sh[VB / 32];
  if (st->status != RUN) return;
  const double rr = sum_parts(part, sh), rz = sum_parts(part + VG, sh);
  if (threadIdx.x == 0) {
    st->rr = rr;
    if (::sqrt(rr) <= tol * st->bnorm) {
      st->status = CONVERGED;
    } else {
      st->beta = rz / st->rz;
      st->rz = rz;
      if (st->it >= max_iters) st->status = MAXITER;
    }
  }
}

// p = z + beta p
__global__ void __launch_bounds__(VB) k_pcg_p(const double* z, double* p, int64_t nd, const PcgState* st) {
  if (st->status != RUN) return;
  const double beta = st->beta;
  for (int64_t i = blockIdx.x * (int64_t)VB + threadIdx.x; i < nd; i += (int64_t)VG * VB) p[i] = z[i] + beta * p[i];
}

}  // namespace

// The solve (see the header). apply_hvp(v, y): y = H v for the matrix-free
// operator (hess null). Returns the iterations and the status word.
void pcg_solve(Problem& p, const double* hess, const std::function<void(const double*, double*)>& apply_hvp,
               const double* inv, const double* b, double tol, int max_iters, double* out, int* iters,
               int* status, cudaStream_t s) {
  if (hess && !p.pattern_ready) throw Error(MG_ERR_STATE, "sparsity pattern not computed");
  const int n = p.n;
  const int64_t V = p.mesh->V, nd = V * n;
  // workspace: r, z, p, y, partials, state
  const int64_t need = 4 * nd + 2 * VG + (int64_t)(sizeof(PcgState) + 7) / 8 + 1;
  if (p.pcg_ws.n < need) p.pcg_ws.alloc(need);
  double* r = p.pcg_ws.p;
  double* z = r + nd;
  double* pv = z + nd;
  double* y = pv + nd;
  double* part = y + nd;
  PcgState* st = reinterpret_cast<PcgState*>(part + 2 * VG);
  k_pcg_init<<<VG, VB, 0, s>>>(b, inv, n, V, out, r, z, pv, part);
  k_pcg_start<<<1, VB, 0, s>>>(part, st, max_iters);
  MG_LAUNCH_CHECK();
  PcgState h{};
  for (int it = 1; it <= max_iters; ++it) {
    if (hess && n >= 1 && n <= 3) {
      if (n == 1) k_pcg_spmv<1><<<VG, VB, 0, s>>>(p.row_offsets.p, p.col32.p, hess, pv, y, V, part, st);
      else if (n == 2) k_pcg_spmv<2><<<VG, VB, 0, s>>>(p.row_offsets.p, p.col32.p, hess, pv, y, V, part, st);
      else k_pcg_spmv<3><<<VG, VB, 0, s>>>(p.row_offsets.p, p.col32.p, hess, pv, y, V, part, st);
    } else {
      if (hess) launch_bsr_matvec(p, hess, pv, y, s);
      else apply_hvp(pv, y);
      k_pcg_dot<<<VG, VB, 0, s>>>(pv, y, nd, part, st);
    }
    k_pcg_curv<<<1, VB, 0, s>>>(part, st);
    k_pcg_update<<<VG, VB, 0, s>>>(pv, y, inv, n, V, out, r, z, part, st);
    k_pcg_conv<<<1, VB, 0, s>>>(part, st, tol, max_iters);
    k_pcg_p<<<VG, VB, 0, s>>>(z, pv, nd, st);
    MG_LAUNCH_CHECK();
    if (it % CHECK_EVERY == 0 || it == max_iters) {
      MG_CUDA(cudaMemcpyAsync(&h, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      if (h.status != RUN) break;
    }
  }
  // non-positive curvature before any progress: the reference returns b
  if (h.status == NEGATIVE && h.it == 1 && !h.progressed)
    MG_CUDA(cudaMemcpyAsync(out, b, sizeof(double) * nd, cudaMemcpyDeviceToDevice, s));
  *iters = h.it;
  *status = h.status;
}

}  // namespace mg
