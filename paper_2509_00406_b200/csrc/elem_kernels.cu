// Element-parallel kernels: one thread per term element, dual numbers in
// registers, outputs scattered with fp64 atomics into caller-zeroed buffers.
// This is the reference's "atomic" accumulation mode (problem.py:16-21,
// 486-499): merge order is whatever the hardware gives, results agree with
// the deterministic path to rounding. The energy is reduced through fixed-
// order per-block partials so it is reproducible in every mode.
//
// Per-element pipeline (problem.py:526-544): lift (seeds) -> term_eval ->
// _extract (symmetrise, optional PSD clamp) -> scatter.
#include "mg_internal.cuh"
#include "psd.cuh"

namespace mg {

namespace {

constexpr int TPB = 128;

struct ElemArgs {
  const double* x;
  const double* w;
  const uint8_t* fixed;
  const uint8_t* owned;  // shard: energy of an element counts where its slot-0 vertex is owned
  const int32_t* sel;
  const int32_t* bids;
  double* grad;
  double* hess;
  double* y;
  double* partials;
  double floor;
  int64_t M;
  // deterministic mode off the patch path: per-element outputs go to scratch
  // ((M,P,N) vectors, (M,P,P,N,N) blocks) and a fixed-order gather sums them
  double* sv;
  double* sh;
};

// Fixed-order block sum (warp shuffle tree, then warp 0 over the warp sums).
__device__ double block_sum(double v) {
  __shared__ double ws[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    r = lane < nw ? ws[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// one slot component of an element's gradient / HVP output: scratch in the
// deterministic gather mode, fp64 atomic otherwise
MG_DI void put_vec(const ElemArgs& a, double* out, int64_t e, int P, int q, int N, int c, int v, double val) {
  if (a.sv) a.sv[(e * P + q) * N + c] = val;
  else atomicAdd(out + (int64_t)v * N + c, val);
}

template <int P, int N, int K, class H>
__device__ __forceinline__ void scatter_hess(const ElemArgs& a, int64_t e, const double* h) {
  const int32_t* b = a.bids + e * P * P;
#pragma unroll
  for (int q1 = 0; q1 < P; ++q1)
#pragma unroll
    for (int q2 = 0; q2 < P; ++q2) {
      const int32_t bid = b[q1 * P + q2];
      if (bid >= 0) {
        if (a.sh) {
          double* dst = a.sh + ((e * P + q1) * P + q2) * N * N;
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int c = 0; c < N; ++c) dst[r * N + c] = h ? h[tri(q1 * N + r, q2 * N + c)] : 0.0;
        } else if (h) {
          double* dst = a.hess + (int64_t)bid * N * N;
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int c = 0; c < N; ++c) atomicAdd(dst + r * N + c, h[tri(q1 * N + r, q2 * N + c)]);
        }
      }
    }
}

template <int TT, int N, int MODE, bool PSD>
__global__ void __launch_bounds__(TPB) k_elem(TermDev t, ElemArgs a) {
  constexpr int P = TermInfo<TT>::P;
  constexpr int K = P * N;
  const int64_t e = blockIdx.x * (int64_t)TPB + threadIdx.x;
  double ev = 0.0;
  if (e < a.M) {
    int vid[P];
#pragma unroll
    for (int q = 0; q < P; ++q) vid[q] = a.sel ? a.sel[e * P + q] : (int)e;
    bool fr[P];
#pragma unroll
    for (int q = 0; q < P; ++q) fr[q] = !a.fixed || !a.fixed[vid[q]];

    if constexpr (MODE == MODE_ENERGY) {
      Vec<Dv<K>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) X[q][c].v = a.x[(int64_t)vid[q] * N + c];
      ev = term_eval<TT, N>(t, e, vid, X).v;
    } else if constexpr (MODE == MODE_GRAD) {
      Vec<Dg<K>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          X[q][c].v = a.x[(int64_t)vid[q] * N + c];
#pragma unroll
          for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c) ? 1.0 : 0.0;
        }
      auto r = term_eval<TT, N>(t, e, vid, X);
      ev = r.v;
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (fr[q])
#pragma unroll
          for (int c = 0; c < N; ++c) put_vec(a, a.grad, e, P, q, N, c, vid[q], r.g[q * N + c]);
    } else if constexpr (MODE == MODE_HESS || (MODE == MODE_HVP && PSD)) {
      Vec<Dh<K, true>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          X[q][c].v = a.x[(int64_t)vid[q] * N + c];
#pragma unroll
          for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c) ? 1.0 : 0.0;
        }
      auto r = term_eval<TT, N>(t, e, vid, X);
      using R = decltype(r);
      ev = r.v;
      if constexpr (MODE == MODE_HESS) {
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (fr[q])
#pragma unroll
            for (int c = 0; c < N; ++c) put_vec(a, a.grad, e, P, q, N, c, vid[q], r.g[q * N + c]);
      }
      // _extract (problem.py:454-476): structural zero -> no Hessian unless
      // a PSD floor is requested (then project(0) = floor*I).
      if constexpr (!R::kZero || PSD) {
        double h[TriN<K>::value];
        if constexpr (R::kZero) {
#pragma unroll
          for (int i = 0; i < TriN<K>::value; ++i) h[i] = 0.0;
        } else {
#pragma unroll
          for (int i = 0; i < TriN<K>::value; ++i) h[i] = r.h[i];
        }
        if constexpr (PSD) {
          // pinned variables are seeded passively by the reference: zero
          // their rows/cols before the clamp so the free block projects alone
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (!fr[q])
#pragma unroll
              for (int c = 0; c < N; ++c)
#pragma unroll
                for (int j = 0; j < K; ++j) h[tri(q * N + c, j)] = 0.0;
          extract_psd<P, N>(h, a.floor);
        } else {
#pragma unroll
          for (int i = 0; i < TriN<K>::value; ++i) h[i] = 0.5 * (h[i] + h[i]);
        }
        if constexpr (MODE == MODE_HESS) {
          scatter_hess<P, N, K, R>(a, e, h);
        } else {
          double vl[K];
#pragma unroll
          for (int q = 0; q < P; ++q)
#pragma unroll
            for (int c = 0; c < N; ++c) vl[q * N + c] = fr[q] ? a.w[(int64_t)vid[q] * N + c] : 0.0;
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (fr[q])
#pragma unroll
              for (int c = 0; c < N; ++c) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < K; ++j) acc += h[tri(q * N + c, j)] * vl[j];
                put_vec(a, a.y, e, P, q, N, c, vid[q], acc);
              }
        }
      } else if constexpr (MODE == MODE_HESS) {
        if (a.sh) scatter_hess<P, N, K, R>(a, e, nullptr);  // structural zero: zero blocks for the gather
      }
    } else {  // MODE_HVP, no PSD: forward-over-forward dual, H never formed
      Vec<Df<K, true>, N> X[P];
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          X[q][c].v = a.x[(int64_t)vid[q] * N + c];
          X[q][c].vd = fr[q] ? a.w[(int64_t)vid[q] * N + c] : 0.0;
#pragma unroll
          for (int i = 0; i < K; ++i) X[q][c].g[i] = (i == q * N + c) ? 1.0 : 0.0;
        }
      auto r = term_eval<TT, N>(t, e, vid, X);
      using R = decltype(r);
      if constexpr (!R::kZero) {
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (fr[q])
#pragma unroll
            for (int c = 0; c < N; ++c) put_vec(a, a.y, e, P, q, N, c, vid[q], r.gd[q * N + c]);
      } else if (a.sv) {
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
          for (int c = 0; c < N; ++c) a.sv[(e * P + q) * N + c] = 0.0;
      }
    }
  }
  if constexpr (MODE != MODE_HVP) {
    if (a.owned && e < a.M && !a.owned[a.sel ? a.sel[e * P] : e]) ev = 0.0;
    const double s = block_sum(ev);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = s;
  }
}

template <int TT, int N>
void launch_tn(const Term& t, Mode mode, bool psd, const ElemArgs& a, cudaStream_t s) {
  const unsigned grid = (unsigned)((a.M + TPB - 1) / TPB);
  switch (mode) {
    case MODE_ENERGY: k_elem<TT, N, MODE_ENERGY, false><<<grid, TPB, 0, s>>>(t.dev, a); break;
    case MODE_GRAD: k_elem<TT, N, MODE_GRAD, false><<<grid, TPB, 0, s>>>(t.dev, a); break;
    case MODE_HESS:
      if (psd) k_elem<TT, N, MODE_HESS, true><<<grid, TPB, 0, s>>>(t.dev, a);
      else k_elem<TT, N, MODE_HESS, false><<<grid, TPB, 0, s>>>(t.dev, a);
      break;
    case MODE_HVP:
      if (psd) k_elem<TT, N, MODE_HVP, true><<<grid, TPB, 0, s>>>(t.dev, a);
      else k_elem<TT, N, MODE_HVP, false><<<grid, TPB, 0, s>>>(t.dev, a);
      break;
  }
  MG_LAUNCH_CHECK();
}

template <int TT>
void launch_t(int n, const Term& t, Mode mode, bool psd, const ElemArgs& a, cudaStream_t s) {
  if constexpr (TT == MG_TERM_SYM_DIRICHLET || TT == MG_TERM_SPHERE) {
    if (n != 2) throw Error(MG_ERR_VALUE, "term requires var_dim == 2");
    launch_tn<TT, 2>(t, mode, psd, a, s);
  } else {
    if (n == 3) launch_tn<TT, 3>(t, mode, psd, a, s);
    else if (n == 2) launch_tn<TT, 2>(t, mode, psd, a, s);
    else throw Error(MG_ERR_UNSUPPORTED, "builtin vertex/edge terms support var_dim 2 or 3");
  }
}

// Fixed-order sum of the energy partials: thread t sums the strided set
// t, t+B, t+2B, ... (coalesced) into 4 independent accumulators (memory-level
// parallelism), combined in a fixed order; then the block tree.
__global__ void __launch_bounds__(1024) k_reduce(const double* __restrict__ partials, int64_t n, double* out,
                                                 int* clear_flag) {
  const int64_t B = blockDim.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t i = threadIdx.x;
  for (; i + 3 * B < n; i += 4 * B) {
    a0 += partials[i];
    a1 += partials[i + B];
    a2 += partials[i + 2 * B];
    a3 += partials[i + 3 * B];
  }
  for (; i < n; i += B) a0 += partials[i];
  const double s = block_sum((a0 + a1) + (a2 + a3));
  if (threadIdx.x == 0) {
    out[0] = s;
    if (clear_flag) *clear_flag = 0;
  }
}

// stage 1 of the two-level fixed-order energy sum: CTA b sums the chunk
// [b C, (b+1) C) (thread t: t, t+256, ...; then the block tree) -> out[b]
constexpr int RED_CHUNK = 2048;
__global__ void __launch_bounds__(256) k_reduce_chunks(const double* __restrict__ partials, int64_t n, double* out) {
  const int64_t base = (int64_t)blockIdx.x * RED_CHUNK;
  double acc[RED_CHUNK / 256];
#pragma unroll
  for (int k = 0; k < RED_CHUNK / 256; ++k) {
    const int64_t i = base + threadIdx.x + (int64_t)k * 256;
    acc[k] = i < n ? partials[i] : 0.0;
  }
#pragma unroll
  for (int w = RED_CHUNK / 512; w > 0; w >>= 1)
#pragma unroll
    for (int k = 0; k < w; ++k) acc[k] += acc[k + w];
  const double s = block_sum(acc[0]);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

template <int N>
__global__ void k_bsr_matvec(const int64_t* ro, const int32_t* col, const double* H, const double* v,
                             double* y, int64_t V) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  double acc[N];
#pragma unroll
  for (int r = 0; r < N; ++r) acc[r] = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    const double* b = H + k * N * N;
    const double* vv = v + (int64_t)col[k] * N;
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) acc[r] += b[r * N + c] * vv[c];
  }
#pragma unroll
  for (int r = 0; r < N; ++r) y[i * N + r] = acc[r];
}

// Block-Jacobi preconditioner (BlockSparseMatrix.diagonal_block_inverses,
// problem.py:118-131; solvers.py:178-186): the inverse of every row's
// diagonal block, identity where a row has none or the block is singular.
template <int N>
__global__ void k_block_jacobi_inv(const int64_t* ro, const int32_t* col, const double* H, int64_t V, double* inv) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= V) return;
  double* out = inv + v * N * N;
  int64_t lo = ro[v], hi = ro[v + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] < v) lo = mid + 1; else hi = mid;
  }
  bool ok = lo < ro[v + 1] && col[lo] == v;
  double a[N * N];
  if (ok)
#pragma unroll
    for (int i = 0; i < N * N; ++i) a[i] = H[lo * N * N + i];
  double r[N * N];
  if (ok) {
    if constexpr (N == 1) {
      ok = a[0] != 0.0;
      r[0] = 1.0 / a[0];
    } else if constexpr (N == 2) {
      const double det = a[0] * a[3] - a[1] * a[2];
      ok = det != 0.0;
      const double id = 1.0 / det;
      r[0] = a[3] * id; r[1] = -a[1] * id; r[2] = -a[2] * id; r[3] = a[0] * id;
    } else {
      const double c00 = a[4] * a[8] - a[5] * a[7], c01 = a[5] * a[6] - a[3] * a[8], c02 = a[3] * a[7] - a[4] * a[6];
      const double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
      ok = det != 0.0;
      const double id = 1.0 / det;
      r[0] = c00 * id; r[1] = (a[2] * a[7] - a[1] * a[8]) * id; r[2] = (a[1] * a[5] - a[2] * a[4]) * id;
      r[3] = c01 * id; r[4] = (a[0] * a[8] - a[2] * a[6]) * id; r[5] = (a[2] * a[3] - a[0] * a[5]) * id;
      r[6] = c02 * id; r[7] = (a[1] * a[6] - a[0] * a[7]) * id; r[8] = (a[0] * a[4] - a[1] * a[3]) * id;
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) out[i * N + j] = ok ? r[i * N + j] : (i == j ? 1.0 : 0.0);
}

template <int N>
__global__ void k_block_apply(const double* inv, const double* r, double* y, int64_t V) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= V) return;
  const double* m = inv + v * N * N;
  double rv[N];
#pragma unroll
  for (int j = 0; j < N; ++j) rv[j] = r[v * N + j];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) acc += m[i * N + j] * rv[j];
    y[v * N + i] = acc;
  }
}

// Any block dim n (traced terms accept var_dim > 3, problem.py:263): one
// thread per scalar row for the SpMV / apply; Gauss-Jordan with partial
// pivoting for the diagonal-block inverse (identity on an exactly zero
// pivot, where numpy.linalg.inv raises and the reference falls back).
__global__ void k_bsr_matvec_n(const int64_t* ro, const int32_t* col, const double* H, const double* v,
                               double* y, int64_t V, int n) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= V * n) return;
  const int64_t i = t / n;
  const int r = (int)(t - i * n);
  double acc = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    const double* b = H + (k * n + r) * n;
    const double* vv = v + (int64_t)col[k] * n;
    for (int c = 0; c < n; ++c) acc += b[c] * vv[c];
  }
  y[t] = acc;
}

__global__ void k_block_jacobi_inv_n(const int64_t* ro, const int32_t* col, const double* H, int64_t V, int n,
                                     double* a_scratch, double* inv) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int64_t nn = (int64_t)n * n;
  double* out = inv + v * nn;
  double* a = a_scratch + v * nn;
  int64_t lo = ro[v], hi = ro[v + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] < v) lo = mid + 1; else hi = mid;
  }
  bool ok = lo < ro[v + 1] && col[lo] == v;
  for (int64_t i = 0; i < nn; ++i) {
    a[i] = ok ? H[lo * nn + i] : 0.0;
    out[i] = (i / n == i % n) ? 1.0 : 0.0;
  }
  for (int c = 0; ok && c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (fabs(a[r * n + c]) > fabs(a[piv * n + c])) piv = r;
    if (a[piv * n + c] == 0.0) { ok = false; break; }
    if (piv != c)
      for (int j = 0; j < n; ++j) {
        double t = a[c * n + j]; a[c * n + j] = a[piv * n + j]; a[piv * n + j] = t;
        t = out[c * n + j]; out[c * n + j] = out[piv * n + j]; out[piv * n + j] = t;
      }
    const double d = 1.0 / a[c * n + c];
    for (int j = 0; j < n; ++j) { a[c * n + j] *= d; out[c * n + j] *= d; }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = a[r * n + c];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) { a[r * n + j] -= f * a[c * n + j]; out[r * n + j] -= f * out[c * n + j]; }
    }
  }
  if (!ok)
    for (int64_t i = 0; i < nn; ++i) out[i] = (i / n == i % n) ? 1.0 : 0.0;
}

__global__ void k_block_apply_n(const double* inv, const double* r, double* y, int64_t V, int n) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= V * n) return;
  const int64_t v = t / n;
  const int i = (int)(t - v * n);
  const double* m = inv + (v * n + i) * n;
  double acc = 0.0;
  for (int j = 0; j < n; ++j) acc += m[j] * r[v * n + j];
  y[t] = acc;
}

}  // namespace

void launch_block_jacobi(const Problem& p, const double* H, double* inv, cudaStream_t s) {
  const int64_t V = p.mesh->V;
  const unsigned grid = (unsigned)((V + 255) / 256);
  if (!V) return;
  switch (p.n) {
    case 1: k_block_jacobi_inv<1><<<grid, 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, V, inv); break;
    case 2: k_block_jacobi_inv<2><<<grid, 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, V, inv); break;
    case 3: k_block_jacobi_inv<3><<<grid, 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, V, inv); break;
    default: {
      // elimination scratch, stream-ordered (freed after the kernel on the same stream)
      double* a = nullptr;
      MG_CUDA(cudaMallocAsync(&a, sizeof(double) * V * p.n * p.n, s));
      k_block_jacobi_inv_n<<<grid, 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, V, p.n, a, inv);
      MG_LAUNCH_CHECK();
      MG_CUDA(cudaFreeAsync(a, s));
    }
  }
  MG_LAUNCH_CHECK();
}

void launch_block_apply(const Problem& p, const double* inv, const double* r, double* y, cudaStream_t s) {
  const int64_t V = p.mesh->V;
  const unsigned grid = (unsigned)((V + 255) / 256);
  if (!V) return;
  switch (p.n) {
    case 1: k_block_apply<1><<<grid, 256, 0, s>>>(inv, r, y, V); break;
    case 2: k_block_apply<2><<<grid, 256, 0, s>>>(inv, r, y, V); break;
    case 3: k_block_apply<3><<<grid, 256, 0, s>>>(inv, r, y, V); break;
    default:
      k_block_apply_n<<<(unsigned)((V * p.n + 255) / 256), 256, 0, s>>>(inv, r, y, V, p.n);
  }
  MG_LAUNCH_CHECK();
}

int64_t elem_partials_needed(const Term& t) { return (t.M + TPB - 1) / TPB; }

int64_t launch_elem(const Problem& p, const Term& t, Mode mode, const LaunchCtx& c,
                    int64_t partial_offset) {
  if (t.M == 0) return 0;
  if (t.jit) {
    jit_launch(p, t, mode, c, partial_offset);
    return mode == MODE_HVP ? 0 : elem_partials_needed(t);
  }
  ElemArgs a;
  a.x = c.x;
  a.w = c.w;
  a.fixed = p.any_fixed ? p.fixed.p : nullptr;
  a.owned = p.mesh->owned.p;
  a.sel = term_sel(*p.mesh, t);
  a.bids = t.bids.p;
  a.grad = c.grad;
  a.hess = c.hess;
  a.y = c.y;
  a.partials = c.partials + partial_offset;
  a.floor = c.floor;
  a.M = t.M;
  a.sv = c.scratch ? p.gsv.p + t.gv_base : nullptr;
  a.sh = c.scratch && mode == MODE_HESS ? p.gsh.p + t.gh_base : nullptr;
  switch (t.dev.type) {
    case MG_TERM_INERTIA: launch_t<MG_TERM_INERTIA>(p.n, t, mode, c.psd, a, c.stream); break;
    case MG_TERM_SPRING: launch_t<MG_TERM_SPRING>(p.n, t, mode, c.psd, a, c.stream); break;
    case MG_TERM_GRAVITY: launch_t<MG_TERM_GRAVITY>(p.n, t, mode, c.psd, a, c.stream); break;
    case MG_TERM_EDGE_LENGTH: launch_t<MG_TERM_EDGE_LENGTH>(p.n, t, mode, c.psd, a, c.stream); break;
    case MG_TERM_SYM_DIRICHLET: launch_t<MG_TERM_SYM_DIRICHLET>(p.n, t, mode, c.psd, a, c.stream); break;
    case MG_TERM_SPHERE: launch_t<MG_TERM_SPHERE>(p.n, t, mode, c.psd, a, c.stream); break;
    default: throw Error(MG_ERR_VALUE, "unknown term type");
  }
  return mode == MODE_HVP ? 0 : elem_partials_needed(t);
}

void reduce_partials(const double* partials, int64_t n, double* out, cudaStream_t s, int* clear_flag) {
  if (n > 4 * RED_CHUNK) {
    // chunk sums land right after the partials (the buffer carries REDUCE_TAIL spare slots)
    const int64_t nb = (n + RED_CHUNK - 1) / RED_CHUNK;
    if (nb > REDUCE_TAIL) throw Error(MG_ERR_UNSUPPORTED, "too many energy partials");
    double* tmp = const_cast<double*>(partials) + n;
    k_reduce_chunks<<<(unsigned)nb, 256, 0, s>>>(partials, n, tmp);
    MG_LAUNCH_CHECK();
    k_reduce<<<1, 1024, 0, s>>>(tmp, nb, out, clear_flag);
  } else {
    k_reduce<<<1, 1024, 0, s>>>(partials, n, out, clear_flag);
  }
  MG_LAUNCH_CHECK();
}

void launch_bsr_matvec(const Problem& p, const double* H, const double* v, double* y, cudaStream_t s) {
  const int64_t V = p.mesh->V;
  const unsigned grid = (unsigned)((V + 255) / 256);
  switch (p.n) {
    case 1: k_bsr_matvec<1><<<grid, 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, v, y, V); break;
    case 2: k_bsr_matvec<2><<<grid, 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, v, y, V); break;
    case 3: k_bsr_matvec<3><<<grid, 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, v, y, V); break;
    default:
      k_bsr_matvec_n<<<(unsigned)((V * p.n + 255) / 256), 256, 0, s>>>(p.row_offsets.p, p.col32.p, H, v, y, V,
                                                                       p.n);
  }
  MG_LAUNCH_CHECK();
}

}  // namespace mg
