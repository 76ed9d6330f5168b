// Deterministic accumulation for the element-parallel path (traced terms,
// problems the patch kernels do not cover): every element writes its slot
// vectors and Hessian blocks to scratch, then one thread per output row /
// block sums its contributions in a fixed (term, element) order — no atomics,
// bitwise reproducible like the reference's "deterministic" mode
// (problem.py:16-21, test_problem.py:360-369).
#include <cub/cub.cuh>

#include "mg_internal.cuh"

namespace mg {

namespace {

constexpr int TPB = 256;
inline unsigned grid_for(int64_t n) { return (unsigned)((n + TPB - 1) / TPB); }

// (row vertex, term, element) -> offset of the element's slot vector
__global__ void k_vec_keys(const int32_t* sel, int P, int64_t M, int t, int N, int64_t base, const uint8_t* fixed,
                           const uint8_t* owned, uint64_t* keys, int64_t* vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * P) return;
  const int64_t e = i / P;
  const int q = (int)(i % P);
  const int v = sel ? sel[e * P + q] : (int)e;
  const bool skip = (fixed && fixed[v]) || (owned && !owned[v]);
  keys[i] = skip ? ~0ull : (((uint64_t)v << 34) | ((uint64_t)t << 30) | (uint64_t)e);
  vals[i] = base + i * N;
}

// (block, term, element) -> offset of the element's (q1, q2) block
__global__ void k_blk_keys(const int32_t* bids, int P, int64_t M, int t, int NN, int64_t base, uint64_t* keys,
                           int64_t* vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * P * P) return;
  const int64_t e = i / (P * P);
  const int32_t b = bids[i];
  keys[i] = b < 0 ? ~0ull : (((uint64_t)b << 34) | ((uint64_t)t << 30) | (uint64_t)e);
  vals[i] = base + i * NN;
}

__global__ void k_bounds(const uint64_t* keys, int64_t n, int64_t rows, int64_t* off) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > rows) return;
  const uint64_t k = (uint64_t)r << 34;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  off[r] = lo;
}

template <int W>
__global__ void k_gather(const int64_t* off, const int64_t* idx, const double* scr, int64_t rows, double* out) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double acc[W];
#pragma unroll
  for (int i = 0; i < W; ++i) acc[i] = 0.0;
  for (int64_t k = off[r]; k < off[r + 1]; ++k) {
    const double* src = scr + idx[k];
#pragma unroll
    for (int i = 0; i < W; ++i) acc[i] += src[i];
  }
#pragma unroll
  for (int i = 0; i < W; ++i) out[r * W + i] = acc[i];
}

// any width (var_dim > 3: the reference accepts any var_dim, problem.py:263):
// one thread per output scalar, same fixed contribution order
__global__ void k_gather_n(const int64_t* off, const int64_t* idx, const double* scr, int64_t rows, int W,
                           double* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows * W) return;
  const int64_t r = t / W;
  const int i = (int)(t - r * W);
  double acc = 0.0;
  for (int64_t k = off[r]; k < off[r + 1]; ++k) acc += scr[idx[k] + i];
  out[t] = acc;
}

// sort (key, value) pairs and drop the ~0 keys; returns the kept count
int64_t sort_pairs(DBuf<uint64_t>& k, DBuf<int64_t>& v, int64_t n, cudaStream_t s) {
  if (n == 0) return 0;
  DBuf<uint64_t> k2;
  DBuf<int64_t> v2;
  k2.alloc(n);
  v2.alloc(n);
  size_t tb = 0;
  MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k.p, k2.p, v.p, v2.p, n, 0, 64, s));
  {
    Tmp t(s, tb);
    MG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, k.p, k2.p, v.p, v2.p, n, 0, 64, s));
  }
  MG_CUDA(cudaStreamSynchronize(s));
  k = std::move(k2);
  v = std::move(v2);
  // count kept: keys sorted, invalid (~0) last
  int64_t lo = 0, hi = n;
  while (lo < hi) {  // host binary search over device keys (log n small copies)
    const int64_t mid = (lo + hi) >> 1;
    uint64_t km = 0;
    MG_CUDA(cudaMemcpy(&km, k.p + mid, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (km == ~0ull) hi = mid; else lo = mid + 1;
  }
  return lo;
}

}  // namespace

void build_gather(Problem& p, cudaStream_t s) {
  const Mesh& m = *p.mesh;
  const int n = p.n;
  int64_t nv = 0, nh = 0, vtot = 0, htot = 0;
  for (auto& t : p.terms) {
    t.gv_base = vtot;
    t.gh_base = htot;
    vtot += t.M * t.dev.P * n;
    nv += t.M * t.dev.P;
    if (p.with_hessian) {
      htot += t.M * t.dev.P * t.dev.P * n * n;
      nh += t.M * t.dev.P * t.dev.P;
    }
  }
  p.gsv.alloc(vtot > 0 ? vtot : 1);
  p.gsh.alloc(htot > 0 ? htot : 1);
  {
    DBuf<uint64_t> keys;
    DBuf<int64_t> vals;
    keys.alloc(nv > 0 ? nv : 1);
    vals.alloc(nv > 0 ? nv : 1);
    int64_t o = 0;
    for (size_t ti = 0; ti < p.terms.size(); ++ti) {
      const Term& t = p.terms[ti];
      const int64_t cnt = t.M * t.dev.P;
      if (cnt)
        k_vec_keys<<<grid_for(cnt), TPB, 0, s>>>(term_sel(m, t), t.dev.P, t.M, (int)ti, n, t.gv_base,
                                                 p.any_fixed ? p.fixed.p : nullptr, m.owned.p, keys.p + o, vals.p + o);
      MG_LAUNCH_CHECK();
      o += cnt;
    }
    const int64_t kept = sort_pairs(keys, vals, nv, s);
    p.gv_off.alloc(m.V + 1);
    k_bounds<<<grid_for(m.V + 1), TPB, 0, s>>>(keys.p, kept, m.V, p.gv_off.p);
    MG_LAUNCH_CHECK();
    p.gv_idx = std::move(vals);
  }
  if (p.with_hessian && p.pattern_ready) {
    DBuf<uint64_t> keys;
    DBuf<int64_t> vals;
    keys.alloc(nh > 0 ? nh : 1);
    vals.alloc(nh > 0 ? nh : 1);
    int64_t o = 0;
    for (size_t ti = 0; ti < p.terms.size(); ++ti) {
      const Term& t = p.terms[ti];
      const int64_t cnt = t.M * t.dev.P * t.dev.P;
      if (cnt)
        k_blk_keys<<<grid_for(cnt), TPB, 0, s>>>(t.bids.p, t.dev.P, t.M, (int)ti, n * n, t.gh_base, keys.p + o,
                                                 vals.p + o);
      MG_LAUNCH_CHECK();
      o += cnt;
    }
    const int64_t kept = sort_pairs(keys, vals, nh, s);
    p.gh_off.alloc(p.nnzb + 1);
    k_bounds<<<grid_for(p.nnzb + 1), TPB, 0, s>>>(keys.p, kept, p.nnzb, p.gh_off.p);
    MG_LAUNCH_CHECK();
    p.gh_idx = std::move(vals);
  }
  MG_CUDA(cudaStreamSynchronize(s));
  p.gather_ready = true;
}

void gather_vec(const Problem& p, double* out, cudaStream_t s) {
  const int64_t V = p.mesh->V;
  if (!V) return;
  switch (p.n) {
    case 1: k_gather<1><<<grid_for(V), TPB, 0, s>>>(p.gv_off.p, p.gv_idx.p, p.gsv.p, V, out); break;
    case 2: k_gather<2><<<grid_for(V), TPB, 0, s>>>(p.gv_off.p, p.gv_idx.p, p.gsv.p, V, out); break;
    case 3: k_gather<3><<<grid_for(V), TPB, 0, s>>>(p.gv_off.p, p.gv_idx.p, p.gsv.p, V, out); break;
    default: k_gather_n<<<grid_for(V * p.n), TPB, 0, s>>>(p.gv_off.p, p.gv_idx.p, p.gsv.p, V, p.n, out);
  }
  MG_LAUNCH_CHECK();
}

void gather_blocks(const Problem& p, double* out, cudaStream_t s) {
  const int64_t nb = p.nnzb;
  if (!nb) return;
  switch (p.n) {
    case 1: k_gather<1><<<grid_for(nb), TPB, 0, s>>>(p.gh_off.p, p.gh_idx.p, p.gsh.p, nb, out); break;
    case 2: k_gather<4><<<grid_for(nb), TPB, 0, s>>>(p.gh_off.p, p.gh_idx.p, p.gsh.p, nb, out); break;
    case 3: k_gather<9><<<grid_for(nb), TPB, 0, s>>>(p.gh_off.p, p.gh_idx.p, p.gsh.p, nb, out); break;
    default:
      k_gather_n<<<grid_for(nb * p.n * p.n), TPB, 0, s>>>(p.gh_off.p, p.gh_idx.p, p.gsh.p, nb, p.n * p.n, out);
  }
  MG_LAUNCH_CHECK();
}

}  // namespace mg
