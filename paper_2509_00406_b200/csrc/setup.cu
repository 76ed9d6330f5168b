// Setup path (runs once per mesh / problem; excluded from timed regions as in
// the reference, apps/smooth.py:104 and PAPER.md:312): edge derivation, the
// block-CSR Hessian pattern and per-element block ids, all on device with CUB.
#include <cub/cub.cuh>

#include "mg_internal.cuh"

namespace mg {

namespace {

constexpr int TPB = 256;
inline unsigned grid_for(int64_t n) { return (unsigned)((n + TPB - 1) / TPB); }

int key_bits(int64_t V) {
  int b = 1;
  while ((int64_t(1) << b) < V) ++b;
  return b;
}

__global__ void k_faces_in(const int64_t* in, int64_t F, int64_t V, int32_t* out, int* bad) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= F) return;
  int64_t a = in[3 * f], b = in[3 * f + 1], c = in[3 * f + 2];
  if (a < 0 || b < 0 || c < 0 || a >= V || b >= V || c >= V) atomicMin(&bad[0], (int)min(f, (int64_t)INT32_MAX));
  else if (a == b || b == c || a == c) atomicMin(&bad[1], (int)min(f, (int64_t)INT32_MAX));
  out[3 * f] = (int32_t)a;
  out[3 * f + 1] = (int32_t)b;
  out[3 * f + 2] = (int32_t)c;
}

// the three sides (0,1),(1,2),(2,0) of every face, canonical, as a*V+b keys
// (mesh.py:187-189)
__global__ void k_face_side_keys(const int32_t* f, int64_t F, int64_t V, uint64_t* keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * F) return;
  int64_t face = i / 3, s = i % 3;
  int64_t a = f[3 * face + s], b = f[3 * face + (s + 1) % 3];
  int64_t lo = a < b ? a : b, hi = a < b ? b : a;
  keys[i] = (uint64_t)(lo * V + hi);
}

__global__ void k_edge_keys_in(const int64_t* e, int64_t E, int64_t V, uint64_t* keys, int* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E) return;
  int64_t a = e[2 * i], b = e[2 * i + 1];
  if (a < 0 || b < 0 || a >= V || b >= V) atomicExch(&bad[0], 1);
  if (a == b) atomicExch(&bad[1], 1);
  int64_t lo = a < b ? a : b, hi = a < b ? b : a;
  keys[i] = (uint64_t)(lo * V + hi);
}

__global__ void k_keys_to_pairs(const uint64_t* keys, int64_t n, int64_t V, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[2 * i] = (int32_t)(keys[i] / (uint64_t)V);
  out[2 * i + 1] = (int32_t)(keys[i] % (uint64_t)V);
}

}  // namespace

// Sort + unique a key array in place (keys buffer reused); returns count.
int64_t sort_unique(uint64_t*& keys, int64_t n, int end_bit, cudaStream_t s) {
  if (n == 0) return 0;
  uint64_t* alt = nullptr;
  MG_CUDA(cudaMallocAsync(&alt, sizeof(uint64_t) * n, s));
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  size_t tb = 0;
  MG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)n, 0, end_bit, s));
  {
    Tmp t(s, tb);
    MG_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tb, db, (int64_t)n, 0, end_bit, s));
  }
  uint64_t* sorted = db.Current();
  uint64_t* out = (sorted == keys) ? alt : keys;
  int64_t* cnt_d = nullptr;
  MG_CUDA(cudaMallocAsync(&cnt_d, sizeof(int64_t), s));
  size_t tu = 0;
  MG_CUDA(cub::DeviceSelect::Unique(nullptr, tu, sorted, out, cnt_d, (int64_t)n, s));
  {
    Tmp t(s, tu);
    MG_CUDA(cub::DeviceSelect::Unique(t.p, tu, sorted, out, cnt_d, (int64_t)n, s));
  }
  int64_t cnt = 0;
  MG_CUDA(cudaMemcpyAsync(&cnt, cnt_d, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(cnt_d, s);
  // hand back the buffer that holds the result; free the other
  if (out == keys) {
    cudaFreeAsync(alt, s);
  } else {
    cudaFreeAsync(keys, s);
    keys = alt;
  }
  return cnt;
}

void mesh_build(Mesh& m, const int64_t* faces_d, const int64_t* edges_d, int64_t num_edges_in,
                const double* pos_d, cudaStream_t s) {
  const int64_t V = m.V, F = m.F;
  if (V >= (int64_t(1) << 31)) throw Error(MG_ERR_UNSUPPORTED, "more than 2^31-1 vertices");
  DBuf<int> bad;
  bad.alloc(2);
  int init[2] = {INT32_MAX, INT32_MAX};
  MG_CUDA(cudaMemcpyAsync(bad.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (pos_d && V) {
    m.pos.alloc(3 * V);
    MG_CUDA(cudaMemcpyAsync(m.pos.p, pos_d, sizeof(double) * 3 * V, cudaMemcpyDeviceToDevice, s));
  }
  if (F > 0) {
    if (edges_d) throw Error(MG_ERR_MESH, "edges are derived from faces; pass explicit edges only for face-free meshes");
    m.faces.alloc(3 * F);
    k_faces_in<<<grid_for(F), TPB, 0, s>>>(faces_d, F, V, m.faces.p, bad.p);
    MG_LAUNCH_CHECK();
    int hb[2];
    MG_CUDA(cudaMemcpyAsync(hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    if (hb[0] != INT32_MAX)
      throw Error(MG_ERR_MESH, "face " + std::to_string(hb[0]) + " references a vertex outside 0.." + std::to_string(V - 1));
    if (hb[1] != INT32_MAX)
      throw Error(MG_ERR_MESH, "face " + std::to_string(hb[1]) + " has repeated vertices");
    uint64_t* keys = nullptr;
    MG_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * 3 * F, s));
    k_face_side_keys<<<grid_for(3 * F), TPB, 0, s>>>(m.faces.p, F, V, keys);
    MG_LAUNCH_CHECK();
    m.E = sort_unique(keys, 3 * F, 2 * key_bits(V), s);
    m.edges.alloc(2 * m.E);
    if (m.E) k_keys_to_pairs<<<grid_for(m.E), TPB, 0, s>>>(keys, m.E, V, m.edges.p);
    MG_LAUNCH_CHECK();
    cudaFreeAsync(keys, s);
  } else if (edges_d && num_edges_in > 0) {
    uint64_t* keys = nullptr;
    MG_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * num_edges_in, s));
    int zero[2] = {0, 0};
    MG_CUDA(cudaMemcpyAsync(bad.p, zero, sizeof(zero), cudaMemcpyHostToDevice, s));
    k_edge_keys_in<<<grid_for(num_edges_in), TPB, 0, s>>>(edges_d, num_edges_in, V, keys, bad.p);
    MG_LAUNCH_CHECK();
    int hb[2];
    MG_CUDA(cudaMemcpyAsync(hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    if (hb[0]) { cudaFreeAsync(keys, s); throw Error(MG_ERR_MESH, "edge references a vertex out of range"); }
    if (hb[1]) { cudaFreeAsync(keys, s); throw Error(MG_ERR_MESH, "edge with identical endpoints"); }
    m.E = sort_unique(keys, num_edges_in, 2 * key_bits(V), s);
    m.edges.alloc(2 * m.E);
    if (m.E) k_keys_to_pairs<<<grid_for(m.E), TPB, 0, s>>>(keys, m.E, V, m.edges.p);
    MG_LAUNCH_CHECK();
    cudaFreeAsync(keys, s);
  } else {
    m.E = 0;
  }
  m.Vr = V;
  mesh_patches(m, s);
  MG_CUDA(cudaStreamSynchronize(s));
}

void mesh_set_owned(Mesh& m, const uint8_t* owned_d, cudaStream_t s) {
  if (!owned_d) {
    m.owned.reset();
  } else {
    m.owned.alloc(m.V > 0 ? m.V : 1);
    if (m.V) MG_CUDA(cudaMemcpyAsync(m.owned.p, owned_d, m.V, cudaMemcpyDeviceToDevice, s));
  }
  mesh_patches(m, s);
  MG_CUDA(cudaStreamSynchronize(s));
}

namespace {

// All ordered vertex pairs (incl. (i,i)) of every element whose both ends are
// free, as a*V+b keys (problem.py:391-396); pinned pairs become ~0 and sort last.
__global__ void k_pair_keys(const int32_t* sel, int P, int64_t M, int64_t V, const uint8_t* fixed,
                            const uint8_t* owned, uint64_t* keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t pp = (int64_t)P * P;
  if (i >= M * pp) return;
  int64_t e = i / pp;
  int r = (int)(i % pp), q1 = r / P, q2 = r % P;
  int64_t a = sel ? sel[e * P + q1] : e;
  int64_t b = sel ? sel[e * P + q2] : e;
  bool ok = !fixed || (!fixed[a] && !fixed[b]);
  ok &= !owned || owned[a];  // shard: only owned rows are assembled here
  keys[i] = ok ? (uint64_t)(a * V + b) : ~0ull;
}

__global__ void k_rows_cols(const uint64_t* keys, int64_t nnzb, int64_t V, int32_t* row_counts,
                            int64_t* cols, int32_t* cols32) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nnzb) return;
  int64_t r = (int64_t)(keys[i] / (uint64_t)V), c = (int64_t)(keys[i] % (uint64_t)V);
  atomicAdd(&row_counts[r], 1);
  cols[i] = c;
  cols32[i] = (int32_t)c;
}

// Per-element block ids by binary search in the sorted unique key list
// (the reference's searchsorted, problem.py:407-414); -1 marks pinned pairs.
__global__ void k_bids(const int32_t* sel, int P, int64_t M, int64_t V, const uint8_t* fixed,
                       const uint8_t* owned, const uint64_t* keys, int64_t nnzb, int32_t* bids) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t pp = (int64_t)P * P;
  if (i >= M * pp) return;
  int64_t e = i / pp;
  int r = (int)(i % pp), q1 = r / P, q2 = r % P;
  int64_t a = sel ? sel[e * P + q1] : e;
  int64_t b = sel ? sel[e * P + q2] : e;
  if ((fixed && (fixed[a] || fixed[b])) || (owned && !owned[a])) { bids[i] = -1; return; }
  uint64_t k = (uint64_t)(a * V + b);
  int64_t lo = 0, hi = nnzb;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  bids[i] = (int32_t)lo;
}

__global__ void k_widen(const int32_t* in, int64_t* out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

}  // namespace

void build_pattern(Problem& p, cudaStream_t s) {
  Mesh& m = *p.mesh;
  const int64_t V = m.V;
  int64_t total = 0;
  for (auto& t : p.terms) total += t.M * t.dev.P * t.dev.P;
  uint64_t* keys = nullptr;
  int64_t nnzb = 0;
  if (total > 0) {
    MG_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * total, s));
    int64_t off = 0;
    for (auto& t : p.terms) {
      int64_t cnt = t.M * t.dev.P * t.dev.P;
      if (cnt) k_pair_keys<<<grid_for(cnt), TPB, 0, s>>>(term_sel(m, t), t.dev.P, t.M, V,
                                                          p.any_fixed ? p.fixed.p : nullptr, m.owned.p, keys + off);
      MG_LAUNCH_CHECK();
      off += cnt;
    }
    nnzb = sort_unique(keys, total, 64, s);
    if (nnzb > 0) {
      uint64_t last = 0;
      MG_CUDA(cudaMemcpyAsync(&last, keys + nnzb - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      if (last == ~0ull) --nnzb;
    }
  }
  if (nnzb >= (int64_t(1) << 31)) throw Error(MG_ERR_UNSUPPORTED, "more than 2^31-1 Hessian blocks");
  p.nnzb = nnzb;
  p.row_offsets.alloc(V + 1);
  p.col_indices.alloc(nnzb > 0 ? nnzb : 1);
  p.col32.alloc(nnzb > 0 ? nnzb : 1);
  DBuf<int32_t> counts;
  counts.alloc(V + 1);
  MG_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int32_t) * (V + 1), s));
  if (nnzb) k_rows_cols<<<grid_for(nnzb), TPB, 0, s>>>(keys, nnzb, V, counts.p, p.col_indices.p, p.col32.p);
  MG_LAUNCH_CHECK();
  {
    // row_offsets = exclusive prefix sum of counts, widened to int64
    DBuf<int64_t> wide;
    wide.alloc(V + 1);
    k_widen<<<grid_for(V + 1), TPB, 0, s>>>(counts.p, wide.p, V + 1);
    MG_LAUNCH_CHECK();
    size_t tb = 0;
    MG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, wide.p, p.row_offsets.p, V + 1, s));
    Tmp t(s, tb);
    MG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, wide.p, p.row_offsets.p, V + 1, s));
    MG_CUDA(cudaStreamSynchronize(s));
  }
  for (auto& t : p.terms) {
    int64_t cnt = t.M * t.dev.P * t.dev.P;
    t.bids.alloc(cnt > 0 ? cnt : 1);
    if (cnt) k_bids<<<grid_for(cnt), TPB, 0, s>>>(term_sel(m, t), t.dev.P, t.M, V,
                                                   p.any_fixed ? p.fixed.p : nullptr, m.owned.p, keys, nnzb, t.bids.p);
    MG_LAUNCH_CHECK();
  }
  MG_CUDA(cudaStreamSynchronize(s));
  if (keys) cudaFreeAsync(keys, s);
  MG_CUDA(cudaStreamSynchronize(s));
  p.pattern_ready = true;
  p.gather_ready = false;
}

}  // namespace mg
