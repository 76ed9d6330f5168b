// Device-built vertex patches with ribbons (the north star's subsystem 1).
//
// The reference partitions FACES by a greedy host BFS (mesh.py:252-279) and
// lets edges/vertices inherit a patch (mesh.py:225-231); there patches only
// decide processing order. Here patches decide *ownership*: a patch owns a
// run of R rows of the Hessian/gradient (vertices, in Morton order of their
// positions so a patch is spatially compact), and one CTA assembles exactly
// those rows. The elements incident to owned rows are listed per patch; the
// ones that straddle two patches (ribbon elements) are evaluated by both
// owners, so every output row is written once, with no atomics and no
// communication (SURVEY 7.2 "owner computes"). The ribbon vertices are the
// non-owned vertices those elements touch; their x is staged alongside the
// owned ones.
//
// Everything is built with sorts/scans on the device; nothing here affects
// the numbers, only the order of floating-point summation.
#include <cstring>
#include <cstdlib>
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "mg_internal.cuh"

namespace mg {

namespace {

constexpr int TPB = 256;
inline unsigned grid_for(int64_t n) { return (unsigned)((n + TPB - 1) / TPB); }

__device__ __forceinline__ uint64_t spread3(uint64_t v) {  // 21 bits -> every 3rd bit
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

__global__ void k_bbox(const double* pos, int64_t V, double* out /* 6 per block */) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < 3; ++c) {
      double v = pos[3 * i + c];
      if (isfinite(v)) { lo[c] = fmin(lo[c], v); hi[c] = fmax(hi[c], v); }
    }
  __shared__ double s[6][TPB];
  for (int c = 0; c < 3; ++c) { s[c][threadIdx.x] = lo[c]; s[3 + c][threadIdx.x] = hi[c]; }
  __syncthreads();
  for (int o = TPB / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int c = 0; c < 3; ++c) {
        s[c][threadIdx.x] = fmin(s[c][threadIdx.x], s[c][threadIdx.x + o]);
        s[3 + c][threadIdx.x] = fmax(s[3 + c][threadIdx.x], s[3 + c][threadIdx.x + o]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) out[blockIdx.x * 6 + threadIdx.x] = s[threadIdx.x][0];
}

__global__ void k_morton(const double* pos, int64_t V, const double* box, const uint8_t* owned, uint64_t* code,
                         int32_t* ids) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  uint64_t m = 0;
  for (int c = 0; c < 3; ++c) {
    double ext = box[3 + c] - box[c];
    double t = ext > 0 ? (pos[3 * i + c] - box[c]) / ext : 0.0;
    t = isfinite(t) ? fmin(fmax(t, 0.0), 1.0) : 0.0;
    m |= spread3((uint64_t)(t * 2097151.0)) << (2 - c);
  }
  code[i] = (owned && !owned[i]) ? ~0ull : m;  // non-owned (halo) vertices sort last
  ids[i] = (int32_t)i;
}

// no positions: owned vertices first, in id order (stable sort on this key)
__global__ void k_owned_key(const uint8_t* owned, int64_t V, uint64_t* code, int32_t* ids) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  code[i] = owned[i] ? 0ull : 1ull;
  ids[i] = (int32_t)i;
}

__global__ void k_iota(int32_t* ids, int64_t V) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < V) ids[i] = (int32_t)i;
}

__global__ void k_count_owned(const uint8_t* owned, int64_t V, int* cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int c = (i < V && owned[i]) ? 1 : 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// rank in patch order; patch of every owned vertex (-1: halo vertex, no row here)
__global__ void k_rank_pov(const int32_t* order, int64_t V, int64_t Vr, int R, int32_t* rank, int32_t* pov) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  rank[order[i]] = (int32_t)i;
  pov[order[i]] = i < Vr ? (int32_t)(i / R) : -1;
}

// (patch, element) pairs: one per distinct patch among the element's vertices
__global__ void k_patch_elem_keys(const int32_t* sel, int P, int64_t M, const int32_t* pov, uint64_t* keys) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= M) return;
  int pq[3];
  for (int q = 0; q < P; ++q) {
    pq[q] = pov[sel[e * P + q]];
    bool dup = pq[q] < 0;  // halo vertex: its rows live on another device
    for (int r = 0; r < q; ++r) dup |= pq[r] == pq[q];
    keys[e * P + q] = dup ? ~0ull : ((uint64_t)pq[q] << 32) | (uint64_t)e;
  }
}

__global__ void k_lower_bounds(const uint64_t* keys, int64_t n, int64_t np, int32_t* off) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p > np) return;
  uint64_t k = (uint64_t)p << 32;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  off[p] = (int32_t)lo;
}

__global__ void k_lower_bounds_rows(const uint64_t* keys, int64_t n, int64_t V, int32_t* off) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > V) return;
  uint64_t k = (uint64_t)r << 32;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  off[r] = (int32_t)lo;
}

__global__ void k_split_entries(const uint64_t* keys, int64_t n, int32_t* elem) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) elem[j] = (int32_t)(keys[j] & 0xffffffffull);
}

__global__ void k_patch_of_entry(const int32_t* off, int64_t np, int32_t* pe) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  for (int j = off[p]; j < off[p + 1]; ++j) pe[j] = (int32_t)p;
}

__global__ void k_ribbon_keys(const int32_t* sel, int P, const int32_t* elem, const int32_t* pe, int64_t n,
                              const int32_t* pov, uint64_t* keys) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t e = elem[j];
  const int p = pe[j];
  for (int q = 0; q < P; ++q) {
    int u = sel[e * P + q];
    keys[j * P + q] = pov[u] == p ? ~0ull : ((uint64_t)p << 32) | (uint64_t)u;
  }
}

__device__ __forceinline__ int owned_count(int64_t p, int R, int64_t V) {
  int64_t c = V - p * R;
  return (int)(c < R ? c : R);
}

__global__ void k_vtx_off(const int32_t* rib_off, int64_t np, int R, int64_t V, int32_t* vtx_off) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p > np) return;
  int64_t owned = p * R < V ? p * R : V;
  vtx_off[p] = (int32_t)(owned + rib_off[p]);
}

__global__ void k_fill_owned(const int32_t* order, int64_t V, int R, const int32_t* vtx_off, int32_t* vtx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  int64_t p = i / R;
  vtx[vtx_off[p] + (i - p * R)] = order[i];
}

__global__ void k_fill_ribbon(const uint64_t* rkeys, int64_t nr, const int32_t* rib_off, int R, int64_t V,
                              const int32_t* vtx_off, int32_t* vtx) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nr) return;
  int64_t p = (int64_t)(rkeys[k] >> 32);
  vtx[vtx_off[p] + owned_count(p, R, V) + (k - rib_off[p])] = (int32_t)(rkeys[k] & 0xffffffffull);
}

__global__ void k_local_ids(const int32_t* sel, int P, const int32_t* elem, const int32_t* pe, int64_t n,
                            const int32_t* pov, const int32_t* rank, int R, int64_t V, const uint64_t* rkeys,
                            const int32_t* rib_off, uint16_t* local, int* overflow) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t e = elem[j];
  const int64_t p = pe[j];
  for (int q = 0; q < P; ++q) {
    const int u = sel[e * P + q];
    int64_t loc;
    if (pov[u] == p) {
      loc = rank[u] - p * R;
    } else {
      const uint64_t k = ((uint64_t)p << 32) | (uint64_t)u;
      int64_t lo = rib_off[p], hi = rib_off[p + 1];
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (rkeys[mid] < k) lo = mid + 1; else hi = mid;
      }
      loc = owned_count(p, R, V) + (lo - rib_off[p]);
    }
    if (loc > 65535) atomicExch(overflow, 1);
    local[j * P + q] = (uint16_t)loc;
  }
}

__global__ void k_positions(const int32_t* sel, int P, const int32_t* elem, const int32_t* pe, int64_t n,
                            const int32_t* pov, const int32_t* bids, const int64_t* ro, uint8_t* pos,
                            int* overflow) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t e = elem[j];
  const int p = pe[j];
  for (int q = 0; q < P; ++q) {
    const int u = sel[e * P + q];
    for (int r = 0; r < P; ++r) {
      int v = 255;
      if (pov[u] == p) {
        const int32_t b = bids[e * P * P + q * P + r];
        if (b >= 0) {
          int64_t d = b - ro[u];
          if (d > 254) atomicExch(overflow, 1);
          v = (int)d;
        }
      }
      pos[(j * P + q) * P + r] = (uint8_t)v;
    }
  }
}

// Greedy coloring per patch (one thread per patch, entries in element order):
// two entries conflict iff they share an owned vertex (they would add into
// the same shared-memory row). masks: (V) x 2 words of scratch, indexed by
// owned position in Morton order.
__global__ void k_color(const uint16_t* local, int P, const int32_t* off, int64_t np, int R, int64_t V,
                        uint64_t* masks, uint8_t* color, int* overflow) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int oc = owned_count(p, R, V);
  uint64_t* m = masks + 2 * p * R;
  for (int i = 0; i < 2 * oc; ++i) m[i] = 0;
  for (int j = off[p]; j < off[p + 1]; ++j) {
    uint64_t u0 = 0, u1 = 0;
    for (int q = 0; q < P; ++q) {
      int l = local[(int64_t)j * P + q];
      if (l < oc) { u0 |= m[2 * l]; u1 |= m[2 * l + 1]; }
    }
    int c;
    if (~u0) c = __ffsll(~u0) - 1;
    else if (~u1) c = 64 + __ffsll(~u1) - 1;
    else { atomicExch(overflow, 1); c = 127; }
    color[j] = (uint8_t)c;
    for (int q = 0; q < P; ++q) {
      int l = local[(int64_t)j * P + q];
      if (l < oc) {
        if (c < 64) m[2 * l] |= 1ull << c; else m[2 * l + 1] |= 1ull << (c - 64);
      }
    }
  }
}

__global__ void k_color_keys(const int32_t* pe, const uint8_t* color, const int32_t* elem, int64_t n,
                             uint64_t* keys, int32_t* idx) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  keys[j] = ((uint64_t)pe[j] << 40) | ((uint64_t)color[j] << 32) | (uint64_t)(uint32_t)elem[j];
  idx[j] = (int32_t)j;
}

template <class T>
__global__ void k_gather_rows(const T* src, const int32_t* idx, int64_t n, int w, T* dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * w) return;
  int64_t j = i / w, c = i % w;
  dst[i] = src[(int64_t)idx[j] * w + c];
}

__global__ void k_row_len_patch_order(const int32_t* order, const int64_t* ro, int64_t V, int32_t* len) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int v = order[i];
  len[i] = (int32_t)(ro[v + 1] - ro[v]);
}

__global__ void k_localize(const int32_t* scan, int64_t V, int R, int32_t* hloc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  hloc[i] = scan[i] - scan[(i / R) * R];
}

__global__ void k_patch_blocks(const int32_t* scan, int64_t V, int R, int64_t np, int* maxb) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  int64_t a = p * R, b = (p + 1) * R < V ? (p + 1) * R : V;
  atomicMax(maxb, scan[b] - scan[a]);
}

__global__ void k_max_diff(const int32_t* off, int64_t np, int* out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  atomicMax(out, off[p + 1] - off[p]);
}

__global__ void k_diag_pos(const int64_t* ro, const int32_t* col, int64_t V, uint8_t* dp) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= V) return;
  int64_t lo = ro[v], hi = ro[v + 1], a = lo, b = hi;
  while (a < b) {
    int64_t mid = (a + b) >> 1;
    if (col[mid] < v) a = mid + 1; else b = mid;
  }
  dp[v] = (a < hi && col[a] == v && a - lo < 255) ? (uint8_t)(a - lo) : 255;
}

// Shared-memory offset (in doubles) of every owned row's Hessian blocks in the
// edge fast path's row buffer: rows stacked in patch order, with one pad
// double where needed so each row has the same 16-byte phase in shared memory
// as in the output (the row is then streamed out with one bulk copy).
__global__ void k_row_smem_offsets(const int32_t* order, const int64_t* ro, int64_t Vr, int R, int64_t np, int NN,
                                   int32_t* hoff, int* maxd) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int64_t a = p * R, b = (p + 1) * R < Vr ? (p + 1) * R : Vr;
  int64_t off = 0;
  for (int64_t i = a; i < b; ++i) {
    const int v = order[i];
    const int64_t r0 = ro[v];
    if ((off - r0 * NN) & 1) ++off;
    hoff[i] = (int32_t)off;
    off += (ro[v + 1] - r0) * NN;
  }
  atomicMax(maxd, (int)off);
}

__global__ void k_vertex_flags(const uint8_t* fixed, const int32_t* vtx, int64_t n, uint8_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = fixed ? fixed[vtx[i]] : 0;
}

// Face-incidence records of the face row kernel: for every face and each
// corner that is an owned row, key = (row, face) (a row's faces in id order),
// value lo = face | slot << 30, hi = position of the next corner in the row |
// position of the one after << 8 | pinned corners << 16 (255: no block).
__global__ void k_row_face_inc(const int32_t* faces, int64_t F, const int32_t* rank, int64_t Vr,
                               const uint8_t* fixed, const int64_t* ro, const int32_t* col, uint64_t* keys,
                               uint64_t* vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * F) return;
  const int64_t f = i / 3;
  const int s = (int)(i % 3);
  const int v = faces[3 * f + s];
  const int64_t row = rank[v];
  if (row >= Vr) {
    keys[i] = ~0ull;
    vals[i] = 0;
    return;
  }
  uint32_t pins = 0;
  for (int q = 0; q < 3; ++q) pins |= (fixed && fixed[faces[3 * f + q]]) ? (1u << q) : 0u;
  uint32_t pos[2];
  for (int k = 1; k <= 2; ++k) {
    const int o = faces[3 * f + (s + k) % 3];
    uint32_t pk = 255;
    if (col && !(fixed && (fixed[v] || fixed[o]))) {
      int64_t lo = ro[v], hi = ro[v + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col[mid] < o) lo = mid + 1; else hi = mid;
      }
      if (lo < ro[v + 1] && col[lo] == o && lo - ro[v] < 255) pk = (uint32_t)(lo - ro[v]);
    }
    pos[k - 1] = pk;
  }
  keys[i] = ((uint64_t)row << 32) | (uint64_t)f;
  const uint32_t lo32 = (uint32_t)f | ((uint32_t)s << 30);
  const uint32_t hi32 = pos[0] | (pos[1] << 8) | (pins << 16);
  vals[i] = ((uint64_t)hi32 << 32) | lo32;
}

// per-row meta word of the edge row kernel: incidence count (saturated at
// 255), pinned flag, diagonal block position
__global__ void k_row_meta(const int32_t* rinc_off, const uint8_t* pfix, const uint8_t* pdp, const int32_t* plen,
                           int64_t Vr, uint32_t* meta) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Vr) return;
  const int c = rinc_off[i + 1] - rinc_off[i];
  const int l = plen ? plen[i] : 0;
  meta[i] = (uint32_t)(c < 255 ? c : 255) | ((uint32_t)(pfix[i] ? 1 : 0) << 8) |
            ((uint32_t)(pdp ? pdp[i] : 255) << 16) | ((uint32_t)(l < 255 ? l : 255) << 24);
}

// ELL copy of the first K incidences of every row, slot-major (slot k of row i
// at k * Vr + i: consecutive rows read consecutive words)
__global__ void k_ell(const int32_t* rinc_off, const uint64_t* rrec, int64_t Vr, int K, uint64_t* ell,
                      int64_t stride = 0) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Vr) return;
  if (!stride) stride = Vr;
  const int k0 = rinc_off[i], c = rinc_off[i + 1] - k0;
  for (int k = 0; k < K; ++k) ell[(int64_t)k * stride + i] = k < c ? rrec[k0 + k] : 0ull;
}

// Vertex-only 32-bit copies of the ELL incidence records (other |
// pinned(other) << 31) for the gradient / HVP row kernels of problems whose EV
// terms read no per-edge attribute (edge_rows.cuh; half the record bytes).
// Unused slots hold the row's own vertex (a valid address, never used). The
// first-vertex flag is other > vertex (canonical edges). Measured: +2% on the
// smoothing HVP / gradient; an edge-id delta variant for the spring was 2%
// slower (the decode sits on the gathers' dependency chain) and was dropped.
__global__ void k_ell32(const int32_t* rinc_off, const uint64_t* rrec, const int32_t* order, int64_t Vr, int K,
                        uint32_t* ell32, int64_t stride) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Vr) return;
  const int k0 = rinc_off[i], c = rinc_off[i + 1] - k0;
  const int64_t g = order ? order[i] : i;
  for (int k = 0; k < K; ++k) ell32[(int64_t)k * stride + i] = k < c ? (uint32_t)(rrec[k0 + k] >> 32) : (uint32_t)g;
}

// face rows: the other two corners (s+1, s+2 mod 3) of each ELL face incidence,
// so the row kernels skip the faces[] lookup (one dependent level less)
__global__ void k_ellv(const int32_t* rinc_off, const uint64_t* rrec, const int32_t* faces, int64_t Vr, int K,
                       uint64_t* ellv, int64_t stride) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Vr) return;
  const int k0 = rinc_off[i], c = rinc_off[i + 1] - k0;
  for (int k = 0; k < K; ++k) {
    uint64_t v = 0;
    if (k < c) {
      const uint32_t lo = (uint32_t)rrec[k0 + k];
      const int64_t f = lo & 0x3fffffffu;
      const int s = (int)(lo >> 30);
      const uint32_t o1 = (uint32_t)faces[3 * f + (s + 1) % 3], o2 = (uint32_t)faces[3 * f + (s + 2) % 3];
      v = (uint64_t)o1 | ((uint64_t)o2 << 32);
    }
    ellv[(int64_t)k * stride + i] = v;
  }
}

// CTA face lists of the face row kernel (k_cta_dirichlet): key (block << 32 |
// face) for every face corner whose row is owned (block = row / RB)
__global__ void k_cf_keys(const int32_t* faces, int64_t F, const int32_t* rank, int64_t Vr, int RB,
                          uint64_t* keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * F) return;
  const int64_t row = rank[faces[i]];
  keys[i] = row < Vr ? ((uint64_t)(row / RB) << 32) | (uint64_t)(i / 3) : ~0ull;
}

// {face | (its corner 0's row is in the block) << 31, corners} (one 16-byte
// coalesced load per face in the kernel: no dependent faces[] gather)
__global__ void k_cf_faces(const uint64_t* keys, int64_t n, const int32_t* faces, const int32_t* rank, int64_t Vr,
                           int RB, int4* cf) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t blk = (int64_t)(keys[i] >> 32);
  const uint32_t f = (uint32_t)keys[i];
  const int v0 = faces[3 * (int64_t)f], v1 = faces[3 * (int64_t)f + 1], v2 = faces[3 * (int64_t)f + 2];
  const int64_t r0 = rank[v0];
  const bool own0 = r0 < Vr && r0 / RB == blk;
  cf[i] = make_int4((int)(f | ((uint32_t)own0 << 31)), v0, v1, v2);
}

// per incidence: its face's slot in the row's block list (binary search, the
// list is sorted by face) | the row's corner << 14; ELL copy of the first K slot-major
__global__ void k_cf_slots(const int32_t* rinc_off, const uint64_t* rrec, int64_t Vr, int RB, int K,
                           const int32_t* cf_off, const int4* cf, uint16_t* rslot, uint16_t* eslot, int* bad,
                           int64_t stride) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= Vr) return;
  const int64_t blk = r / RB;
  const int b0 = cf_off[blk], b1 = cf_off[blk + 1];
  const int k0 = rinc_off[r], c = rinc_off[r + 1] - k0;
  for (int k = 0; k < c; ++k) {
    const uint32_t f = (uint32_t)rrec[k0 + k] & 0x3fffffffu;
    int lo = b0, hi = b1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (((uint32_t)cf[mid].x & 0x7fffffffu) < f) lo = mid + 1; else hi = mid;
    }
    if (lo >= b1 || ((uint32_t)cf[lo].x & 0x7fffffffu) != f || lo - b0 >= (1 << 14)) *bad = 1;
    // slot | the row's corner in the face << 14 (all the gradient / HVP rows need)
    const uint16_t sl = (uint16_t)((lo - b0) | (((uint32_t)rrec[k0 + k] >> 30) << 14));
    rslot[k0 + k] = sl;
    if (k < K) eslot[(int64_t)k * stride + r] = sl;
  }
  for (int k = c; k < K; ++k) eslot[(int64_t)k * stride + r] = 0;
}

// Face rows: order each row's incidences around its vertex (face j's second
// other corner is face j+1's first: consistently oriented manifold fans, open
// or closed, at most 16 faces) and flag the row (meta bit 9); other rows keep
// face-id order. Records keep their contents, only their order changes.
__global__ void k_fan_order(const int32_t* rinc_off, uint64_t* rrec, const int32_t* faces, int64_t Vr,
                            uint32_t* meta) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= Vr) return;
  const int k0 = rinc_off[r], c = rinc_off[r + 1] - k0;
  if (c < 1 || c > 16) return;
  uint64_t rec[16];
  int o1[16], o2[16];
  for (int k = 0; k < c; ++k) {
    rec[k] = rrec[k0 + k];
    const uint32_t lo = (uint32_t)rec[k];
    const int64_t f = lo & 0x3fffffffu;
    const int s = (int)(lo >> 30);
    o1[k] = faces[3 * f + (s + 1) % 3];
    o2[k] = faces[3 * f + (s + 2) % 3];
  }
  // start: the face whose first other corner ends no other face (open fan), else face 0
  int start = -1, nstart = 0;
  for (int k = 0; k < c; ++k) {
    int preds = 0;
    for (int j = 0; j < c; ++j) preds += (o2[j] == o1[k]) ? 1 : 0;
    if (preds > 1) return;  // non-manifold
    if (preds == 0) {
      ++nstart;
      start = k;
    }
  }
  if (nstart > 1) return;  // several fans
  if (start < 0) start = 0;
  int order[16];
  unsigned used = 1u << start;
  order[0] = start;
  for (int step = 1; step < c; ++step) {
    const int cur = order[step - 1];
    int nxt = -1;
    for (int j = 0; j < c; ++j)
      if (!((used >> j) & 1) && o1[j] == o2[cur]) {
        if (nxt >= 0) return;
        nxt = j;
      }
    if (nxt < 0) return;
    used |= 1u << nxt;
    order[step] = nxt;
  }
  for (int k = 0; k < c; ++k) rrec[k0 + k] = rec[order[k]];
  meta[r] |= 1u << 9;
}

__global__ void k_patch_rows(const int32_t* order, const int64_t* ro, const uint8_t* dp, int64_t Vr,
                             int64_t* pro, int32_t* plen, uint8_t* pdp) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Vr) return;
  const int v = order[i];
  pro[i] = ro[v];
  plen[i] = (int32_t)(ro[v + 1] - ro[v]);
  pdp[i] = dp[v];
}


// Row-incidence records of the edge row kernel: for every edge and each
// endpoint that is an owned row, key = (row in patch order, other endpoint),
// value = (edge | slot << 31, other | pinned(other) << 31). Sorted by key, a
// row's records are its incident edges in column order.
__global__ void k_row_inc(const int32_t* edges, int64_t E, const int32_t* rank, int64_t Vr, const uint8_t* fixed,
                          uint64_t* keys, uint64_t* vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 2 * E) return;
  const int64_t e = i >> 1;
  const int q = (int)(i & 1);
  const int v = edges[2 * e + q], o = edges[2 * e + 1 - q];
  const int64_t row = rank[v];
  if (row < Vr) {
    keys[i] = ((uint64_t)row << 32) | (uint32_t)o;
    const uint32_t hi = (uint32_t)o | ((fixed && fixed[o]) ? 0x80000000u : 0u);
    const uint32_t lo = (uint32_t)e | ((uint32_t)q << 31);
    vals[i] = ((uint64_t)hi << 32) | lo;
  } else {
    keys[i] = ~0ull;
    vals[i] = 0;
  }
}

int to_host_int(const int* d, cudaStream_t s) {
  int h = 0;
  MG_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  return h;
}

// translation regularity of the caller's numbering: edges (i,j) (sorted,
// canonical) whose shifted pair (i+1,j+1) is also an edge
__global__ void k_edge_regularity(const int32_t* edges, int64_t E, unsigned long long* hits) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool hit = false;
  if (e < E) {
    const int32_t a = edges[2 * e] + 1, b = edges[2 * e + 1] + 1;
    int64_t lo = e + 1, hi = E;  // (a,b) sorts after (a-1,b-1)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const int32_t ma = edges[2 * mid], mb = edges[2 * mid + 1];
      if (ma < a || (ma == a && mb < b)) lo = mid + 1; else hi = mid;
    }
    hit = lo < E && edges[2 * lo] == a && edges[2 * lo + 1] == b;
  }
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(hits, (unsigned long long)__popc(m));
}

int key_bits(int64_t v) {
  int b = 1;
  while ((int64_t(1) << b) <= v) ++b;
  return b;
}

}  // namespace

void mesh_patches(Mesh& m, cudaStream_t s) {
  const int64_t V = m.V;
  PatchSet& ps = m.patches;
  const uint8_t* owned = m.owned.p;
  ps.R = m.patch_vertices;
  if (owned) {
    DBuf<int> cnt;
    cnt.alloc(1);
    MG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), s));
    k_count_owned<<<grid_for(V), TPB, 0, s>>>(owned, V, cnt.p);
    MG_LAUNCH_CHECK();
    m.Vr = to_host_int(cnt.p, s);
  } else {
    m.Vr = V;
  }
  ps.num = (m.Vr + ps.R - 1) / ps.R;
  ps.order.alloc(V > 0 ? V : 1);
  ps.rank.alloc(V > 0 ? V : 1);
  ps.patch_of_vertex.alloc(V > 0 ? V : 1);
  if (V == 0) return;
  // row order (mg_row_order): explicit, the MG_ROW_ORDER env knob, or the
  // regularity test of the caller's numbering
  int order = m.row_order;
  const char* ro_env = getenv("MG_ROW_ORDER");
  if (ro_env && !strcmp(ro_env, "identity")) order = MG_ROW_IDENTITY;
  if (ro_env && !strcmp(ro_env, "morton")) order = MG_ROW_MORTON;
  if (m.E > 0) {
    DBuf<unsigned long long> hits;
    hits.alloc(1);
    MG_CUDA(cudaMemsetAsync(hits.p, 0, sizeof(unsigned long long), s));
    k_edge_regularity<<<grid_for(m.E), TPB, 0, s>>>(m.edges.p, m.E, hits.p);
    MG_LAUNCH_CHECK();
    unsigned long long h = 0;
    MG_CUDA(cudaMemcpyAsync(&h, hits.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    m.regularity = (double)h / (double)m.E;
  }
  if (order == MG_ROW_AUTO) order = m.regularity >= 0.5 ? MG_ROW_IDENTITY : MG_ROW_MORTON;
  if (!m.pos.p) order = MG_ROW_IDENTITY;
  m.row_order_used = order;
  const bool ident = order == MG_ROW_IDENTITY;
  if ((m.pos.p && !ident) || owned) {
    DBuf<uint64_t> code, code2;
    DBuf<int32_t> ids;
    code.alloc(V);
    code2.alloc(V);
    ids.alloc(V);
    if (m.pos.p && !ident) {
      const int nb = 256;
      DBuf<double> part, box;
      part.alloc(6 * nb);
      box.alloc(6);
      k_bbox<<<nb, TPB, 0, s>>>(m.pos.p, V, part.p);
      MG_LAUNCH_CHECK();
      std::vector<double> hp(6 * nb);
      MG_CUDA(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * 6 * nb, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      double hb[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int b = 0; b < nb; ++b)
        for (int c = 0; c < 3; ++c) {
          hb[c] = std::fmin(hb[c], hp[6 * b + c]);
          hb[3 + c] = std::fmax(hb[3 + c], hp[6 * b + 3 + c]);
        }
      MG_CUDA(cudaMemcpyAsync(box.p, hb, sizeof(hb), cudaMemcpyHostToDevice, s));
      k_morton<<<grid_for(V), TPB, 0, s>>>(m.pos.p, V, box.p, owned, code.p, ids.p);
      MG_CUDA(cudaStreamSynchronize(s));
    } else {
      k_owned_key<<<grid_for(V), TPB, 0, s>>>(owned, V, code.p, ids.p);
    }
    MG_LAUNCH_CHECK();
    size_t tb = 0;
    MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, code.p, code2.p, ids.p, ps.order.p, (int64_t)V, 0, 64, s));
    Tmp t(s, tb);
    MG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, code.p, code2.p, ids.p, ps.order.p, (int64_t)V, 0, 64, s));
    MG_CUDA(cudaStreamSynchronize(s));
  } else {
    k_iota<<<grid_for(V), TPB, 0, s>>>(ps.order.p, V);
    MG_LAUNCH_CHECK();
  }
  k_rank_pov<<<grid_for(V), TPB, 0, s>>>(ps.order.p, V, m.Vr, ps.R, ps.rank.p, ps.patch_of_vertex.p);
  MG_LAUNCH_CHECK();
  MG_CUDA(cudaStreamSynchronize(s));
}

// Layout of the edge row kernel (edge_kernels.cu): rows in patch (Morton)
// order, per-row incidence records, static per-row streams and the shared-
// memory row offsets of each ROW_BLOCK-row CTA.

// ---- staged edge tiles (k_tile_hvp in edge_kernels.cu) --------------------
// Tile b = rows [b T, (b+1) T) in patch order. Its vertex table lists the
// tile's rows, then the halo (other vertices of the tile's edges); its edge
// table lists every edge incident to a row of the tile once.

MG_DI int tile_rows(int64_t b, int64_t Vr, int T) {
  const int64_t r = Vr - b * T;
  return (int)(r < T ? r : T);
}

__global__ void k_tile_inc_keys(const int32_t* rinc_off, const uint64_t* rrec, const int32_t* rank, int64_t Vr, int T,
                                uint64_t* hkeys, uint64_t* ekeys) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= Vr) return;
  const int64_t b = r / T;
  for (int k = rinc_off[r]; k < rinc_off[r + 1]; ++k) {
    const uint64_t rec = rrec[k];
    const int32_t o = (int32_t)((rec >> 32) & 0x7fffffffu);
    const int64_t ro = rank[o];
    const bool inside = ro < Vr && ro / T == b;
    hkeys[k] = inside ? ~0ull : (((uint64_t)b << 32) | (uint32_t)o);
    ekeys[k] = ((uint64_t)b << 32) | ((uint32_t)rec & 0x7fffffffu);
  }
}

__global__ void k_tile_counts(const int32_t* hoff, const int32_t* eoff, int64_t nt, int64_t Vr, int T, int32_t* cnt,
                              int* maxv, int* maxe) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b > nt) return;
  if (b == nt) { cnt[b] = 0; return; }
  const int nv = tile_rows(b, Vr, T) + hoff[b + 1] - hoff[b];
  cnt[b] = nv;
  atomicMax(maxv, nv);
  atomicMax(maxe, eoff[b + 1] - eoff[b]);
}

__global__ void k_tile_fill_rows(const int32_t* order, const uint8_t* fixed, int64_t Vr, int T, int MV, uint32_t* tv) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= Vr) return;
  const int64_t b = r / T;
  const int32_t g = order[r];
  tv[b * MV + (r - b * T)] = (uint32_t)g | ((fixed && fixed[g]) ? 0x80000000u : 0u);
}

__global__ void k_tile_fill_halo(const uint64_t* hkeys, int64_t nh, const int32_t* hoff, const uint8_t* fixed,
                                 int64_t Vr, int T, int MV, uint32_t* tv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nh) return;
  const int64_t b = (int64_t)(hkeys[i] >> 32);
  const uint32_t o = (uint32_t)hkeys[i];
  tv[b * MV + tile_rows(b, Vr, T) + (i - hoff[b])] = o | ((fixed && fixed[o]) ? 0x80000000u : 0u);
}

__global__ void k_tile_counts2(const int32_t* cnt, const int32_t* eoff, int64_t nt, int2* tcnt) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nt) return;
  tcnt[b] = make_int2(cnt[b], eoff[b + 1] - eoff[b]);
}

MG_DI int64_t seg_find(const uint64_t* keys, int64_t lo, int64_t hi, uint64_t k) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_tile_edges(const uint64_t* ekeys, int64_t ne, const int32_t* edges, const int32_t* rank,
                             const uint64_t* hkeys, const int32_t* hoff, const int32_t* eoff, int64_t Vr, int T, int ME,
                             uint64_t* te) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ne) return;
  const int64_t b = (int64_t)(ekeys[i] >> 32);
  const uint32_t e = (uint32_t)ekeys[i];
  uint32_t loc[2];
  for (int q = 0; q < 2; ++q) {
    const int32_t v = edges[2 * (int64_t)e + q];
    const int64_t rv = rank[v];
    if (rv < Vr && rv / T == b) {
      loc[q] = (uint32_t)(rv - b * T);
    } else {
      const int64_t j = seg_find(hkeys, hoff[b], hoff[b + 1], ((uint64_t)b << 32) | (uint32_t)v);
      loc[q] = (uint32_t)(tile_rows(b, Vr, T) + (j - hoff[b]));
    }
  }
  te[b * ME + (i - eoff[b])] = (uint64_t)e | ((uint64_t)(loc[0] & 0xffffu) << 32) | ((uint64_t)(loc[1] & 0xffffu) << 48);
}

__global__ void k_tile_islot(const int32_t* rinc_off, const uint64_t* rrec, const uint64_t* ekeys,
                             const int32_t* eoff, int64_t Vr, int T, uint16_t* islot) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= Vr) return;
  const int64_t b = r / T;
  for (int k = rinc_off[r]; k < rinc_off[r + 1]; ++k) {
    const uint32_t lo = (uint32_t)rrec[k];
    const int64_t j = seg_find(ekeys, eoff[b], eoff[b + 1], ((uint64_t)b << 32) | (lo & 0x7fffffffu));
    islot[k] = (uint16_t)((j - eoff[b]) | ((lo >> 31) << 15));
  }
}

__global__ void k_tile_islot8(const int32_t* rinc_off, const uint16_t* islot, int64_t Vr, uint16_t* out) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= Vr) return;
  const int k0 = rinc_off[r], n = rinc_off[r + 1] - k0;
  for (int j = 0; j < 8; ++j) out[r * 8 + j] = j < n ? islot[k0 + j] : (uint16_t)0;
}

void build_tiles_ev(Problem& p, cudaStream_t s) {
  Mesh& m = *p.mesh;
  const int64_t Vr = m.Vr;
  const int T = EV_TILE_ROWS;
  const int64_t nt = (Vr + T - 1) / T;
  p.tiles_ready = false;
  if (!nt) return;
  int64_t ninc = 0;
  {
    int32_t h = 0;
    MG_CUDA(cudaMemcpyAsync(&h, p.rinc_off.p + Vr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    ninc = h;
  }
  if (!ninc) return;
  uint64_t *hk = nullptr, *ek = nullptr;
  MG_CUDA(cudaMallocAsync(&hk, sizeof(uint64_t) * ninc, s));
  MG_CUDA(cudaMallocAsync(&ek, sizeof(uint64_t) * ninc, s));
  k_tile_inc_keys<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, m.patches.rank.p, Vr, T, hk, ek);
  MG_LAUNCH_CHECK();
  int64_t nh = sort_unique(hk, ninc, 64, s);
  if (nh > 0) {
    uint64_t last = 0;
    MG_CUDA(cudaMemcpyAsync(&last, hk + nh - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    if (last == ~0ull) --nh;
  }
  const int64_t ne = sort_unique(ek, ninc, 64, s);
  DBuf<int32_t> hoff, cnt;
  hoff.alloc(nt + 1);
  cnt.alloc(nt + 1);
  p.te_off.alloc(nt + 1);
  k_lower_bounds<<<grid_for(nt + 1), TPB, 0, s>>>(hk, nh, nt, hoff.p);
  k_lower_bounds<<<grid_for(nt + 1), TPB, 0, s>>>(ek, ne, nt, p.te_off.p);
  MG_LAUNCH_CHECK();
  DBuf<int> mx;
  mx.alloc(2);
  MG_CUDA(cudaMemsetAsync(mx.p, 0, 2 * sizeof(int), s));
  k_tile_counts<<<grid_for(nt + 1), TPB, 0, s>>>(hoff.p, p.te_off.p, nt, Vr, T, cnt.p, mx.p, mx.p + 1);
  MG_LAUNCH_CHECK();
  int hm[2] = {0, 0};
  MG_CUDA(cudaMemcpyAsync(hm, mx.p, sizeof(hm), cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  // padded tables (tile b at b * MV / b * ME): the kernel addresses them from
  // the tile index alone; the pipeline holds a tile's share in registers
  const int MV = hm[0], ME = hm[1];
  const bool fits = MV <= EV_TILE_VPT * T && ME <= EV_TILE_EPT * T && nt * MV < (int64_t(1) << 31) &&
                    nt * (int64_t)MV <= 2 * (Vr + nh) + 64 * nt && nt * (int64_t)ME <= 2 * ne + 64 * nt;
  if (getenv("MG_DEBUG_TILES"))
    fprintf(stderr, "edge tiles: %lld tiles, max_v %d, max_e %d, halo %lld, edges %lld, fits %d\n", (long long)nt, MV,
            ME, (long long)nh, (long long)ne, (int)fits);
  if (fits) {
    const uint8_t* fx = p.any_fixed ? p.fixed.p : nullptr;
    p.tv.alloc(nt * MV);
    k_tile_fill_rows<<<grid_for(Vr), TPB, 0, s>>>(m.patches.order.p, fx, Vr, T, MV, p.tv.p);
    if (nh) k_tile_fill_halo<<<grid_for(nh), TPB, 0, s>>>(hk, nh, hoff.p, fx, Vr, T, MV, p.tv.p);
    p.te.alloc(nt * ME > 0 ? nt * ME : 1);
    if (ne) k_tile_edges<<<grid_for(ne), TPB, 0, s>>>(ek, ne, m.edges.p, m.patches.rank.p, hk, hoff.p, p.te_off.p, Vr, T,
                                                      ME, p.te.p);
    p.tcnt.alloc(nt);
    k_tile_counts2<<<grid_for(nt), TPB, 0, s>>>(cnt.p, p.te_off.p, nt, p.tcnt.p);
    p.islot.alloc(ninc);
    k_tile_islot<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, ek, p.te_off.p, Vr, T, p.islot.p);
    p.islot8.alloc(Vr * 8);
    k_tile_islot8<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.islot.p, Vr, p.islot8.p);
    MG_LAUNCH_CHECK();
    p.tile_max_v = MV;
    p.tile_max_e = ME;
  }
  MG_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(hk, s);
  cudaFreeAsync(ek, s);
  MG_CUDA(cudaStreamSynchronize(s));
  p.tiles_ready = fits;
}

void build_rows_ev(Problem& p, cudaStream_t s, bool tiles) {
  Mesh& m = *p.mesh;
  PatchSet& ps = m.patches;
  const int64_t V = m.V, Vr = m.Vr, E = m.E;
  const int RB = EV_ROW_BLOCK;
  const int64_t nb = (Vr + RB - 1) / RB;
  DBuf<int> mx;
  mx.alloc(1);
  {
    DBuf<uint64_t> k1, k2, v1, v2;
    const int64_t n = 2 * E > 0 ? 2 * E : 1;
    k1.alloc(n); k2.alloc(n); v1.alloc(n); v2.alloc(n);
    if (E) k_row_inc<<<grid_for(2 * E), TPB, 0, s>>>(m.edges.p, E, ps.rank.p, Vr, p.any_fixed ? p.fixed.p : nullptr,
                                                     k1.p, v1.p);
    MG_LAUNCH_CHECK();
    if (E) {
      size_t tb = 0;
      MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1.p, k2.p, v1.p, v2.p, 2 * E, 0, 64, s));
      Tmp t(s, tb);
      MG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, k1.p, k2.p, v1.p, v2.p, 2 * E, 0, 64, s));
    }
    p.rinc_off.alloc(Vr + 1);
    k_lower_bounds_rows<<<grid_for(Vr + 1), TPB, 0, s>>>(k2.p, 2 * E, Vr, p.rinc_off.p);
    MG_LAUNCH_CHECK();
    MG_CUDA(cudaStreamSynchronize(s));
    p.rrec = std::move(v2);
  }
  p.pfix.alloc(Vr > 0 ? Vr : 1);
  if (Vr) k_vertex_flags<<<grid_for(Vr), TPB, 0, s>>>(p.any_fixed ? p.fixed.p : nullptr, ps.order.p, Vr, p.pfix.p);
  MG_LAUNCH_CHECK();
  p.max_patch_hdoubles = 0;
  if (p.with_hessian && p.pattern_ready) {
    p.diag_pos.alloc(V > 0 ? V : 1);
    if (V) k_diag_pos<<<grid_for(V), TPB, 0, s>>>(p.row_offsets.p, p.col32.p, V, p.diag_pos.p);
    const int64_t Vpad = (Vr + RB - 1) / RB * RB;  // whole row blocks (staged kernels' bulk copies)
    p.prow_ro.alloc(Vpad > 0 ? Vpad : 1);
    if (Vpad) MG_CUDA(cudaMemsetAsync(p.prow_ro.p, 0, sizeof(int64_t) * Vpad, s));
    p.prow_len.alloc(Vr > 0 ? Vr : 1);
    p.prow_dp.alloc(Vr > 0 ? Vr : 1);
    if (Vr) k_patch_rows<<<grid_for(Vr), TPB, 0, s>>>(ps.order.p, p.row_offsets.p, p.diag_pos.p, Vr, p.prow_ro.p,
                                                     p.prow_len.p, p.prow_dp.p);
    MG_LAUNCH_CHECK();
    p.hoff.alloc(Vpad > 0 ? Vpad : 1);
    if (Vpad) MG_CUDA(cudaMemsetAsync(p.hoff.p, 0, sizeof(int32_t) * Vpad, s));
    MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
    if (nb) k_row_smem_offsets<<<grid_for(nb), TPB, 0, s>>>(ps.order.p, p.row_offsets.p, Vr, RB, nb, p.n * p.n,
                                                           p.hoff.p, mx.p);
    MG_LAUNCH_CHECK();
    p.max_patch_hdoubles = to_host_int(mx.p, s);
  }
  // the edge rows' per-row streams padded to whole row blocks (slot stride
  // Vp = a multiple of EV_ROW_BLOCK): every block's slice of every stream is
  // one aligned bulk (TMA) copy for the staged gradient / HVP kernels
  const int64_t Vp = (Vr + RB - 1) / RB * RB;
  p.ell_stride = Vp;
  p.rmeta.alloc(Vp > 0 ? Vp : 1);
  p.ell.alloc(Vp > 0 ? (int64_t)EV_ELL_K * Vp : 1);
  if (Vp) {
    MG_CUDA(cudaMemsetAsync(p.rmeta.p, 0, sizeof(uint32_t) * Vp, s));
    MG_CUDA(cudaMemsetAsync(p.ell.p, 0, sizeof(uint64_t) * EV_ELL_K * Vp, s));
  }
  if (Vr) {
    k_row_meta<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.pfix.p, p.prow_dp.p, p.prow_len.p, Vr, p.rmeta.p);
    k_ell<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, Vr, EV_ELL_K, p.ell.p, Vp);
  }
  MG_LAUNCH_CHECK();
  {
    const bool ident = m.row_order_used == MG_ROW_IDENTITY && !m.owned.p;
    p.order_pad.alloc(!ident && Vp > 0 ? Vp : 1);
    if (!ident && Vp) {
      MG_CUDA(cudaMemsetAsync(p.order_pad.p, 0, sizeof(int32_t) * Vp, s));
      MG_CUDA(cudaMemcpyAsync(p.order_pad.p, ps.order.p, sizeof(int32_t) * Vr, cudaMemcpyDeviceToDevice, s));
    }
  }
  // vertex-only records for the gradient / HVP kernels when no edge term reads
  // a per-edge attribute (the kernels of such problems read only these)
  {
    bool vo = true;
    for (auto& t : p.terms)
      if (t.dev.op == MG_OP_EV) vo &= t.jit ? t.jit_attrs.empty() : t.dev.type == MG_TERM_EDGE_LENGTH;
    p.ell32_ok = vo && Vr > 0;
    p.ell32.alloc(p.ell32_ok ? (int64_t)EV_ELL_K * Vp : 1);
    const bool ident = m.row_order_used == MG_ROW_IDENTITY && !m.owned.p;
    if (p.ell32_ok) {
      MG_CUDA(cudaMemsetAsync(p.ell32.p, 0, sizeof(uint32_t) * EV_ELL_K * Vp, s));
      k_ell32<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, ident ? nullptr : ps.order.p, Vr, EV_ELL_K,
                                           p.ell32.p, Vp);
    }
    MG_LAUNCH_CHECK();
  }
  MG_CUDA(cudaStreamSynchronize(s));
  p.redo.alloc(1);
  MG_CUDA(cudaMemsetAsync(p.redo.p, 0, sizeof(int), s));
  if (!p.exact_runs.p) {
    p.exact_runs.alloc(1);
    MG_CUDA(cudaMemsetAsync(p.exact_runs.p, 0, sizeof(int), s));
  }
  MG_CUDA(cudaStreamSynchronize(s));
  p.recomputed_elements = 0;
  if (tiles) build_tiles_ev(p, s);
  p.ev_fast = true;
  p.layout_ready = true;
}

// Layout of the face row kernel (face_kernels.cu): as build_rows_ev, with
// face incidences (and row lengths in the meta word, the kernel clears its row).
void build_rows_fv(Problem& p, cudaStream_t s) {
  Mesh& m = *p.mesh;
  PatchSet& ps = m.patches;
  const int64_t V = m.V, Vr = m.Vr;
  const int RB = EV_ROW_BLOCK;
  const int64_t nb = (Vr + RB - 1) / RB;
  DBuf<int> mx;
  mx.alloc(1);
  {
    DBuf<uint64_t> k1, k2, v1, v2;
    const int64_t F = m.F;
    const int64_t n = 3 * F > 0 ? 3 * F : 1;
    k1.alloc(n); k2.alloc(n); v1.alloc(n); v2.alloc(n);
    const bool pat = p.with_hessian && p.pattern_ready;
    if (F) k_row_face_inc<<<grid_for(3 * F), TPB, 0, s>>>(m.faces.p, F, ps.rank.p, Vr, p.any_fixed ? p.fixed.p : nullptr,
                                                          pat ? p.row_offsets.p : nullptr, pat ? p.col32.p : nullptr,
                                                          k1.p, v1.p);
    MG_LAUNCH_CHECK();
    if (F) {
      size_t tb = 0;
      MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1.p, k2.p, v1.p, v2.p, 3 * F, 0, 64, s));
      Tmp t(s, tb);
      MG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, k1.p, k2.p, v1.p, v2.p, 3 * F, 0, 64, s));
    }
    p.rinc_off.alloc(Vr + 1);
    k_lower_bounds_rows<<<grid_for(Vr + 1), TPB, 0, s>>>(k2.p, 3 * F, Vr, p.rinc_off.p);
    MG_LAUNCH_CHECK();
    MG_CUDA(cudaStreamSynchronize(s));
    p.rrec = std::move(v2);
  }
  p.pfix.alloc(Vr > 0 ? Vr : 1);
  if (Vr) k_vertex_flags<<<grid_for(Vr), TPB, 0, s>>>(p.any_fixed ? p.fixed.p : nullptr, ps.order.p, Vr, p.pfix.p);
  MG_LAUNCH_CHECK();
  p.max_patch_hdoubles = 0;
  if (p.with_hessian && p.pattern_ready) {
    p.diag_pos.alloc(V > 0 ? V : 1);
    if (V) k_diag_pos<<<grid_for(V), TPB, 0, s>>>(p.row_offsets.p, p.col32.p, V, p.diag_pos.p);
    const int64_t Vpad = (Vr + RB - 1) / RB * RB;  // whole row blocks (staged kernels' bulk copies)
    p.prow_ro.alloc(Vpad > 0 ? Vpad : 1);
    if (Vpad) MG_CUDA(cudaMemsetAsync(p.prow_ro.p, 0, sizeof(int64_t) * Vpad, s));
    p.prow_len.alloc(Vr > 0 ? Vr : 1);
    p.prow_dp.alloc(Vr > 0 ? Vr : 1);
    if (Vr) k_patch_rows<<<grid_for(Vr), TPB, 0, s>>>(ps.order.p, p.row_offsets.p, p.diag_pos.p, Vr, p.prow_ro.p,
                                                     p.prow_len.p, p.prow_dp.p);
    MG_LAUNCH_CHECK();
    p.hoff.alloc(Vpad > 0 ? Vpad : 1);
    if (Vpad) MG_CUDA(cudaMemsetAsync(p.hoff.p, 0, sizeof(int32_t) * Vpad, s));
    MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
    if (nb) k_row_smem_offsets<<<grid_for(nb), TPB, 0, s>>>(ps.order.p, p.row_offsets.p, Vr, RB, nb, p.n * p.n,
                                                           p.hoff.p, mx.p);
    MG_LAUNCH_CHECK();
    p.max_patch_hdoubles = to_host_int(mx.p, s);
  }
  // per-row streams padded to whole row blocks (the staged kernels' bulk copies)
  const int64_t Vp = (Vr + RB - 1) / RB * RB;
  p.ell_stride = Vp;
  p.rmeta.alloc(Vp > 0 ? Vp : 1);
  p.ell.alloc(Vp > 0 ? (int64_t)EV_ELL_K * Vp : 1);
  p.ellv.alloc(Vp > 0 ? (int64_t)EV_ELL_K * Vp : 1);
  if (Vp) {
    MG_CUDA(cudaMemsetAsync(p.rmeta.p, 0, sizeof(uint32_t) * Vp, s));
    MG_CUDA(cudaMemsetAsync(p.ell.p, 0, sizeof(uint64_t) * EV_ELL_K * Vp, s));
    MG_CUDA(cudaMemsetAsync(p.ellv.p, 0, sizeof(uint64_t) * EV_ELL_K * Vp, s));
  }
  {
    const bool ident = m.row_order_used == MG_ROW_IDENTITY && !m.owned.p;
    p.order_pad.alloc(!ident && Vp > 0 ? Vp : 1);
    if (!ident && Vp) {
      MG_CUDA(cudaMemsetAsync(p.order_pad.p, 0, sizeof(int32_t) * Vp, s));
      MG_CUDA(cudaMemcpyAsync(p.order_pad.p, ps.order.p, sizeof(int32_t) * Vr, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (Vr) {
    k_row_meta<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.pfix.p, p.prow_dp.p, p.prow_len.p, Vr, p.rmeta.p);
    if (p.with_hessian && p.pattern_ready)
      k_fan_order<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, m.faces.p, Vr, p.rmeta.p);
    k_ell<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, Vr, EV_ELL_K, p.ell.p, Vp);
    k_ellv<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, m.faces.p, Vr, EV_ELL_K, p.ellv.p, Vp);
  }
  MG_LAUNCH_CHECK();
  // CTA face lists (k_cta_dirichlet): each block's distinct faces, per
  // incidence the face's slot in its block list
  p.cf_max = 0;
  if (Vr && m.F) {
    const int64_t F = m.F;
    uint64_t* keys = nullptr;
    MG_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * 3 * F, s));
    k_cf_keys<<<grid_for(3 * F), TPB, 0, s>>>(m.faces.p, F, ps.rank.p, Vr, RB, keys);
    MG_LAUNCH_CHECK();
    int64_t n = sort_unique(keys, 3 * F, 64, s);
    if (n > 0) {
      uint64_t last = 0;
      MG_CUDA(cudaMemcpyAsync(&last, keys + n - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      if (last == ~0ull) --n;
    }
    p.cf_off.alloc(nb + 1);
    p.cf_face.alloc(n > 0 ? n : 1);
    k_lower_bounds<<<grid_for(nb + 1), TPB, 0, s>>>(keys, n, nb, p.cf_off.p);
    if (n) k_cf_faces<<<grid_for(n), TPB, 0, s>>>(keys, n, m.faces.p, ps.rank.p, Vr, RB, p.cf_face.p);
    MG_LAUNCH_CHECK();
    cudaFreeAsync(keys, s);
    int32_t ninc = 0;
    MG_CUDA(cudaMemcpyAsync(&ninc, p.rinc_off.p + Vr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    p.rslot.alloc(ninc > 0 ? ninc : 1);
    p.eslot.alloc((int64_t)EV_ELL_K * Vp);
    MG_CUDA(cudaMemsetAsync(p.eslot.p, 0, sizeof(uint16_t) * EV_ELL_K * Vp, s));
    MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
    k_cf_slots<<<grid_for(Vr), TPB, 0, s>>>(p.rinc_off.p, p.rrec.p, Vr, RB, EV_ELL_K, p.cf_off.p, p.cf_face.p,
                                           p.rslot.p, p.eslot.p, mx.p, Vp);
    MG_LAUNCH_CHECK();
    const bool bad = to_host_int(mx.p, s) != 0;
    MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
    k_max_diff<<<grid_for(nb), TPB, 0, s>>>(p.cf_off.p, nb, mx.p);
    MG_LAUNCH_CHECK();
    p.cf_max = bad ? 0 : to_host_int(mx.p, s);
  }
  MG_CUDA(cudaStreamSynchronize(s));
  p.redo.alloc(1);
  MG_CUDA(cudaMemsetAsync(p.redo.p, 0, sizeof(int), s));
  if (!p.exact_runs.p) {
    p.exact_runs.alloc(1);
    MG_CUDA(cudaMemsetAsync(p.exact_runs.p, 0, sizeof(int), s));
  }
  MG_CUDA(cudaStreamSynchronize(s));
  p.fv_fast = true;
}

void build_patch_layout(Problem& p, cudaStream_t s) {
  Mesh& m = *p.mesh;
  PatchSet& ps = m.patches;
  const int64_t V = m.V, Vr = m.Vr, np = ps.num;  // Vr: rows in patch order
  const int R = ps.R;
  p.layout_ready = false;
  p.ev_jit = false;
  if (V == 0 || np == 0) return;
  p.ev_fast = false;
  {
    bool fast = false;
    for (auto& t : p.terms) fast |= t.dev.op == MG_OP_EV;
    for (auto& t : p.terms)
      fast &= t.dev.op == MG_OP_V || t.dev.type == MG_TERM_SPRING || t.dev.type == MG_TERM_EDGE_LENGTH;
    fast &= m.E < (int64_t(1) << 31);
    if (fast) {
      build_rows_ev(p, s);
      return;
    }
  }
  DBuf<int> flag;
  flag.alloc(1);
  MG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));

  // ops present, and the first term of each op (its bids give row positions)
  const Term* first[2] = {nullptr, nullptr};
  for (auto& t : p.terms) {
    int k = t.dev.op == MG_OP_EV ? 0 : t.dev.op == MG_OP_FV ? 1 : -1;
    if (k >= 0 && !first[k]) first[k] = &t;
  }
  // per-op entry lists
  DBuf<int32_t> pe_of[2];
  uint64_t* rib_keys_all = nullptr;
  int64_t rib_total_keys = 0;
  std::vector<uint64_t*> rib_parts;
  std::vector<int64_t> rib_counts;
  for (int k = 0; k < 2; ++k) {
    OpLayout& L = p.lay[k];
    L.count = 0;
    L.op = -1;
    if (!first[k]) continue;
    const int op = first[k]->dev.op, P = first[k]->dev.P;
    const int64_t M = op_count(m, op);
    const int32_t* sel = op_sel(m, op);
    L.op = op;
    L.P = P;
    uint64_t* keys = nullptr;
    MG_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * (M * P > 0 ? M * P : 1), s));
    if (M) k_patch_elem_keys<<<grid_for(M), TPB, 0, s>>>(sel, P, M, ps.patch_of_vertex.p, keys);
    MG_LAUNCH_CHECK();
    int64_t n = sort_unique(keys, M * P, 64, s);
    if (n > 0) {
      uint64_t last = 0;
      MG_CUDA(cudaMemcpyAsync(&last, keys + n - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      if (last == ~0ull) --n;
    }
    if (n >= (int64_t(1) << 31)) throw Error(MG_ERR_UNSUPPORTED, "patch element lists exceed 2^31 entries");
    L.count = n;
    L.off.alloc(np + 1);
    L.elem.alloc(n > 0 ? n : 1);
    k_lower_bounds<<<grid_for(np + 1), TPB, 0, s>>>(keys, n, np, L.off.p);
    if (n) k_split_entries<<<grid_for(n), TPB, 0, s>>>(keys, n, L.elem.p);
    MG_LAUNCH_CHECK();
    cudaFreeAsync(keys, s);
    pe_of[k].alloc(n > 0 ? n : 1);
    k_patch_of_entry<<<grid_for(np), TPB, 0, s>>>(L.off.p, np, pe_of[k].p);
    MG_LAUNCH_CHECK();
    // ribbon candidates of this op
    uint64_t* rk = nullptr;
    MG_CUDA(cudaMallocAsync(&rk, sizeof(uint64_t) * (n * P > 0 ? n * P : 1), s));
    if (n) k_ribbon_keys<<<grid_for(n), TPB, 0, s>>>(sel, P, L.elem.p, pe_of[k].p, n, ps.patch_of_vertex.p, rk);
    MG_LAUNCH_CHECK();
    rib_parts.push_back(rk);
    rib_counts.push_back(n * P);
    rib_total_keys += n * P;
  }
  // merged ribbon list over all ops
  MG_CUDA(cudaMallocAsync(&rib_keys_all, sizeof(uint64_t) * (rib_total_keys > 0 ? rib_total_keys : 1), s));
  {
    int64_t o = 0;
    for (size_t i = 0; i < rib_parts.size(); ++i) {
      if (rib_counts[i])
        MG_CUDA(cudaMemcpyAsync(rib_keys_all + o, rib_parts[i], sizeof(uint64_t) * rib_counts[i],
                                cudaMemcpyDeviceToDevice, s));
      o += rib_counts[i];
      cudaFreeAsync(rib_parts[i], s);
    }
  }
  int64_t nr = sort_unique(rib_keys_all, rib_total_keys, 64, s);
  if (nr > 0) {
    uint64_t last = 0;
    MG_CUDA(cudaMemcpyAsync(&last, rib_keys_all + nr - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    if (last == ~0ull) --nr;
  }
  ps.ribbon_total = nr;
  DBuf<int32_t> rib_off;
  rib_off.alloc(np + 1);
  k_lower_bounds<<<grid_for(np + 1), TPB, 0, s>>>(rib_keys_all, nr, np, rib_off.p);
  MG_LAUNCH_CHECK();
  p.vtx_off.alloc(np + 1);
  k_vtx_off<<<grid_for(np + 1), TPB, 0, s>>>(rib_off.p, np, R, Vr, p.vtx_off.p);
  p.vtx.alloc(Vr + nr > 0 ? Vr + nr : 1);
  if (Vr) k_fill_owned<<<grid_for(Vr), TPB, 0, s>>>(ps.order.p, Vr, R, p.vtx_off.p, p.vtx.p);
  if (nr) k_fill_ribbon<<<grid_for(nr), TPB, 0, s>>>(rib_keys_all, nr, rib_off.p, R, Vr, p.vtx_off.p, p.vtx.p);
  MG_LAUNCH_CHECK();
  {
    DBuf<int> mx;
    mx.alloc(1);
    MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
    k_max_diff<<<grid_for(np), TPB, 0, s>>>(p.vtx_off.p, np, mx.p);
    MG_LAUNCH_CHECK();
    p.max_patch_vertices = to_host_int(mx.p, s);
  }

  // local ids, row positions, colors; then sort entries by (patch, color, element)
  DBuf<uint64_t> masks;
  masks.alloc(2 * np * R);
  p.recomputed_elements = 0;
  for (int k = 0; k < 2; ++k) {
    OpLayout& L = p.lay[k];
    if (L.op < 0) continue;
    const int P = L.P;
    const int64_t n = L.count;
    const int32_t* sel = op_sel(m, L.op);
    L.local.alloc(n * P > 0 ? n * P : 1);
    if (n) k_local_ids<<<grid_for(n), TPB, 0, s>>>(sel, P, L.elem.p, pe_of[k].p, n, ps.patch_of_vertex.p,
                                                   ps.rank.p, R, Vr, rib_keys_all, rib_off.p, L.local.p, flag.p);
    MG_LAUNCH_CHECK();
    L.pos.alloc(n * P * P > 0 ? n * P * P : 1);
    MG_CUDA(cudaMemsetAsync(L.pos.p, 0xff, n * P * P > 0 ? n * P * P : 1, s));
    if (p.with_hessian && p.pattern_ready && n)
      k_positions<<<grid_for(n), TPB, 0, s>>>(sel, P, L.elem.p, pe_of[k].p, n, ps.patch_of_vertex.p,
                                              first[k]->bids.p, p.row_offsets.p, L.pos.p, flag.p);
    MG_LAUNCH_CHECK();
    L.color.alloc(n > 0 ? n : 1);
    k_color<<<grid_for(np), TPB, 0, s>>>(L.local.p, P, L.off.p, np, R, Vr, masks.p, L.color.p, flag.p);
    MG_LAUNCH_CHECK();
    if (to_host_int(flag.p, s)) {
      // pathological valence / patch: keep the element-parallel path
      cudaFreeAsync(rib_keys_all, s);
      MG_CUDA(cudaStreamSynchronize(s));
      return;
    }
    // reorder entries by (patch, color, element)
    DBuf<uint64_t> ck, ck2;
    DBuf<int32_t> idx, idx2;
    ck.alloc(n > 0 ? n : 1);
    ck2.alloc(n > 0 ? n : 1);
    idx.alloc(n > 0 ? n : 1);
    idx2.alloc(n > 0 ? n : 1);
    if (n) {
      k_color_keys<<<grid_for(n), TPB, 0, s>>>(pe_of[k].p, L.color.p, L.elem.p, n, ck.p, idx.p);
      MG_LAUNCH_CHECK();
      size_t tb = 0;
      MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ck.p, ck2.p, idx.p, idx2.p, n, 0, 64, s));
      {
        Tmp t(s, tb);
        MG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, ck.p, ck2.p, idx.p, idx2.p, n, 0, 64, s));
      }
      DBuf<int32_t> e2;
      DBuf<uint16_t> l2;
      DBuf<uint8_t> p2, c2;
      e2.alloc(n);
      l2.alloc(n * P);
      p2.alloc(n * P * P);
      c2.alloc(n);
      k_gather_rows<<<grid_for(n), TPB, 0, s>>>(L.elem.p, idx2.p, n, 1, e2.p);
      k_gather_rows<<<grid_for(n * P), TPB, 0, s>>>(L.local.p, idx2.p, n, P, l2.p);
      k_gather_rows<<<grid_for(n * P * P), TPB, 0, s>>>(L.pos.p, idx2.p, n, P * P, p2.p);
      k_gather_rows<<<grid_for(n), TPB, 0, s>>>(L.color.p, idx2.p, n, 1, c2.p);
      MG_LAUNCH_CHECK();
      MG_CUDA(cudaStreamSynchronize(s));
      L.elem = std::move(e2);
      L.local = std::move(l2);
      L.pos = std::move(p2);
      L.color = std::move(c2);
    }
    p.recomputed_elements += n - op_count(m, L.op);
  }
  cudaFreeAsync(rib_keys_all, s);

  // shared-memory row offsets of owned rows (patch order) and diagonal positions
  p.hloc.alloc(Vr > 0 ? Vr : 1);
  p.diag_pos.alloc(V);
  p.max_patch_blocks = 0;
  if (p.with_hessian && p.pattern_ready) {
    DBuf<int32_t> len, scan;
    len.alloc(Vr + 1);
    scan.alloc(Vr + 1);
    MG_CUDA(cudaMemsetAsync(len.p + Vr, 0, sizeof(int32_t), s));
    if (Vr) k_row_len_patch_order<<<grid_for(Vr), TPB, 0, s>>>(ps.order.p, p.row_offsets.p, Vr, len.p);
    MG_LAUNCH_CHECK();
    size_t tb = 0;
    MG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, scan.p, Vr + 1, s));
    {
      Tmp t(s, tb);
      MG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, len.p, scan.p, Vr + 1, s));
    }
    if (Vr) k_localize<<<grid_for(Vr), TPB, 0, s>>>(scan.p, Vr, R, p.hloc.p);
    DBuf<int> mx;
    mx.alloc(1);
    MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
    k_patch_blocks<<<grid_for(np), TPB, 0, s>>>(scan.p, Vr, R, np, mx.p);
    k_diag_pos<<<grid_for(V), TPB, 0, s>>>(p.row_offsets.p, p.col32.p, V, p.diag_pos.p);
    MG_LAUNCH_CHECK();
    p.max_patch_blocks = to_host_int(mx.p, s);
  }
  MG_CUDA(cudaStreamSynchronize(s));
  p.fv_fast = false;
  {
    const int t0 = p.terms.size() == 1 ? p.terms[0].dev.type : 0;
    bool fv = (t0 == MG_TERM_SYM_DIRICHLET || t0 == MG_TERM_SPHERE) && p.n == 2 && m.F < (int64_t(1) << 30) &&
              m.F > 0;
    if (fv) build_rows_fv(p, s);
  }
  if (p.patch_module && rows_jit_supported(p)) {  // traced radial edge terms: the row layout too
    build_rows_ev(p, s, false);
    p.ev_fast = false;
    p.ev_jit = true;
  }
  p.layout_ready = true;
}

}  // namespace mg
