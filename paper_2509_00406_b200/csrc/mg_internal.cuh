// Library-internal state shared by the setup, kernel and ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

#include "../../include/meshgrad_b200.h"
#include "terms.cuh"

namespace mg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MG_CUDA(expr)                                                                       \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      throw ::mg::Error(MG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define MG_LAUNCH_CHECK() MG_CUDA(cudaGetLastError())

// Owned device buffer (library-owned state only; caller buffers are raw pointers).
template <class T>
struct DBuf {
  T* p = nullptr;
  int64_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept { reset(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; return *this; }
  ~DBuf() { reset(); }
  void alloc(int64_t count) {
    reset();
    if (count > 0) MG_CUDA(cudaMalloc(&p, sizeof(T) * count));
    n = count;
  }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// Stream-ordered temporary (setup paths).
struct Tmp {
  void* p = nullptr;
  cudaStream_t s;
  explicit Tmp(cudaStream_t st, size_t bytes) : s(st) {
    if (bytes) MG_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  ~Tmp() { if (p) cudaFreeAsync(p, s); }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Vertex patches (RXMesh-style, re-designed for row-owner assembly):
//   owned rows: a contiguous run of the Morton-ordered vertex list;
//   ribbon: vertices referenced by elements incident to owned rows but owned
//   by another patch. Elements incident to owned rows are listed per patch
//   (ribbon elements therefore appear in two or three patches: the owner
//   computes, nobody communicates).
struct PatchSet {
  int64_t num = 0;
  int R = 128;                  // owned rows per patch (last patch may hold fewer)
  DBuf<int32_t> order;          // (V) vertex ids in Morton order; patch p owns order[p*R, p*R+R)
  DBuf<int32_t> rank;           // (V) inverse of order
  DBuf<int32_t> patch_of_vertex;
  int64_t ribbon_total = 0;     // of the most recent problem layout
};

// Per-op element lists of every patch: the elements incident to the patch's
// owned rows (owned + ribbon elements), sorted by (color, element id).
struct OpLayout {
  int op = -1, P = 0;
  int64_t count = 0;
  DBuf<int32_t> off;      // (num_patches+1)
  DBuf<int32_t> elem;     // element id
  DBuf<uint16_t> local;   // (count, P) patch-local vertex index
  DBuf<uint8_t> pos;      // (count, P, P) column position of slot q' in the row of owned slot q (255: none)
  DBuf<uint8_t> color;    // conflict-free color: no two same-color entries share an owned vertex
  int num_colors = 0;
};

struct Mesh {
  int64_t V = 0, E = 0, F = 0;
  // rows this device assembles: all V vertices, or an owned subset when the
  // mesh is one shard of a multi-GPU partition (mg_mesh_set_owned). Patches
  // cover owned vertices only; the others are ribbon (halo) vertices whose x
  // is read but whose rows belong to another device.
  int64_t Vr = 0;
  DBuf<uint8_t> owned;   // (V) 1 = owned, or empty = all owned
  DBuf<int32_t> faces;   // (F,3)
  DBuf<int32_t> edges;   // (E,2) canonical, sorted
  DBuf<double> pos;      // (V,3) or empty
  PatchSet patches;
  int patch_vertices = 128;
  // row processing order: MG_ROW_AUTO picks the caller's numbering when it is
  // translation-regular (consecutive rows have shifted neighbourhoods, as in
  // a structured grid: a warp's neighbour gathers are then contiguous), else
  // Morton order of the positions; row_order_used is the resolved choice
  int row_order = 0;       // MG_ROW_AUTO / MG_ROW_MORTON / MG_ROW_IDENTITY
  int row_order_used = 0;
  double regularity = 0.0;  // fraction of edges (i,j) whose (i+1,j+1) is an edge
};

struct Term {
  TermDev dev;
  int64_t M = 0;               // elements
  DBuf<int32_t> bids;          // (M,P,P) Hessian block ids, -1 = pinned pair
  // traced (JIT) term: driver-API module with the six mode kernels and its
  // per-element attribute streams (caller-owned device arrays)
  bool jit = false;
  void* jit_module = nullptr;
  void* jit_fn[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  std::vector<const double*> jit_attrs;
  // explicit element vertex lists (M, P) (caller-owned device array), e.g. the
  // VV neighbourhoods of one valence group; null: the op's mesh arrays
  const int32_t* sel = nullptr;
  // deterministic gather mode: this term's offsets in the problem's scratch
  int64_t gv_base = 0, gh_base = 0;
};

constexpr int EV_ROW_BLOCK = 64;  // rows (threads) per CTA of the edge row kernel
#ifndef MG_TILE_ROWS
#define MG_TILE_ROWS 128
#endif
constexpr int EV_TILE_ROWS = MG_TILE_ROWS;  // rows per tile of the staged edge kernel (edge_kernels.cu)
#ifndef MG_TILE_VPT
#define MG_TILE_VPT 2
#endif
constexpr int EV_TILE_VPT = MG_TILE_VPT;    // vertex-table entries per thread (max_v <= VPT * rows)
constexpr int EV_TILE_EPT = 5;    // edge-table entries per thread
constexpr int EV_ELL_K = 6;       // incidences per row stored slot-major (ELL); the rest stay CSR

struct Problem {
  Mesh* mesh = nullptr;
  int n = 3;
  bool with_hessian = true;
  bool deterministic = true;
  DBuf<uint8_t> fixed;         // (V)
  bool any_fixed = false;
  std::vector<Term> terms;
  bool pattern_ready = false;
  bool layout_ready = false;
  int64_t nnzb = 0;
  DBuf<int64_t> row_offsets;   // (V+1)
  DBuf<int64_t> col_indices;   // (nnzb)
  DBuf<int32_t> col32;         // (nnzb)
  DBuf<double> partials;       // energy partials
  int64_t partial_cap = 0;
  int last_launches = 0;
  // patch-owner assembly state (build_patch_layout)
  OpLayout lay[2];             // [0] EV, [1] FV
  DBuf<int32_t> vtx_off;       // (num_patches+1) patch vertex lists: owned rows, then ribbon
  DBuf<int32_t> vtx;
  DBuf<int32_t> hloc;          // (V, patch order) smem block offset of each owned row
  DBuf<uint8_t> diag_pos;      // (V) position of the diagonal block in its row (255: none)
  int max_patch_vertices = 0;
  int max_patch_blocks = 0;
  int max_patch_elems = 0;     // max EV entries of one patch
  // edge row kernel (all EV terms radial, no FV terms): one thread per owned
  // row, rows in patch order; per row its incident edges in column order
  bool ev_fast = false;
  // staged edge tiles (tile_setup in patch_setup.cu, kernels in edge_kernels.cu):
  // per tile of EV_TILE_ROWS rows, its vertex table (rows, then halo vertices;
  // vertex | pinned << 31), its edge table (edge | local a << 32 | local b << 48)
  // and, per incidence (parallel to rrec), the edge's slot | (row is b) << 15
  bool tiles_ready = false;
  DBuf<int32_t> te_off;         // setup only
  DBuf<int2> tcnt;              // (tiles) vertex / edge table lengths
  DBuf<uint32_t> tv;            // (tiles, max_v) padded
  DBuf<uint64_t> te;            // (tiles, max_e) padded
  DBuf<uint16_t> islot, islot8;
  int tile_max_v = 0, tile_max_e = 0;
  bool fv_fast = false;        // face row kernel (single SymDirichlet term), generic path as exact fallback
  DBuf<int32_t> rinc_off;      // (Vr+1)
  DBuf<uint64_t> rrec;         // (incidences) lo: edge | slot << 31, hi: other | pinned(other) << 31
  DBuf<uint8_t> pfix;          // (Vr) pinned flag of each row
  DBuf<uint32_t> rmeta;        // (Vr) incidence count (sat. 255) | pinned << 8 | diagonal position << 16
  DBuf<uint64_t> ell;          // (EV_ELL_K, Vr) first incidences of each row, slot-major
  DBuf<uint32_t> ell32;        // (EV_ELL_K, Vr) vertex-only 32-bit records (k_ell32): gradient / HVP edge rows
  int64_t ell_stride = 0;      // edge rows: slot stride of ell / ell32 (Vr padded to whole row blocks)
  DBuf<int32_t> order_pad;     // edge rows: the row order padded to whole row blocks (staged kernels)
  bool ell32_ok = false;       // built (no EV term reads a per-edge attribute)
  DBuf<uint64_t> ellv;         // face rows: (EV_ELL_K, Vr) the incidence's other two corners (s+1 | s+2 << 32)
  // face rows, CTA face lists (k_cta_dirichlet): per EV_ROW_BLOCK rows its
  // distinct faces (face | corner 0 in block << 31); per incidence its slot
  DBuf<int32_t> cf_off;        // (blocks + 1)
  DBuf<int4> cf_face;          // {face | corner 0 in block << 31, corners}
  DBuf<uint16_t> eslot;        // (EV_ELL_K, Vr)
  DBuf<uint16_t> rslot;        // (incidences), parallel to rrec
  int cf_max = 0;              // max faces of one block; 0: lists not built
  DBuf<int64_t> prow_ro;       // (Vr) row start
  DBuf<int32_t> prow_len;      // (Vr) row length (blocks)
  DBuf<uint8_t> prow_dp;       // (Vr) diagonal block position (255: none)
  DBuf<int32_t> hoff;          // (Vr) row-buffer offset (doubles) in its CTA, 16-byte phase matched
  int max_patch_hdoubles = 0;  // max row-buffer doubles of one CTA
  DBuf<int> redo;              // (1) non-finite lane seen by the radial kernel; cleared by the energy reduction
  DBuf<int> exact_runs;        // (1) calls whose exact re-run executed (diagnostics)
  mutable DBuf<double> vscr;   // sphere face kernel: per-vertex retraction scratch (V, 6)
  mutable DBuf<double> fpsd;   // Dirichlet face kernel under a PSD clamp: per face P_f(M) (F, 10)
  mutable DBuf<double> fpsd6;  // ... and for faces with a pinned corner the clamped masked 6x6 (F, 21)
  // deterministic element-parallel mode (gather.cu): per-element output
  // scratch and, per output row / block, its contributions in fixed order
  bool gather_ready = false;
  DBuf<double> gsv, gsh;
  DBuf<int64_t> gv_off, gv_idx, gh_off, gh_idx;
  // optional device timing of the main assembly kernel (benchmarks)
  bool timing = false;
  mutable std::vector<cudaEvent_t> ev_pool;
  mutable std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pairs;
  mutable cudaEvent_t ev_open = nullptr;
  int64_t recomputed_elements = 0;
  // traced terms on the patch path (jit_patch.cuh): the problem's generated
  // patch module (5 mode kernels) and its terms' attribute-pointer table
  void* patch_module = nullptr;
  void* patch_fn[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  mutable DBuf<const double*> jattr;
  mutable bool jattr_dirty = true;
  DBuf<double> pcg_ws;         // device PCG workspace (pcg.cu)
  // traced terms on the edge row kernel (jit_rows.cuh): every EV callback
  // radial (proved by the tracer), V terms at the row; the patch module is
  // the exact re-run. ev_jit: its row layout is built.
  void* row_module = nullptr;
  void* row_fn[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool ev_jit = false;
  // fp32 storage of x, w, gradient, Hessian values, HVP and the builtin terms'
  // attributes (mg_problem_set_storage): the edge row kernels only
  bool store32 = false;
};

// element vertex ids of an op (nullptr for V: the element is the vertex)
inline const int32_t* op_sel(const Mesh& m, int op) {
  if (op == MG_OP_FV) return m.faces.p;
  if (op == MG_OP_EV) return m.edges.p;
  return nullptr;
}
inline const int32_t* term_sel(const Mesh& m, const Term& t) { return t.sel ? t.sel : op_sel(m, t.dev.op); }
inline int64_t op_count(const Mesh& m, int op) {
  if (op == MG_OP_FV) return m.F;
  if (op == MG_OP_EV) return m.E;
  return m.V;
}

// setup.cu
void mesh_build(Mesh& m, const int64_t* faces_d, const int64_t* edges_d, int64_t num_edges_in,
                const double* pos_d, cudaStream_t s);
void build_pattern(Problem& p, cudaStream_t s);
void build_patch_layout(Problem& p, cudaStream_t s);
void build_rows_ev(Problem& p, cudaStream_t s, bool tiles = true);
void build_rows_fv(Problem& p, cudaStream_t s);
void mesh_patches(Mesh& m, cudaStream_t s);
void mesh_set_owned(Mesh& m, const uint8_t* owned_d, cudaStream_t s);
int64_t sort_unique(uint64_t*& keys, int64_t n, int end_bit, cudaStream_t s);

// jit_host.cu (traced terms through the driver API)
struct LaunchCtx;
void jit_load(Term& t, const void* image);
void jit_unload(Term& t);
void jit_patch_load(Problem& p, const void* image);
void jit_patch_unload(Problem& p);
void jit_rows_load(Problem& p, const void* image);
void jit_rows_unload(Problem& p);


// elem_kernels.cu (element-parallel, atomic accumulation)
enum Mode { MODE_ENERGY = 0, MODE_GRAD = 1, MODE_HESS = 2, MODE_HVP = 3 };
// launch the problem's traced patch kernel for a mode (args: the filled
// patch::PatchArgs, passed as void* to keep this header light)
void jit_patch_launch(const Problem& p, Mode mode, bool psd, void* args, int64_t np, int nvp_max,
                      int blocks_max, size_t smem, cudaStream_t s, int64_t grid = -1);
// launch the problem's traced row kernel (args: a filled rows::EvArgs)
void jit_rows_launch(const Problem& p, Mode mode, bool psd, void* args, int64_t grid, int block, size_t smem,
                     cudaStream_t s, bool persistent);

struct LaunchCtx {
  const double* x;
  const double* w;     // hvp direction
  const uint8_t* fixed;
  double* grad;
  double* hess;
  double* y;
  double* partials;    // energy partials
  bool psd;
  double floor;
  cudaStream_t stream;
  bool scratch = false;  // deterministic gather mode: elements write Problem::gsv / gsh
};
// Launch one term element-parallel; returns number of energy partials written.
int64_t launch_elem(const Problem& p, const Term& t, Mode mode, const LaunchCtx& c,
                    int64_t partial_offset);
void jit_launch(const Problem& p, const Term& t, Mode mode, const LaunchCtx& c, int64_t partial_offset);
int64_t elem_partials_needed(const Term& t);
// patch_kernels.cu (deterministic row-owner assembly)
int64_t launch_patch(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset);
// edge_kernels.cu (two-point edge fast path of the patch-owner assembly)
int64_t launch_patch_ev(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset);
// ... with the problem's traced row module (returns the energy partials written)
int64_t launch_rows_jit(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset);
bool rows_jit_supported(const Problem& p);
// face_kernels.cu (face row kernel)
int64_t launch_patch_fv(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset);
// timing hooks around the main kernel (no-ops unless p.timing)
void timing_begin(const Problem& p, cudaStream_t s);
void timing_end(const Problem& p, cudaStream_t s);
bool patch_supported(const Problem& p);
// gather.cu (deterministic element-parallel accumulation)
void build_gather(Problem& p, cudaStream_t s);
void gather_vec(const Problem& p, double* out, cudaStream_t s);
void gather_blocks(const Problem& p, double* out, cudaStream_t s);
// fixed-order reduction of energy partials -> out[0]
// (partials buffers carry REDUCE_TAIL spare slots after the largest n: chunk sums)
constexpr int64_t REDUCE_TAIL = 1 << 16;
void reduce_partials(const double* partials, int64_t n, double* out, cudaStream_t s, int* clear_flag = nullptr);
inline int reduce_launches(int64_t n) { return n > 4 * 2048 ? 2 : 1; }
void launch_bsr_matvec(const Problem& p, const double* H, const double* v, double* y, cudaStream_t s);
void launch_block_jacobi(const Problem& p, const double* H, double* inv, cudaStream_t s);
void launch_block_apply(const Problem& p, const double* inv, const double* r, double* y, cudaStream_t s);
// pcg.cu: truncated block-Jacobi PCG on the device (status: 1 converged,
// 2 non-positive curvature, 3 max iterations)
void pcg_solve(Problem& p, const double* hess, const std::function<void(const double*, double*)>& apply_hvp,
               const double* inv, const double* b, double tol, int max_iters, double* out, int* iters,
               int* status, cudaStream_t s);

}  // namespace mg
