// C ABI (include/meshgrad_b200.h): state management and orchestration.
#include <cstring>
#include <string>

#include "jit_abi.h"
#include "mg_internal.cuh"

using namespace mg;

struct mg_mesh {
  Mesh m;
};
struct mg_problem {
  Problem p;
  mg_mesh* mesh;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return MG_OK;
  } catch (const Error& e) {
    return fail(e.code, e.what());
  } catch (const std::exception& e) {
    return fail(MG_ERR_CUDA, e.what());
  }
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int natural_op(int type) {
  switch (type) {
    case MG_TERM_INERTIA: return MG_OP_V;
    case MG_TERM_SPRING: return MG_OP_EV;
    case MG_TERM_GRAVITY: return MG_OP_V;
    case MG_TERM_EDGE_LENGTH: return MG_OP_EV;
    case MG_TERM_SYM_DIRICHLET: return MG_OP_FV;
    case MG_TERM_SPHERE: return MG_OP_FV;
    default: return -1;
  }
}
int natural_P(int op) { return op == MG_OP_FV ? 3 : op == MG_OP_EV ? 2 : 1; }
int attrs_needed(int type) {
  switch (type) {
    case MG_TERM_INERTIA: return 2;
    case MG_TERM_SPRING: return 1;
    case MG_TERM_GRAVITY: return 1;
    case MG_TERM_EDGE_LENGTH: return 0;
    case MG_TERM_SYM_DIRICHLET: return 2;
    case MG_TERM_SPHERE: return 3;
    default: return 0;
  }
}
const char* op_name(int op) {
  switch (op) {
    case MG_OP_FV: return "FV";
    case MG_OP_EV: return "EV";
    case MG_OP_VV: return "VV";
    default: return "V";
  }
}

void ensure_ready(Problem& p, cudaStream_t s) {
  if (p.terms.empty()) throw Error(MG_ERR_VALUE, "no energy terms registered");
  if (p.with_hessian && !p.pattern_ready) build_pattern(p, s);
  if (p.deterministic && !p.layout_ready && patch_supported(p)) build_patch_layout(p, s);
}

void ensure_partials(Problem& p, int64_t need) {
  need += REDUCE_TAIL;
  if (need > p.partial_cap) {
    p.partials.alloc(need);
    p.partial_cap = need;
  }
}

// fp32 storage runs on the edge row kernels only
void require_storage(const Problem& p) {
  if (p.store32 && !(p.ev_fast && p.layout_ready && p.deterministic))
    throw Error(MG_ERR_UNSUPPORTED, "float32 storage runs on the edge row kernels: deterministic problems with "
                                    "builtin vertex and radial edge terms only");
}

int64_t partials_needed(const Problem& p) {
  int64_t need = 1;
  for (auto& t : p.terms) need += elem_partials_needed(t);
  if (p.mesh->patches.num > need) need = p.mesh->patches.num;
  // edge row / tile kernels: one partial per warp of (tile-rounded) rows
  const int64_t nwarps = (p.mesh->Vr + EV_TILE_ROWS - 1) / EV_TILE_ROWS * (EV_TILE_ROWS / 32);
  if (nwarps > need) need = nwarps;
  return need + 1;
}

}  // namespace

namespace mg {
static cudaEvent_t take_event(const Problem& p) {
  if (!p.ev_pool.empty()) {
    cudaEvent_t e = p.ev_pool.back();
    p.ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  MG_CUDA(cudaEventCreate(&e));
  return e;
}
void timing_begin(const Problem& p, cudaStream_t s) {
  if (!p.timing) return;
  p.ev_open = take_event(p);
  MG_CUDA(cudaEventRecord(p.ev_open, s));
}
void timing_end(const Problem& p, cudaStream_t s) {
  if (!p.timing || !p.ev_open) return;
  cudaEvent_t e = take_event(p);
  MG_CUDA(cudaEventRecord(e, s));
  p.ev_pairs.emplace_back(p.ev_open, e);
  p.ev_open = nullptr;
}
}  // namespace mg

extern "C" {

const char* mg_last_error(void) { return g_err.c_str(); }
int mg_abi_version(void) { return MG_ABI_VERSION; }

int mg_mesh_create(const int64_t* faces_d, int64_t num_faces, const int64_t* edges_d,
                   int64_t num_edges, int64_t num_vertices, const double* positions_d,
                   int patch_vertices, void* stream, mg_mesh** out) {
  if (!out) return fail(MG_ERR_VALUE, "out is NULL");
  if (num_vertices < 0 || num_faces < 0 || num_edges < 0) return fail(MG_ERR_VALUE, "negative size");
  // the face / edge row kernels write one energy partial per 32-row warp; a
  // patch of >= 32 rows keeps the generic patch kernel's partial count within it
  if (patch_vertices > 0 && patch_vertices < 32) return fail(MG_ERR_VALUE, "patch_vertices must be >= 32");
  auto* h = new mg_mesh();
  int rc = guard([&] {
    h->m.V = num_vertices;
    h->m.F = num_faces;
    h->m.patch_vertices = patch_vertices > 0 ? patch_vertices : 128;
    mesh_build(h->m, faces_d, edges_d, num_edges, positions_d, S(stream));
  });
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return MG_OK;
}

int mg_mesh_counts(const mg_mesh* mesh, int64_t* V, int64_t* E, int64_t* F, int64_t* P) {
  if (!mesh) return fail(MG_ERR_VALUE, "mesh is NULL");
  if (V) *V = mesh->m.V;
  if (E) *E = mesh->m.E;
  if (F) *F = mesh->m.F;
  if (P) *P = mesh->m.patches.num;
  return MG_OK;
}

namespace {
__global__ void k_widen_pairs(const int32_t* in, int64_t n, int64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}
}  // namespace

int mg_mesh_copy_edges(const mg_mesh* mesh, int64_t* edges_d, void* stream) {
  if (!mesh) return fail(MG_ERR_VALUE, "mesh is NULL");
  return guard([&] {
    int64_t n = 2 * mesh->m.E;
    if (n) k_widen_pairs<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(mesh->m.edges.p, n, edges_d);
    MG_LAUNCH_CHECK();
  });
}

int mg_mesh_copy_vertex_patches(const mg_mesh* mesh, int32_t* patch_d, void* stream) {
  if (!mesh) return fail(MG_ERR_VALUE, "mesh is NULL");
  if (!mesh->m.patches.num) return fail(MG_ERR_STATE, "patches are built with the first deterministic problem");
  return guard([&] {
    MG_CUDA(cudaMemcpyAsync(patch_d, mesh->m.patches.patch_of_vertex.p, sizeof(int32_t) * mesh->m.V,
                            cudaMemcpyDeviceToDevice, S(stream)));
  });
}

int mg_mesh_set_owned(mg_mesh* mesh, const uint8_t* owned_d, void* stream) {
  if (!mesh) return fail(MG_ERR_VALUE, "mesh is NULL");
  return guard([&] { mesh_set_owned(mesh->m, owned_d, S(stream)); });
}

int mg_mesh_set_row_order(mg_mesh* mesh, int order, void* stream) {
  if (!mesh) return fail(MG_ERR_VALUE, "mesh is NULL");
  if (order < MG_ROW_AUTO || order > MG_ROW_IDENTITY) return fail(MG_ERR_VALUE, "unknown row order");
  return guard([&] {
    if (mesh->m.row_order == order) return;
    mesh->m.row_order = order;
    mesh_patches(mesh->m, S(stream));
    MG_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int mg_mesh_row_order(const mg_mesh* mesh, int* order, double* regularity) {
  if (!mesh || !order) return fail(MG_ERR_VALUE, "NULL argument");
  *order = mesh->m.row_order_used;
  if (regularity) *regularity = mesh->m.regularity;
  return MG_OK;
}

int mg_mesh_destroy(mg_mesh* mesh) {
  delete mesh;
  return MG_OK;
}

int mg_problem_create(mg_mesh* mesh, int var_dim, int with_hessian, const uint8_t* fixed_mask_d,
                      int deterministic, mg_problem** out) {
  if (!mesh || !out) return fail(MG_ERR_VALUE, "mesh/out is NULL");
  if (var_dim < 1) return fail(MG_ERR_VALUE, "var_dim must be at least 1");
  auto* h = new mg_problem();
  int rc = guard([&] {
    h->mesh = mesh;
    Problem& p = h->p;
    p.mesh = &mesh->m;
    p.n = var_dim;
    p.with_hessian = with_hessian != 0;
    p.deterministic = deterministic != 0;
    const int64_t V = mesh->m.V;
    p.fixed.alloc(V > 0 ? V : 1);
    if (fixed_mask_d && V) {
      MG_CUDA(cudaMemcpy(p.fixed.p, fixed_mask_d, V, cudaMemcpyDeviceToDevice));
      std::vector<uint8_t> hm(V);
      MG_CUDA(cudaMemcpy(hm.data(), fixed_mask_d, V, cudaMemcpyDeviceToHost));
      for (auto b : hm) p.any_fixed |= (b != 0);
    } else if (V) {
      MG_CUDA(cudaMemset(p.fixed.p, 0, V));
    }
  });
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return MG_OK;
}

int mg_problem_add_term(mg_problem* prob, int term_type, int op, const double* params, int num_params,
                        const double* const* attrs_d, int num_attrs, int* term_id) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  const int nat = natural_op(term_type);
  if (nat < 0) return fail(MG_ERR_VALUE, "unknown builtin term type " + std::to_string(term_type));
  if (op != MG_OP_FV && op != MG_OP_EV && op != MG_OP_VV && op != MG_OP_V)
    return fail(MG_ERR_VALUE, "op does not resolve to vertex variables; terms support FV, EV, VV, V");
  if (op != nat)
    return fail(MG_ERR_VALUE, std::string("builtin term iterates over op ") + op_name(nat) + ", not " + op_name(op));
  if (num_params < 0 || num_params > 6) return fail(MG_ERR_VALUE, "at most 6 scalar params");
  if (num_attrs != attrs_needed(term_type))
    return fail(MG_ERR_VALUE, "term needs " + std::to_string(attrs_needed(term_type)) + " attribute arrays");
  if (term_type == MG_TERM_GRAVITY && num_params != 1 + prob->p.n)
    return fail(MG_ERR_VALUE, "gravity needs params [h2, g_0..g_{n-1}]");
  if ((term_type == MG_TERM_SYM_DIRICHLET || term_type == MG_TERM_SPHERE) && prob->p.n != 2)
    return fail(MG_ERR_VALUE, "term requires var_dim == 2");
  if ((term_type != MG_TERM_SYM_DIRICHLET && term_type != MG_TERM_SPHERE) && (prob->p.n < 2 || prob->p.n > 3))
    return fail(MG_ERR_UNSUPPORTED, "builtin vertex/edge terms support var_dim 2 or 3");
  Term t;
  std::memset(&t.dev, 0, sizeof(t.dev));
  t.dev.type = term_type;
  t.dev.op = op;
  t.dev.P = natural_P(op);
  for (int i = 0; i < num_params; ++i) t.dev.c[i] = params[i];
  for (int i = 0; i < num_attrs; ++i) t.dev.a[i] = attrs_d[i];
  t.M = op_count(prob->p.mesh[0], op);
  prob->p.terms.push_back(std::move(t));
  jit_patch_unload(prob->p);  // a generated patch / row module covers the terms it was built for
    jit_rows_unload(prob->p);
  prob->p.pattern_ready = false;
  prob->p.layout_ready = false;
  prob->p.gather_ready = false;
  if (term_id) *term_id = (int)prob->p.terms.size() - 1;
  return MG_OK;
}

int mg_problem_add_jit_term(mg_problem* prob, int op, int var_dim, const void* image, const double* const* attrs_d,
                            int num_attrs, int* term_id) {
  if (!prob || !image) return fail(MG_ERR_VALUE, "problem/image is NULL");
  if (op != MG_OP_FV && op != MG_OP_EV && op != MG_OP_V)
    return fail(MG_ERR_UNSUPPORTED, "traced terms support the FV, EV and V ops");
  if (var_dim != prob->p.n) return fail(MG_ERR_VALUE, "traced module was generated for another var_dim");
  if (num_attrs < 0 || num_attrs > JIT_MAX_ATTRS) return fail(MG_ERR_VALUE, "at most 64 attribute streams");
  return guard([&] {
    Term t;
    std::memset(&t.dev, 0, sizeof(t.dev));
    t.dev.type = MG_TERM_JIT;
    t.dev.op = op;
    t.dev.P = natural_P(op);
    t.M = op_count(prob->p.mesh[0], op);
    t.jit = true;
    for (int i = 0; i < num_attrs; ++i) t.jit_attrs.push_back(attrs_d[i]);
    jit_load(t, image);
    prob->p.terms.push_back(std::move(t));
  jit_patch_unload(prob->p);  // a generated patch / row module covers the terms it was built for
    jit_rows_unload(prob->p);
    prob->p.pattern_ready = false;
    prob->p.layout_ready = false;
    prob->p.gather_ready = false;
    if (term_id) *term_id = (int)prob->p.terms.size() - 1;
  });
}

int mg_problem_add_jit_term_sel(mg_problem* prob, int op, int var_dim, int P, const int32_t* sel_d, int64_t M,
                                const void* image, const double* const* attrs_d, int num_attrs, int* term_id) {
  if (!prob || !image) return fail(MG_ERR_VALUE, "problem/image is NULL");
  if (op != MG_OP_VV) return fail(MG_ERR_UNSUPPORTED, "explicit selections are for VV neighbourhood terms");
  if (var_dim != prob->p.n) return fail(MG_ERR_VALUE, "traced module was generated for another var_dim");
  if (P < 1 || P > 33) return fail(MG_ERR_VALUE, "VV neighbourhoods have 1..33 vertices (valence cap 32)");
  if (M < 0 || (M > 0 && !sel_d)) return fail(MG_ERR_VALUE, "selection is NULL");
  if (num_attrs < 0 || num_attrs > JIT_MAX_ATTRS) return fail(MG_ERR_VALUE, "at most 64 attribute streams");
  return guard([&] {
    Term t;
    std::memset(&t.dev, 0, sizeof(t.dev));
    t.dev.type = MG_TERM_JIT;
    t.dev.op = op;
    t.dev.P = P;
    t.M = M;
    t.sel = sel_d;
    t.jit = true;
    for (int i = 0; i < num_attrs; ++i) t.jit_attrs.push_back(attrs_d[i]);
    jit_load(t, image);
    prob->p.terms.push_back(std::move(t));
  jit_patch_unload(prob->p);  // a generated patch / row module covers the terms it was built for
    jit_rows_unload(prob->p);
    prob->p.pattern_ready = false;
    prob->p.layout_ready = false;
    prob->p.gather_ready = false;
    if (term_id) *term_id = (int)prob->p.terms.size() - 1;
  });
}

int mg_problem_set_patch_module(mg_problem* prob, const void* image) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  return guard([&] {
    Problem& p = prob->p;
    if (!image) {
      jit_patch_unload(p);
    } else {
      for (auto& t : p.terms)
        if (!t.jit || t.dev.op == MG_OP_VV) throw Error(MG_ERR_VALUE, "a patch module needs every term traced (no VV)");
      jit_patch_load(p, image);
    }
    p.layout_ready = false;  // the next call builds (or drops) the patch layout
  });
}

int mg_problem_set_row_module(mg_problem* prob, const void* image) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  return guard([&] {
    Problem& p = prob->p;
    if (!image) {
      jit_rows_unload(p);
    } else {
      for (auto& t : p.terms)
        if (!t.jit || (t.dev.op != MG_OP_V && t.dev.op != MG_OP_EV))
          throw Error(MG_ERR_VALUE, "a row module needs every term traced, V or EV");
      jit_rows_load(p, image);
    }
    p.layout_ready = false;  // the next call builds (or drops) the row layout
  });
}

int mg_problem_set_storage(mg_problem* prob, int bits) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  if (bits != 32 && bits != 64) return fail(MG_ERR_VALUE, "storage is 32 or 64 bits");
  prob->p.store32 = bits == 32;
  return MG_OK;
}

int mg_problem_set_jit_attr(mg_problem* prob, int term_id, int slot, const double* attr_d) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  if (term_id < 0 || term_id >= (int)prob->p.terms.size() || !prob->p.terms[term_id].jit)
    return fail(MG_ERR_VALUE, "not a traced term");
  auto& at = prob->p.terms[term_id].jit_attrs;
  if (slot < 0 || slot >= (int)at.size()) return fail(MG_ERR_VALUE, "bad attribute slot");
  at[slot] = attr_d;
  prob->p.jattr_dirty = true;
  return MG_OK;
}

int mg_problem_set_attr(mg_problem* prob, int term_id, int slot, const double* attr_d) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  if (term_id < 0 || term_id >= (int)prob->p.terms.size()) return fail(MG_ERR_VALUE, "bad term id");
  if (slot < 0 || slot >= 4) return fail(MG_ERR_VALUE, "bad attribute slot");
  prob->p.terms[term_id].dev.a[slot] = attr_d;
  return MG_OK;
}

int mg_precompute_sparsity(mg_problem* prob, int64_t* nnzb, void* stream) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  return guard([&] {
    Problem& p = prob->p;
    if (p.terms.empty()) throw Error(MG_ERR_VALUE, "no energy terms registered");
    build_pattern(p, S(stream));
    if (p.deterministic && patch_supported(p)) build_patch_layout(p, S(stream));
    if (nnzb) *nnzb = p.nnzb;
  });
}

int mg_copy_pattern(const mg_problem* prob, int64_t* row_offsets_d, int64_t* col_indices_d, void* stream) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  if (!prob->p.pattern_ready) return fail(MG_ERR_STATE, "sparsity pattern not computed");
  return guard([&] {
    const Problem& p = prob->p;
    MG_CUDA(cudaMemcpyAsync(row_offsets_d, p.row_offsets.p, sizeof(int64_t) * (p.mesh->V + 1),
                            cudaMemcpyDeviceToDevice, S(stream)));
    if (p.nnzb)
      MG_CUDA(cudaMemcpyAsync(col_indices_d, p.col_indices.p, sizeof(int64_t) * p.nnzb,
                              cudaMemcpyDeviceToDevice, S(stream)));
  });
}

int mg_eval(mg_problem* prob, const double* x_d, int use_psd, double psd_floor, double* energy_d,
            double* grad_d, double* hess_d, void* stream) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  Problem& p = prob->p;
  if (use_psd && !p.with_hessian) return fail(MG_ERR_VALUE, "psd_floor requires a Hessian-mode problem");
  if (use_psd && !(psd_floor > 0)) return fail(MG_ERR_VALUE, "floor must be positive");
  if (!x_d || !energy_d || !grad_d) return fail(MG_ERR_VALUE, "x/energy/grad must be non-NULL");
  if (p.with_hessian && !hess_d && p.nnzb) return fail(MG_ERR_VALUE, "hess must be non-NULL in Hessian mode");
  return guard([&] {
    cudaStream_t s = S(stream);
    ensure_ready(p, s);
    require_storage(p);
    ensure_partials(p, partials_needed(p));
    LaunchCtx c{x_d, nullptr, p.any_fixed ? p.fixed.p : nullptr, grad_d, hess_d, nullptr,
                p.partials.p, use_psd != 0, psd_floor, s};
    const Mode mode = p.with_hessian ? MODE_HESS : MODE_GRAD;
    int launches = 0;
    int64_t np = 0;
    if (p.deterministic && p.layout_ready) {
      np = launch_patch(p, mode, c, 0);
      launches += (p.ev_fast || p.fv_fast || p.ev_jit) ? 2 : 1;
    } else if (p.deterministic) {  // element-parallel into scratch, fixed-order gather
      if (!p.gather_ready) build_gather(p, s);
      c.scratch = true;
      for (auto& t : p.terms) {
        np += launch_elem(p, t, mode, c, np);
        ++launches;
      }
      gather_vec(p, grad_d, s);
      ++launches;
      if (p.with_hessian && p.nnzb) {
        gather_blocks(p, hess_d, s);
        ++launches;
      }
    } else {
      MG_CUDA(cudaMemsetAsync(grad_d, 0, sizeof(double) * p.n * p.mesh->V, s));
      if (p.with_hessian && p.nnzb)
        MG_CUDA(cudaMemsetAsync(hess_d, 0, sizeof(double) * p.n * p.n * p.nnzb, s));
      for (auto& t : p.terms) {
        np += launch_elem(p, t, mode, c, np);
        ++launches;
      }
    }
    reduce_partials(p.partials.p, np, energy_d, s,
                    (p.ev_fast || p.fv_fast || p.ev_jit) && p.deterministic && p.layout_ready ? p.redo.p : nullptr);
    p.last_launches = launches + reduce_launches(np);
  });
}

int mg_energy(mg_problem* prob, const double* x_d, double* energy_d, void* stream) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  Problem& p = prob->p;
  if (!x_d || !energy_d) return fail(MG_ERR_VALUE, "x/energy must be non-NULL");
  if (p.terms.empty()) return fail(MG_ERR_VALUE, "no energy terms registered");
  return guard([&] {
    cudaStream_t s = S(stream);
    if (p.store32) {
      ensure_ready(p, s);
      require_storage(p);
    }
    ensure_partials(p, partials_needed(p));
    LaunchCtx c{x_d, nullptr, nullptr, nullptr, nullptr, nullptr, p.partials.p, false, 0.0, s};
    int64_t np = 0;
    int launches = 0;
    if (p.ev_fast && p.layout_ready) {
      // builtin radial terms: the edge row kernel's probe mode (each edge at its
      // first vertex, every value in the reference's own operations)
      np = launch_patch_ev(p, MODE_ENERGY, c, 0);
      launches = 1;
    } else {
      for (auto& t : p.terms) {
        np += launch_elem(p, t, MODE_ENERGY, c, np);
        ++launches;
      }
    }
    reduce_partials(p.partials.p, np, energy_d, s);
    p.last_launches = launches + reduce_launches(np);
  });
}

int mg_hvp(mg_problem* prob, const double* x_d, const double* v_d, int use_psd, double psd_floor,
           double* y_d, void* stream) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  Problem& p = prob->p;
  if (use_psd && !(psd_floor > 0)) return fail(MG_ERR_VALUE, "floor must be positive");
  if (!x_d || !v_d || !y_d) return fail(MG_ERR_VALUE, "x/v/y must be non-NULL");
  if (p.terms.empty()) return fail(MG_ERR_VALUE, "no energy terms registered");
  return guard([&] {
    cudaStream_t s = S(stream);
    if (p.deterministic) ensure_ready(p, s);
    require_storage(p);
    ensure_partials(p, partials_needed(p));
    LaunchCtx c{x_d, v_d, p.any_fixed ? p.fixed.p : nullptr, nullptr, nullptr, y_d,
                p.partials.p, use_psd != 0, psd_floor, s};
    int launches = 0;
    if (p.deterministic && p.layout_ready) {
      launch_patch(p, MODE_HVP, c, 0);
      launches = 1;
      if (p.ev_fast || p.fv_fast || p.ev_jit) {
        MG_CUDA(cudaMemsetAsync(p.redo.p, 0, sizeof(int), s));
        launches = 2;
      }
    } else if (p.deterministic) {
      if (!p.gather_ready) build_gather(p, s);
      c.scratch = true;
      for (auto& t : p.terms) {
        launch_elem(p, t, MODE_HVP, c, 0);
        ++launches;
      }
      gather_vec(p, y_d, s);
      ++launches;
    } else {
      MG_CUDA(cudaMemsetAsync(y_d, 0, sizeof(double) * p.n * p.mesh->V, s));
      for (auto& t : p.terms) {
        launch_elem(p, t, MODE_HVP, c, 0);
        ++launches;
      }
    }
    p.last_launches = launches;
  });
}

int mg_bsr_matvec(const mg_problem* prob, const double* hess_d, const double* v_d, double* y_d, void* stream) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  if (prob->p.store32) return fail(MG_ERR_UNSUPPORTED, "the BSR kernels are fp64 (float32 storage: eval / hvp / energy)");
  if (!prob->p.pattern_ready) return fail(MG_ERR_STATE, "sparsity pattern not computed");
  return guard([&] { launch_bsr_matvec(prob->p, hess_d, v_d, y_d, S(stream)); });
}

int mg_bsr_block_jacobi(const mg_problem* prob, const double* hess_d, double* inv_d, void* stream) {
  if (!prob || !hess_d || !inv_d) return fail(MG_ERR_VALUE, "NULL argument");
  if (!prob->p.pattern_ready) return fail(MG_ERR_STATE, "sparsity pattern not computed");
  return guard([&] { launch_block_jacobi(prob->p, hess_d, inv_d, S(stream)); });
}

int mg_block_apply(const mg_problem* prob, const double* inv_d, const double* r_d, double* y_d, void* stream) {
  if (!prob || !inv_d || !r_d || !y_d) return fail(MG_ERR_VALUE, "NULL argument");
  return guard([&] { launch_block_apply(prob->p, inv_d, r_d, y_d, S(stream)); });
}

int mg_pcg(mg_problem* prob, const double* hess_d, const double* x_eval_d, int use_psd, double psd_floor,
           const double* inv_d, const double* b_d, double tol, int max_iters, double* out_d, int* iters, int* status,
           void* stream) {
  if (!prob || !b_d || !out_d || !iters || !status) return fail(MG_ERR_VALUE, "NULL argument");
  if (!hess_d && !x_eval_d) return fail(MG_ERR_VALUE, "mg_pcg needs the assembled Hessian or the HVP point");
  if (max_iters < 1) return fail(MG_ERR_VALUE, "max_iters must be at least 1");
  if (use_psd && !(psd_floor > 0)) return fail(MG_ERR_VALUE, "floor must be positive");
  return guard([&] {
    auto hvp = [&](const double* v, double* y) {
      const int rc = mg_hvp(prob, x_eval_d, v, use_psd, psd_floor, y, stream);
      if (rc != MG_OK) throw Error(rc, g_err);
    };
    pcg_solve(prob->p, hess_d, hvp, inv_d, b_d, tol, max_iters, out_d, iters, status, S(stream));
  });
}

int mg_problem_destroy(mg_problem* prob) {
  if (prob) {
    for (auto& t : prob->p.terms)
      if (t.jit) jit_unload(t);
    jit_patch_unload(prob->p);
    jit_rows_unload(prob->p);
    for (auto& pr : prob->p.ev_pairs) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    for (auto e : prob->p.ev_pool) cudaEventDestroy(e);
  }
  delete prob;
  return MG_OK;
}

int mg_problem_exact_runs(const mg_problem* prob, int64_t* runs) {
  if (!prob || !runs) return fail(MG_ERR_VALUE, "NULL argument");
  return guard([&] {
    int h = 0;
    if (prob->p.exact_runs.p) MG_CUDA(cudaMemcpy(&h, prob->p.exact_runs.p, sizeof(int), cudaMemcpyDeviceToHost));
    *runs = h;
  });
}

int mg_problem_set_timing(mg_problem* prob, int enable) {
  if (!prob) return fail(MG_ERR_VALUE, "problem is NULL");
  prob->p.timing = enable != 0;
  return MG_OK;
}

int mg_problem_kernel_time(mg_problem* prob, double* total_ms, int* count) {
  if (!prob || !total_ms || !count) return fail(MG_ERR_VALUE, "NULL argument");
  return guard([&] {
    Problem& p = prob->p;
    double t = 0.0;
    for (auto& pr : p.ev_pairs) {
      MG_CUDA(cudaEventSynchronize(pr.second));
      float ms = 0.f;
      MG_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
      t += ms;
      p.ev_pool.push_back(pr.first);
      p.ev_pool.push_back(pr.second);
    }
    *total_ms = t;
    *count = (int)p.ev_pairs.size();
    p.ev_pairs.clear();
  });
}

int mg_last_launch_count(const mg_problem* prob, int* launches) {
  if (!prob || !launches) return fail(MG_ERR_VALUE, "NULL argument");
  *launches = prob->p.last_launches;
  return MG_OK;
}

int mg_problem_patch_stats(const mg_problem* prob, int64_t* stats4) {
  if (!prob || !stats4) return fail(MG_ERR_VALUE, "NULL argument");
  const Problem& p = prob->p;
  stats4[0] = p.mesh->patches.num;
  stats4[1] = p.mesh->V;
  stats4[2] = p.mesh->patches.ribbon_total;
  stats4[3] = p.recomputed_elements;
  return MG_OK;
}

}  // extern "C"
