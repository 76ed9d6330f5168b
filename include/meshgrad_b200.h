/*
 * meshgrad_b200 — C ABI of the B200-native per-element forward-mode AD engine.
 *
 * Drop-in boundary for the reference's `Problem` hot path
 * (/root/reference/pkg/src/meshgrad/problem.py). The reference is pure
 * Python/numpy, so its "FFI" is the Python method surface of `Problem`; every
 * entry point below replaces one of those methods (cited per function) and is
 * bound from Python with ctypes (paper_2509_00406_b200/_lib.py; the binding a
 * maintainer would add to the reference is shown in INTEGRATION.md).
 *
 * Conventions
 *  - Plain pointers and sizes only. Arrays named *_d are DEVICE pointers owned
 *    by the caller (torch tensors on the host side); the library owns the mesh
 *    topology, patches, the Hessian pattern and its scratch.
 *  - `stream` is a cudaStream_t passed as void*. All calls are stream-ordered
 *    and asynchronous unless stated otherwise.
 *  - Every function returns 0 on success or a nonzero MG_ERR_* code; the
 *    message (mirroring the reference's exception text) is available from
 *    mg_last_error() (thread-local).
 *  - Numerical infeasibility is NOT an error: NaN/Inf propagate into outputs
 *    (reference problem.py:16-21, test_problem.py:157-161).
 *  - fp64 everywhere (reference arithmetic is float64, active.py:333).
 */
#ifndef MESHGRAD_B200_H
#define MESHGRAD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MG_API __attribute__((visibility("default")))
#else
#define MG_API
#endif

#define MG_ABI_VERSION 1

enum mg_status {
  MG_OK = 0,
  MG_ERR_VALUE = 1,   /* bad argument: reference raises ValueError        */
  MG_ERR_MESH = 2,    /* malformed mesh: reference raises MeshError        */
  MG_ERR_STATE = 3,   /* call out of order (e.g. pattern before terms)     */
  MG_ERR_CUDA = 4,    /* CUDA runtime failure                              */
  MG_ERR_UNSUPPORTED = 5
};

/* Neighbourhood ops that resolve to vertex variables (mesh.py:50-66, problem.py:44). */
enum mg_op { MG_OP_FV = 0, MG_OP_EV = 1, MG_OP_VV = 2, MG_OP_V = 3 };

/* Builtin per-element energies (the reference apps' callbacks).
 * params / attrs per type (attrs are device fp64 arrays, caller-owned):
 *  INERTIA       V,  0.5*m_i*|x_i - t_i|^2         (apps/cloth.py:102-104)
 *                params: -             attrs: [masses (V), target (V*n)]
 *  SPRING        EV, c*l2*(|x_i-x_j|^2/l2 - 1)^2   (apps/cloth.py:106-110)
 *                params: [c]           attrs: [rest_len2 (E)]
 *  GRAVITY       V,  (-h2)*(m_i*(x_i . g))          (apps/cloth.py:112-113)
 *                params: [h2, g_0..g_{n-1}]        attrs: [masses (V)]
 *  EDGE_LENGTH   EV, |x_i - x_j|^2                  (apps/smooth.py:22-31)
 *  SYM_DIRICHLET FV n=2, area*(|J|^2 + |J|^2/det^2) (apps/param.py:170-177)
 *                params: -             attrs: [rest_inv (F*4, row-major 2x2), areas (F)]
 *  SPHERE        FV n=2, -log det[p] + sum |p_a-p_b|^2 through the
 *                retraction p = normalize(s + x0 b1 + x1 b2) (apps/sphere.py:71-99)
 *                params: [include_barrier, include_stretch]
 *                attrs: [base (V*3), b1 (V*3), b2 (V*3)]
 */
enum mg_term_type {
  MG_TERM_INERTIA = 1,
  MG_TERM_SPRING = 2,
  MG_TERM_GRAVITY = 3,
  MG_TERM_EDGE_LENGTH = 4,
  MG_TERM_SYM_DIRICHLET = 5,
  MG_TERM_SPHERE = 6,
  MG_TERM_JIT = 100  /* traced user callback (mg_problem_add_jit_term) */
};

typedef struct mg_mesh mg_mesh;
typedef struct mg_problem mg_problem;

/* Thread-local message for the last nonzero status. */
MG_API const char* mg_last_error(void);
MG_API int mg_abi_version(void);

/* Mesh topology on the device.
 * Replaces Mesh.__init__ validation + _derive_edges (mesh.py:139-202) and the
 * patching used by the hot path (partition_patches/_inherit_patch, mesh.py:225-279),
 * re-designed as Morton-ordered vertex patches with ribbons built on device.
 *   faces_d      (F,3) int64 device, or NULL when F == 0
 *   edges_d      (E,2) int64 device explicit edges for face-free meshes, else NULL
 *   positions_d  (V,3) fp64 device (patch locality only; may be NULL)
 *   patch_vertices  owned vertices per patch (0 = default 128)
 * Edges come out canonical (i<j) and lexicographically sorted: bit-identical
 * to the reference's mesh.edges. Synchronizes `stream` before returning. */
MG_API int mg_mesh_create(const int64_t* faces_d, int64_t num_faces, const int64_t* edges_d,
                   int64_t num_edges, int64_t num_vertices, const double* positions_d,
                   int patch_vertices, void* stream, mg_mesh** out);
MG_API int mg_mesh_counts(const mg_mesh* mesh, int64_t* num_vertices, int64_t* num_edges,
                   int64_t* num_faces, int64_t* num_patches);
/* Copy the derived (E,2) edge list into a caller device buffer (int64). */
MG_API int mg_mesh_copy_edges(const mg_mesh* mesh, int64_t* edges_d, void* stream);
/* Patch id of every vertex (int32, device) — diagnostics / multi-GPU partitioning. */
MG_API int mg_mesh_copy_vertex_patches(const mg_mesh* mesh, int32_t* patch_d, void* stream);
/* Multi-GPU shard (no reference counterpart: the reference is single-process).
 * Restrict the rows this mesh assembles to the vertices flagged in owned_d
 * ((V,) uint8 device, 1 = owned; NULL = all). The other vertices are ribbon
 * (halo) vertices: their x is read, their gradient / Hessian / HVP rows are
 * left to the device that owns them (pattern rows empty, outputs untouched),
 * and an element's energy counts only where its first vertex is owned, so the
 * per-shard energies sum to the global energy. Call before creating problems
 * on the mesh. Synchronizes `stream`. */
/* Row processing order of the assembly kernels (never changes results beyond
 * summation order; the outputs stay in the caller's numbering). AUTO (the
 * default at mg_mesh_create) keeps the caller's vertex numbering when it is
 * translation-regular (>= half the edges (i,j) have (i+1,j+1) as an edge:
 * structured grids, where consecutive rows' neighbour gathers coalesce) and
 * uses a Morton order of the positions otherwise. Setting it rebuilds the
 * patches; call before creating problems on the mesh. No reference
 * counterpart (the reference's patch order, mesh.py:252-279, only affects
 * rounding too). */
enum mg_row_order { MG_ROW_AUTO = 0, MG_ROW_MORTON = 1, MG_ROW_IDENTITY = 2 };
MG_API int mg_mesh_set_row_order(mg_mesh* mesh, int order, void* stream);
/* resolved order (MG_ROW_MORTON / MG_ROW_IDENTITY) and the regularity score */
MG_API int mg_mesh_row_order(const mg_mesh* mesh, int* order, double* regularity);

MG_API int mg_mesh_set_owned(mg_mesh* mesh, const uint8_t* owned_d, void* stream);
MG_API int mg_mesh_destroy(mg_mesh* mesh);

/* Problem state. Replaces Problem.__init__ (problem.py:259-297).
 *   fixed_mask_d  (V,) uint8 device, 1 = pinned (may be NULL)
 *   deterministic 1: patch-owner assembly, bitwise reproducible;
 *                 0: element-parallel atomics ("atomic" accumulation, problem.py:16-21) */
MG_API int mg_problem_create(mg_mesh* mesh, int var_dim, int with_hessian, const uint8_t* fixed_mask_d,
                      int deterministic, mg_problem** out);
/* Replaces Problem.add_term (problem.py:301-310) for builtin terms.
 * Validates kind/op pairing via `op` and the term's natural op. */
MG_API int mg_problem_add_term(mg_problem* prob, int term_type, int op, const double* params,
                        int num_params, const double* const* attrs_d, int num_attrs,
                        int* term_id);
/* Register a traced user callback (the reference's general callback protocol,
 * problem.py:8-14 / 301-310): `image` is a cubin built by
 * paper_2509_00406_b200/jit.py from csrc/jit_kernel.cuh for this var_dim,
 * exporting mg_jit_{energy,grad,hess,hess_psd,hvp,hvp_psd}; attrs_d are its
 * per-element attribute streams (device fp64, caller-owned, at most 64). Problems with a
 * traced term assemble element-parallel: into per-element scratch plus a
 * fixed-order gather when deterministic, with fp64 atomics otherwise. */
MG_API int mg_problem_add_jit_term(mg_problem* prob, int op, int var_dim, const void* image,
                                   const double* const* attrs_d, int num_attrs, int* term_id);
/* A traced VV (vertex-neighbourhood) term over an explicit selection: sel_d is
 * (M, P) int32 on the device (caller-owned), row = center vertex then its
 * one-ring ascending (ref problem.py:340-353); the reference groups VV
 * elements by valence, so register one term per valence group (P = 1 + d,
 * d <= 32). The module is traced for that P. */
MG_API int mg_problem_add_jit_term_sel(mg_problem* prob, int op, int var_dim, int P, const int32_t* sel_d, int64_t M,
                                       const void* image, const double* const* attrs_d, int num_attrs,
                                       int* term_id);
/* Traced terms on the patch-owner path: `image` is a cubin generated by
 * paper_2509_00406_b200/jit.py for THIS problem's traced terms (in
 * registration order; csrc/jit_patch.cuh) exporting mg_patch_{grad, hess,
 * hess_psd, hvp, hvp_psd}. With it, eval / hvp assemble the traced terms
 * with the same deterministic patch kernel body as the builtin terms instead
 * of element-parallel scratch + gather. NULL drops it; adding a term drops
 * it. Every term must be traced (V / EV / FV). Same numbers as the element
 * path up to summation order (reference problem.py:504-617). */
MG_API int mg_problem_set_patch_module(mg_problem* prob, const void* image);
/* Traced terms on the edge row kernel: `image` is a cubin generated by
 * paper_2509_00406_b200/jit.py (csrc/jit_rows.cuh) for THIS problem's traced
 * terms when every EV callback depends on x only through |x_i - x_j|^2 (the
 * tracer proves it on the recorded operations) and the others are V terms;
 * it exports mg_rows_{grad, hess, hess_psd, hvp, hvp_psd} and needs the
 * problem's patch module as its exact re-run (non-finite lanes). Replaces
 * the per-element evaluation of Problem.eval_terms / hvp (reference
 * problem.py:504-549, 578-617) by one thread per row with phi(r) on a
 * one-variable second-order dual; results agree with the full-dual path to
 * rounding. NULL drops it; adding a term drops it. */
MG_API int mg_problem_set_row_module(mg_problem* prob, const void* image);
/* Storage precision of x, the HVP direction, the gradient, the Hessian values,
 * the HVP result and the builtin terms' attribute arrays: 64 (default, the
 * reference's float64) or 32 (half the bytes; every kernel computes in fp64
 * and rounds on store). fp32 storage runs on the edge row kernels only —
 * deterministic problems whose terms are builtin vertex and radial edge terms
 * (cloth, smoothing) — for mg_eval, mg_hvp and mg_energy (energy in fp64);
 * other calls and problems return MG_ERR_UNSUPPORTED. Non-finite values keep
 * the closed forms' propagation (no exact re-run). Set before the first call. */
MG_API int mg_problem_set_storage(mg_problem* prob, int bits);
MG_API int mg_problem_set_jit_attr(mg_problem* prob, int term_id, int slot, const double* attr_d);
/* Rebind one attribute pointer of a registered term (closure arrays that the
 * reference rewrites in place between calls, apps/cloth.py:128, sphere.py:121-127). */
MG_API int mg_problem_set_attr(mg_problem* prob, int term_id, int slot, const double* attr_d);
/* Replaces Problem.precompute_sparsity (problem.py:383-416): device-built
 * block-CSR pattern; returns nnzb. Synchronizes `stream`. */
MG_API int mg_precompute_sparsity(mg_problem* prob, int64_t* nnzb, void* stream);
/* row_offsets (V+1) / col_indices (nnzb), int64, bit-exact with the reference. */
MG_API int mg_copy_pattern(const mg_problem* prob, int64_t* row_offsets_d, int64_t* col_indices_d,
                    void* stream);
/* Replaces Problem.eval_terms (problem.py:504-549).
 *   use_psd/psd_floor: per-element eigenvalue clamp (floor <= 0 -> MG_ERR_VALUE,
 *   active.py:497-498; psd without Hessian mode -> MG_ERR_VALUE, problem.py:515-516)
 *   energy_d: 1 fp64 (device)   grad_d: n*V fp64 (device)
 *   hess_d:   nnzb*n*n fp64 (device) or NULL when with_hessian == 0.
 * Outputs are fully overwritten (zeroing is the callee's job, problem.py:519-521). */
MG_API int mg_eval(mg_problem* prob, const double* x_d, int use_psd, double psd_floor, double* energy_d,
            double* grad_d, double* hess_d, void* stream);
/* Replaces Problem.eval_energy_only (problem.py:551-576). */
MG_API int mg_energy(mg_problem* prob, const double* x_d, double* energy_d, void* stream);
/* Replaces Problem.hvp (problem.py:578-617): y = sum_j S_j^T H_j S_j v, matrix
 * free; pinned rows of y are 0 and pinned components of v are ignored. */
MG_API int mg_hvp(mg_problem* prob, const double* x_d, const double* v_d, int use_psd, double psd_floor,
           double* y_d, void* stream);
/* Block-CSR SpMV y = H v on an assembled Hessian (BlockSparseMatrix.matvec,
 * problem.py:100-106). */
MG_API int mg_bsr_matvec(const mg_problem* prob, const double* hess_d, const double* v_d, double* y_d,
                  void* stream);
/* Block-Jacobi preconditioner of the assembled Hessian: inv_d (V, n, n) =
 * inverse of each row's diagonal block, identity where there is none or it is
 * singular (BlockSparseMatrix.diagonal_block_inverses, problem.py:118-131). */
MG_API int mg_bsr_block_jacobi(const mg_problem* prob, const double* hess_d, double* inv_d, void* stream);
/* y_v = inv_v r_v per vertex (the preconditioner apply, solvers.py:178-186). */
MG_API int mg_block_apply(const mg_problem* prob, const double* inv_d, const double* r_d, double* y_d, void* stream);
/* Truncated CG on the device, block-Jacobi preconditioned when inv_d (the
 * mg_bsr_block_jacobi inverses) is given — the inner solver of the reference's
 * cg_linear_solve (solvers.py:142-175) as used by newton_solve (:244-263,
 * hess_d = the assembled Hessian values) and newton_cg_solve (:266-287,
 * hess_d NULL: the operator is mg_hvp at x_eval_d, clamped when use_psd).
 * Solves A out = b from out = 0; stops at |r| <= tol |b|, at non-positive
 * curvature (returning b itself when no step was taken, like the reference)
 * or after max_iters. Scalars and decisions stay on the device; the host
 * waits once per 8 iterations. *iters = iterations run, *status = 1
 * converged, 2 non-positive curvature, 3 max iterations. */
MG_API int mg_pcg(mg_problem* prob, const double* hess_d, const double* x_eval_d, int use_psd, double psd_floor,
                  const double* inv_d, const double* b_d, double tol, int max_iters, double* out_d, int* iters,
                  int* status, void* stream);
MG_API int mg_problem_destroy(mg_problem* prob);

/* Introspection for benchmarks/tests: number of kernel launches issued by the
 * most recent mg_eval/mg_energy/mg_hvp call, and the problem's patch stats
 * (patches, owned rows, ribbon vertices, recomputed ribbon elements). */
MG_API int mg_last_launch_count(const mg_problem* prob, int* launches);
/* Device timing of the main assembly / HVP kernel (benchmarks): when enabled,
 * every mg_eval / mg_hvp records CUDA events around that kernel on the call's
 * stream; mg_problem_kernel_time synchronizes, returns the summed duration
 * (ms) and the number of launches timed since the previous query, and resets. */
MG_API int mg_problem_set_timing(mg_problem* prob, int enable);
/* Number of calls so far whose exact re-run executed (a fast row kernel met a
 * non-finite lane, or pinned corners under a PSD clamp). Synchronizes. */
MG_API int mg_problem_exact_runs(const mg_problem* prob, int64_t* runs);
MG_API int mg_problem_kernel_time(mg_problem* prob, double* total_ms, int* count);
MG_API int mg_problem_patch_stats(const mg_problem* prob, int64_t* stats4);

#ifdef __cplusplus
}
#endif
#endif /* MESHGRAD_B200_H */
