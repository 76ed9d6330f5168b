// Deterministic patch-owner assembly: one CTA per vertex patch.
//
// A CTA owns R consecutive rows (Morton order) of the gradient / HVP / block
// Hessian. It
//   1. stages x (and the HVP direction) of its owned + ribbon vertices in
//      shared memory,
//   2. evaluates the V terms of its owned vertices (one thread per row),
//   3. evaluates every EV / FV element incident to an owned row (ribbon
//      elements are evaluated by each owning patch), holding the element's
//      dual-number result in registers, and adds the owned-row parts into
//      shared-memory row accumulators in conflict-free color phases
//      (elements are pre-sorted by color: a fixed, race-free summation order),
//   4. writes each owned row once, coalesced: no memset, no atomics, bitwise
//      reproducible.
// The energy is summed per patch over the elements whose first vertex is
// owned, then reduced in fixed order.
//
// Term types dispatch at runtime inside the kernel (warp-uniform switch);
// families bound which types are compiled in, to keep register allocation of
// light problems (cloth) independent of heavy terms (sphere).
#include "mg_internal.cuh"
#include "psd.cuh"
#include "elem_eval.cuh"

#include "patch_kernel.cuh"

namespace mg {

namespace {

using namespace patch;

// type masks of the compiled families
constexpr unsigned bit(int t) { return 1u << t; }
constexpr unsigned FAM_LIGHT = bit(MG_TERM_INERTIA) | bit(MG_TERM_SPRING) | bit(MG_TERM_GRAVITY) | bit(MG_TERM_EDGE_LENGTH);
constexpr unsigned FAM_UV = FAM_LIGHT | bit(MG_TERM_SYM_DIRICHLET);
constexpr unsigned FAM_ALL = FAM_UV | bit(MG_TERM_SPHERE);

// builtin terms: runtime dispatch on the term type (warp-uniform switch)
template <unsigned FAM>
struct BuiltinPolicy {
  template <int N, int MODE, bool PSD>
  MG_DI static void vterms(const PatchArgs& a, const Smem& s, int oc, double& eacc) {
    for (int ti = 0; ti < a.nterms; ++ti) {
      const TermDev& t = a.terms[ti];
      if (t.op != MG_OP_V) continue;
      switch (t.type) {
        case MG_TERM_INERTIA:
          if constexpr ((FAM & bit(MG_TERM_INERTIA)) != 0) run_vterm_g<N, MODE, PSD>(a, BuiltinEval<MG_TERM_INERTIA, N>{t}, s, oc, eacc);
          break;
        case MG_TERM_GRAVITY:
          if constexpr ((FAM & bit(MG_TERM_GRAVITY)) != 0) run_vterm_g<N, MODE, PSD>(a, BuiltinEval<MG_TERM_GRAVITY, N>{t}, s, oc, eacc);
          break;
        default: break;
      }
    }
  }
  template <int N, int MODE, bool PSD>
  MG_DI static void eterms(const PatchArgs& a, int p, const Smem& s, int oc, double& eacc) {
    for (int ti = 0; ti < a.nterms; ++ti) {
      const TermDev& t = a.terms[ti];
      switch (t.type) {
        case MG_TERM_SPRING:
          if constexpr ((FAM & bit(MG_TERM_SPRING)) != 0) run_eterm_g<2, N, MODE, PSD>(a, BuiltinEval<MG_TERM_SPRING, N>{t}, a.ev, p, s, oc, eacc);
          break;
        case MG_TERM_EDGE_LENGTH:
          if constexpr ((FAM & bit(MG_TERM_EDGE_LENGTH)) != 0) run_eterm_g<2, N, MODE, PSD>(a, BuiltinEval<MG_TERM_EDGE_LENGTH, N>{t}, a.ev, p, s, oc, eacc);
          break;
        case MG_TERM_SYM_DIRICHLET:
          if constexpr ((FAM & bit(MG_TERM_SYM_DIRICHLET)) != 0 && N == 2) run_eterm_g<3, N, MODE, PSD>(a, BuiltinEval<MG_TERM_SYM_DIRICHLET, N>{t}, a.fv, p, s, oc, eacc);
          break;
        case MG_TERM_SPHERE:
          if constexpr ((FAM & bit(MG_TERM_SPHERE)) != 0 && N == 2) run_eterm_g<3, N, MODE, PSD>(a, BuiltinEval<MG_TERM_SPHERE, N>{t}, a.fv, p, s, oc, eacc);
          break;
        default: break;
      }
    }
  }
};

template <int N, unsigned FAM, int MODE, bool PSD>
__global__ void __launch_bounds__(PT) k_patch(const __grid_constant__ PatchArgs a, int nvp_max, int blocks_max) {
  patch_body<N, MODE, PSD, BuiltinPolicy<FAM>>(a, nvp_max, blocks_max);
}


template <int N, unsigned FAM, int MODE, bool PSD>
void launch_fam(const PatchArgs& a, int64_t np, int nvp_max, int blocks_max, cudaStream_t st) {
  auto kern = k_patch<N, FAM, MODE, PSD>;
  const size_t sm = smem_bytes(N, MODE, a.R, nvp_max, blocks_max);
  if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "patch does not fit in shared memory");
  MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int64_t grid = np;
  if (a.redo) {  // exact re-run: a small persistent grid that exits unless the flag is raised
    int dev = 0, sms = 148;
    MG_CUDA(cudaGetDevice(&dev));
    MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = np < (int64_t)sms * 4 ? np : (int64_t)sms * 4;
  }
  kern<<<(unsigned)grid, PT, sm, st>>>(a, nvp_max, blocks_max);
  MG_LAUNCH_CHECK();
}

template <int N, unsigned FAM>
void launch_mode(const PatchArgs& a, int64_t np, int nvp, int nb, Mode mode, bool psd, cudaStream_t st) {
  switch (mode) {
    case MODE_GRAD: launch_fam<N, FAM, MODE_GRAD, false>(a, np, nvp, nb, st); break;
    case MODE_HESS:
      if (psd) launch_fam<N, FAM, MODE_HESS, true>(a, np, nvp, nb, st);
      else launch_fam<N, FAM, MODE_HESS, false>(a, np, nvp, nb, st);
      break;
    case MODE_HVP:
      if (psd) launch_fam<N, FAM, MODE_HVP, true>(a, np, nvp, nb, st);
      else launch_fam<N, FAM, MODE_HVP, false>(a, np, nvp, nb, st);
      break;
    default: throw Error(MG_ERR_UNSUPPORTED, "patch kernels assemble grad / Hessian / HVP only");
  }
}

}  // namespace

bool patch_supported(const Problem& p) {
  if (p.terms.empty() || p.terms.size() > MAXT) return false;
  bool any_jit = false;
  for (auto& t : p.terms) {
    if (t.dev.op == MG_OP_VV) return false;
    any_jit |= t.jit;
  }
  if (any_jit) {  // traced terms: through the problem's generated patch module only, all terms traced
    if (!p.patch_module) return false;
    for (auto& t : p.terms)
      if (!t.jit) return false;
    return p.mesh->patches.num > 0;
  }
  if (p.n != 2 && p.n != 3) return false;
  return p.mesh->patches.num > 0;
}

int64_t launch_patch(const Problem& p, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  const Mesh& m = *p.mesh;
  if (p.ev_fast) return launch_patch_ev(p, mode, c, partial_offset);
  int64_t n_fast = 0;
  // face row kernels: Dirichlet in every mode; sphere for gradient / HVP
  bool fast = p.fv_fast && (p.terms[0].dev.type != MG_TERM_SPHERE || mode == MODE_GRAD || mode == MODE_HVP);
  if (fast) n_fast = launch_patch_fv(p, mode, c, partial_offset);
  // traced terms with radial edge callbacks: the generated row kernel
  if (p.ev_jit && p.patch_module) {
    n_fast = launch_rows_jit(p, mode, c, partial_offset);
    fast = true;
  }
  // the exact re-run writes one partial per patch; without it the partials
  // past the fast kernel's must read as zero
  if (fast && mode != MODE_HVP && m.patches.num > n_fast)
    MG_CUDA(cudaMemsetAsync(c.partials + partial_offset + n_fast, 0, sizeof(double) * (m.patches.num - n_fast),
                            c.stream));
  PatchArgs a;
  a.R = m.patches.R;
  a.nterms = (int)p.terms.size();
  a.V = m.Vr;
  a.np = m.patches.num;
  a.redo = fast ? p.redo.p : nullptr;  // after a face row kernel: exact re-run only on its flag
  a.exact_runs = p.exact_runs.p;
  a.np_total = n_fast;
  a.vtx_off = p.vtx_off.p;
  a.vtx = p.vtx.p;
  a.hloc = p.hloc.p;
  a.diag_pos = p.diag_pos.p;
  a.row_offsets = p.row_offsets.p;
  a.fixed = p.any_fixed ? p.fixed.p : nullptr;
  a.x = c.x;
  a.w = c.w;
  a.grad = c.grad;
  a.hess = c.hess;
  a.y = c.y;
  a.partials = c.partials + partial_offset;
  a.floor = c.floor;
  const OpLayout& ev = p.lay[0];
  const OpLayout& fv = p.lay[1];
  a.ev = OpView{ev.off.p, ev.elem.p, ev.local.p, ev.pos.p, ev.color.p};
  a.fv = OpView{fv.off.p, fv.elem.p, fv.local.p, fv.pos.p, fv.color.p};
  a.jattr = nullptr;
  const int64_t np = m.patches.num;
  const int nvp = p.max_patch_vertices, nb = p.max_patch_blocks;
  if (p.patch_module) {  // traced terms: the problem's generated patch kernels (jit_patch.cuh)
    if (p.jattr_dirty) {
      std::vector<const double*> h((size_t)a.nterms * JATTR, nullptr);
      for (int i = 0; i < a.nterms; ++i)
        for (size_t k = 0; k < p.terms[i].jit_attrs.size() && k < (size_t)JATTR; ++k)
          h[(size_t)i * JATTR + k] = p.terms[i].jit_attrs[k];
      p.jattr.alloc(h.size());
      MG_CUDA(cudaMemcpyAsync(p.jattr.p, h.data(), h.size() * sizeof(const double*), cudaMemcpyHostToDevice,
                              c.stream));
      MG_CUDA(cudaStreamSynchronize(c.stream));
      p.jattr_dirty = false;
    }
    a.jattr = p.jattr.p;
    for (int i = 0; i < a.nterms; ++i) a.terms[i] = p.terms[i].dev;
    const size_t sm = smem_bytes(p.n, mode, a.R, nvp, nb);
    if (sm > 227 * 1024) throw Error(MG_ERR_UNSUPPORTED, "patch does not fit in shared memory");
    if (!fast) timing_begin(p, c.stream);
    int64_t grid = np;
    if (a.redo) {  // exact re-run: a small persistent grid that exits unless the flag is raised
      int dev = 0, sms = 148;
      MG_CUDA(cudaGetDevice(&dev));
      MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      grid = np < (int64_t)sms * 4 ? np : (int64_t)sms * 4;
    }
    jit_patch_launch(p, mode, c.psd, &a, np, nvp, nb, sm, c.stream, grid);
    if (!fast) timing_end(p, c.stream);
    if (mode == MODE_HVP) return 0;
    return np > n_fast ? np : n_fast;
  }
  unsigned used = 0;
  for (int i = 0; i < a.nterms; ++i) {
    a.terms[i] = p.terms[i].dev;
    used |= 1u << p.terms[i].dev.type;
  }
  if (!fast) timing_begin(p, c.stream);
  if (p.n == 3) {
    if (used & ~FAM_LIGHT) throw Error(MG_ERR_UNSUPPORTED, "term not available for var_dim 3");
    launch_mode<3, FAM_LIGHT>(a, np, nvp, nb, mode, c.psd, c.stream);
  } else {
    if (used & bit(MG_TERM_SPHERE)) launch_mode<2, FAM_ALL>(a, np, nvp, nb, mode, c.psd, c.stream);
    else if (used & bit(MG_TERM_SYM_DIRICHLET)) launch_mode<2, FAM_UV>(a, np, nvp, nb, mode, c.psd, c.stream);
    else launch_mode<2, FAM_LIGHT>(a, np, nvp, nb, mode, c.psd, c.stream);
  }
  if (!fast) timing_end(p, c.stream);
  if (mode == MODE_HVP) return 0;
  return np > n_fast ? np : n_fast;
}

}  // namespace mg
