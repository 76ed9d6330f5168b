// Patch-owner assembly of traced (JIT) energy terms.
//
// paper_2509_00406_b200/jit.py emits one functor per traced callback (the
// recorded SSA over the engine's duals, jit_kernel.cuh) and a policy that
// runs them through the same patch kernel body as the builtin terms
// (patch_kernel.cuh): the patch's vertices staged in shared memory, every
// element incident to an owned row evaluated with its duals in registers,
// colour-phased shared-memory row accumulators, each owned row and Hessian
// row written once — deterministic, no scratch, no atomics. The module is
// compiled per problem (its traced terms, in registration order) and handed
// to the library with mg_problem_set_patch_module.
#pragma once
#include "jit_kernel.cuh"
#include "patch_kernel.cuh"

namespace mg {
namespace patch {

// a traced functor as a patch evaluator: A = the term's attribute streams
template <class F, int N>
struct JitEval {
  const double* const* A;
  template <class S>
  MG_DI auto operator()(int64_t e, const int*, const Vec<S, N>* X) const {
    return F{}.template operator()<N>(A, e, X);
  }
};

}  // namespace patch
}  // namespace mg

#define MG_PATCH_JIT_KERNEL(POL, N, NAME, MODE, PSD)                                                   \
  extern "C" __global__ void __launch_bounds__(mg::patch::PT)                                          \
      NAME(const __grid_constant__ mg::patch::PatchArgs a, int nvp_max, int blocks_max) {              \
    mg::patch::patch_body<N, MODE, PSD, POL>(a, nvp_max, blocks_max);                                  \
  }

#define MG_PATCH_JIT_INSTANTIATE(POL, N)                                  \
  MG_PATCH_JIT_KERNEL(POL, N, mg_patch_grad, mg::MODE_GRAD, false)        \
  MG_PATCH_JIT_KERNEL(POL, N, mg_patch_hess, mg::MODE_HESS, false)        \
  MG_PATCH_JIT_KERNEL(POL, N, mg_patch_hess_psd, mg::MODE_HESS, true)     \
  MG_PATCH_JIT_KERNEL(POL, N, mg_patch_hvp, mg::MODE_HVP, false)          \
  MG_PATCH_JIT_KERNEL(POL, N, mg_patch_hvp_psd, mg::MODE_HVP, true)
