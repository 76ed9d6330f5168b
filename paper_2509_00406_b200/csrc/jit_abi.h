// Launch ABI between the library and traced (JIT) term kernels
// (jit_kernel.cuh, compiled at runtime by paper_2509_00406_b200/jit.py and
// loaded with mg_problem_add_jit_term). Both sides include this header.
#pragma once
#include <cstdint>

namespace mg {

constexpr int JIT_TPB = 128;
constexpr int JIT_MAX_ATTRS = 64;
enum JitMode { JIT_ENERGY = 0, JIT_GRAD = 1, JIT_HESS = 2, JIT_HVP = 3 };

struct JitArgs {
  const double* x;
  const double* w;
  const uint8_t* fixed;
  const uint8_t* owned;    // shard: energy counts where the element's first vertex is owned
  const int32_t* sel;      // (M, P) element vertices, or null for vertex terms
  const int32_t* bids;     // (M, P, P) Hessian block ids, -1 = pinned pair
  double* grad;
  double* hess;
  double* y;
  double* partials;
  double floor;
  int64_t M;
  const double* attrs[JIT_MAX_ATTRS];  // per-element attribute streams (device)
  double* sv;  // deterministic gather mode: (M,P,N) slot vectors, (M,P,P,N,N) blocks
  double* sh;
};

}  // namespace mg
