// Traced (JIT) terms: module loading and launches through the CUDA driver API.
//
// libcuda is opened lazily with dlopen so the library still loads (and its
// symbols can be inspected) on machines without a GPU driver.
#include <dlfcn.h>

#include <cstring>

#include "jit_abi.h"
#include "mg_internal.cuh"

namespace mg {

namespace {

typedef int (*PFN_load)(void**, const void*);
typedef int (*PFN_getfn)(void**, void*, const char*);
typedef int (*PFN_launch)(void*, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, void*,
                          void**, void**);
typedef int (*PFN_unload)(void*);
typedef int (*PFN_errstr)(int, const char**);

struct Driver {
  PFN_load load = nullptr;
  PFN_getfn getfn = nullptr;
  PFN_launch launch = nullptr;
  PFN_unload unload = nullptr;
  PFN_errstr errstr = nullptr;
};

Driver& driver() {
  static Driver d;
  static bool init = false;
  if (!init) {
    init = true;
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      d.load = (PFN_load)dlsym(h, "cuModuleLoadData");
      d.getfn = (PFN_getfn)dlsym(h, "cuModuleGetFunction");
      d.launch = (PFN_launch)dlsym(h, "cuLaunchKernel");
      d.unload = (PFN_unload)dlsym(h, "cuModuleUnload");
      d.errstr = (PFN_errstr)dlsym(h, "cuGetErrorString");
    }
  }
  if (!d.load || !d.getfn || !d.launch) throw Error(MG_ERR_CUDA, "CUDA driver API (libcuda) unavailable");
  return d;
}

void drv_check(int rc, const char* what) {
  if (rc == 0) return;
  const char* s = nullptr;
  if (driver().errstr) driver().errstr(rc, &s);
  throw Error(MG_ERR_CUDA, std::string(what) + ": " + (s ? s : "driver error " + std::to_string(rc)));
}

const char* kNames[6] = {"mg_jit_energy", "mg_jit_grad", "mg_jit_hess", "mg_jit_hess_psd", "mg_jit_hvp",
                         "mg_jit_hvp_psd"};

}  // namespace

void jit_load(Term& t, const void* image) {
  MG_CUDA(cudaFree(nullptr));  // make the runtime's primary context current for the driver calls
  Driver& d = driver();
  drv_check(d.load(&t.jit_module, image), "cuModuleLoadData");
  for (int i = 0; i < 6; ++i) drv_check(d.getfn(&t.jit_fn[i], t.jit_module, kNames[i]), kNames[i]);
}

void jit_unload(Term& t) {
  if (t.jit_module && driver().unload) driver().unload(t.jit_module);
  t.jit_module = nullptr;
}

void jit_launch(const Problem& p, const Term& t, Mode mode, const LaunchCtx& c, int64_t partial_offset) {
  JitArgs a;
  std::memset(&a, 0, sizeof(a));
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
  for (size_t i = 0; i < t.jit_attrs.size() && i < (size_t)JIT_MAX_ATTRS; ++i) a.attrs[i] = t.jit_attrs[i];
  a.sv = c.scratch ? p.gsv.p + t.gv_base : nullptr;
  a.sh = c.scratch && mode == MODE_HESS ? p.gsh.p + t.gh_base : nullptr;
  int k;
  switch (mode) {
    case MODE_ENERGY: k = 0; break;
    case MODE_GRAD: k = 1; break;
    case MODE_HESS: k = c.psd ? 3 : 2; break;
    default: k = c.psd ? 5 : 4; break;
  }
  void* params[1] = {&a};
  const unsigned grid = (unsigned)((t.M + JIT_TPB - 1) / JIT_TPB);
  if (grid) drv_check(driver().launch(t.jit_fn[k], grid, 1, 1, JIT_TPB, 1, 1, 0, c.stream, params, nullptr),
                      "cuLaunchKernel");
}

}  // namespace mg
