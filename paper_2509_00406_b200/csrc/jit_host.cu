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
typedef int (*PFN_setattr)(void*, int, int);
typedef int (*PFN_occ)(int*, void*, int, size_t);

struct Driver {
  PFN_load load = nullptr;
  PFN_getfn getfn = nullptr;
  PFN_launch launch = nullptr;
  PFN_unload unload = nullptr;
  PFN_errstr errstr = nullptr;
  PFN_setattr setattr = nullptr;
  PFN_occ occupancy = nullptr;
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
      d.setattr = (PFN_setattr)dlsym(h, "cuFuncSetAttribute");
      d.occupancy = (PFN_occ)dlsym(h, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
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

const char* kPatchNames[5] = {"mg_patch_grad", "mg_patch_hess", "mg_patch_hess_psd", "mg_patch_hvp",
                              "mg_patch_hvp_psd"};

void jit_patch_load(Problem& p, const void* image) {
  MG_CUDA(cudaFree(nullptr));
  Driver& d = driver();
  jit_patch_unload(p);
  drv_check(d.load(&p.patch_module, image), "cuModuleLoadData (patch module)");
  for (int i = 0; i < 5; ++i) drv_check(d.getfn(&p.patch_fn[i], p.patch_module, kPatchNames[i]), kPatchNames[i]);
  p.jattr_dirty = true;
}

void jit_patch_unload(Problem& p) {
  if (p.patch_module && driver().unload) driver().unload(p.patch_module);
  p.patch_module = nullptr;
  for (auto& f : p.patch_fn) f = nullptr;
}

void jit_patch_launch(const Problem& p, Mode mode, bool psd, void* args, int64_t np, int nvp_max, int blocks_max,
                      size_t smem, cudaStream_t s, int64_t grid) {
  Driver& d = driver();
  const int k = mode == MODE_GRAD ? 0 : mode == MODE_HESS ? (psd ? 2 : 1) : (psd ? 4 : 3);
  if (mode != MODE_GRAD && mode != MODE_HESS && mode != MODE_HVP)
    throw Error(MG_ERR_UNSUPPORTED, "traced patch kernels assemble grad / Hessian / HVP only");
  if (d.setattr) drv_check(d.setattr(p.patch_fn[k], 8 /* CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES */,
                                     (int)smem), "cuFuncSetAttribute");
  void* params[3] = {args, &nvp_max, &blocks_max};
  if (grid < 0 || grid > np) grid = np;
  if (grid > 0)
    drv_check(d.launch(p.patch_fn[k], (unsigned)grid, 1, 1, 128, 1, 1, (unsigned)smem, s, params, nullptr),
              "cuLaunchKernel (patch module)");
}

const char* kRowNames[5] = {"mg_rows_grad", "mg_rows_hess", "mg_rows_hess_psd", "mg_rows_hvp", "mg_rows_hvp_psd"};

void jit_rows_load(Problem& p, const void* image) {
  MG_CUDA(cudaFree(nullptr));
  Driver& d = driver();
  jit_rows_unload(p);
  drv_check(d.load(&p.row_module, image), "cuModuleLoadData (row module)");
  for (int i = 0; i < 5; ++i) drv_check(d.getfn(&p.row_fn[i], p.row_module, kRowNames[i]), kRowNames[i]);
}

void jit_rows_unload(Problem& p) {
  if (p.row_module && driver().unload) driver().unload(p.row_module);
  p.row_module = nullptr;
  for (auto& f : p.row_fn) f = nullptr;
  p.ev_jit = false;
}

void jit_rows_launch(const Problem& p, Mode mode, bool psd, void* args, int64_t grid, int block, size_t smem,
                     cudaStream_t s, bool persistent) {
  Driver& d = driver();
  if (mode != MODE_GRAD && mode != MODE_HESS && mode != MODE_HVP)
    throw Error(MG_ERR_UNSUPPORTED, "traced row kernels assemble grad / Hessian / HVP only");
  const int k = mode == MODE_GRAD ? 0 : mode == MODE_HESS ? (psd ? 2 : 1) : (psd ? 4 : 3);
  if (d.setattr) drv_check(d.setattr(p.row_fn[k], 8 /* CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES */,
                                     (int)smem), "cuFuncSetAttribute");
  if (persistent && d.occupancy) {  // the staged kernels walk row blocks grid-stride: as many CTAs as are resident
    int per_sm = 0, dev = 0, sms = 148;
    drv_check(d.occupancy(&per_sm, p.row_fn[k], block, smem), "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    MG_CUDA(cudaGetDevice(&dev));
    MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm > 0 && (int64_t)sms * per_sm < grid) grid = (int64_t)sms * per_sm;
  }
  void* params[1] = {args};
  if (grid > 0)
    drv_check(d.launch(p.row_fn[k], (unsigned)grid, 1, 1, (unsigned)block, 1, 1, (unsigned)smem, s, params, nullptr),
              "cuLaunchKernel (row module)");
}

}  // namespace mg
