// Deterministic patch-owner assembly (placeholder until the patch layout lands).
#include "mg_internal.cuh"

namespace mg {

bool patch_supported(const Problem&) { return false; }
void build_patch_layout(Problem& p, cudaStream_t) { p.layout_ready = false; }
int64_t launch_patch(const Problem&, Mode, const LaunchCtx&, int64_t) {
  throw Error(MG_ERR_UNSUPPORTED, "patch assembly not available");
}

}  // namespace mg
