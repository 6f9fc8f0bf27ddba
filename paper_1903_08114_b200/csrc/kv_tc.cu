// tcgen05 (5th-gen tensor core) fused K·V kernel for sm_100a — see DESIGN.md.
// Placeholder until the tensor-core path lands: reports "not compiled".
#include "gp_common.cuh"

namespace gp {
bool kv_tc_supported(const gp_kv_desc*, int) { return false; }
size_t kv_tc_workspace(const gp_kv_desc*, int) { return 0; }
int kv_tc(const gp_kv_desc*, const float*, int64_t, int, float*, int64_t, void*, size_t, cudaStream_t) {
  return set_error(GP_EUNSUPPORTED, "tcgen05 K·V kernel not compiled in");
}
}  // namespace gp

extern "C" int gp_has_tcgen05(void) { return 0; }
