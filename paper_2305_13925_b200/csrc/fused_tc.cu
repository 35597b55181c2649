// Fused tcgen05 precoder kernel for complex64 (placeholder until implemented).
#include "xl_common.cuh"
#include "fused_tc.cuh"

namespace xl {
bool fused_supported(int, int, int, int) { return false; }
size_t fused_ws_bytes(int, int, int64_t, int, int) { return 0; }
int launch_fused(int, int, int, const void*, int64_t, int, int, double, const double*, double, int,
                 double, void*, void*, double*, double*, double*, void*, int32_t*, void*, size_t,
                 cudaStream_t) {
  set_error("fused path not built");
  return XL_ERR_UNSUPPORTED;
}
}  // namespace xl
