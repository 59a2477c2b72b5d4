// tcgen05 prefill / fine-tune GEMMs (placeholder until the tcgen05 kernel lands).
#include "qeft_common.cuh"
#include "qeft_internal.h"

namespace qeft {

size_t gemm_workspace_bytes(const qeft_linear_t* L, int T) { (void)L; (void)T; return 0; }

int gemm_fwd(const qeft_linear_t*, const void*, int64_t, void*, int64_t, int, void*, size_t, cudaStream_t) {
  set_error("gemm_fwd: not built");
  return QEFT_ERR_LAYOUT;
}
int gemm_dgrad(const qeft_linear_t*, const void*, int64_t, void*, int64_t, int, int, void*, size_t,
               cudaStream_t) {
  set_error("gemm_dgrad: not built");
  return QEFT_ERR_LAYOUT;
}
int gemm_wgrad(const qeft_linear_t*, const void*, int64_t, const void*, int64_t, float*, int, int, void*,
               size_t, cudaStream_t) {
  set_error("gemm_wgrad: not built");
  return QEFT_ERR_LAYOUT;
}

}  // namespace qeft
