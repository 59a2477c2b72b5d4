// Decode GEMV kernels for 3-bit codes, __nv_bfloat16 activations (see qeft_gemv2.cuh).
#define QEFT_GEMV2_KERNELS
#include "qeft_gemv2.cuh"

namespace qeft {
namespace g2 {
int dispatch_3b(const G2Args& a, int gt, cudaStream_t st) { return dispatch2<3, __nv_bfloat16>(a, gt, st); }
}  // namespace g2
}  // namespace qeft
