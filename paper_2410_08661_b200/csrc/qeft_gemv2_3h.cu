// Decode GEMV kernels for 3-bit codes, __half activations (see qeft_gemv2.cuh).
#define QEFT_GEMV2_KERNELS
#include "qeft_gemv2.cuh"

namespace qeft {
namespace g2 {
int dispatch_3h(const G2Args& a, int gt, cudaStream_t st) { return dispatch2<3, __half>(a, gt, st); }
}  // namespace g2
}  // namespace qeft
