// Offline RTN quantization on device, bit-exact with the reference's
// _minmax_params (pkg/src/qeft/quantizer.py:115-120) and _nearest_codes
// (quantizer.py:211-218): per (row, group) min/max in fp32, scale computed in
// fp64 and stored fp32, codes = clip(rint((w64 - z) / s), 0, 2^b - 1) in fp64
// (CUDA rint is round-half-to-even like np.rint).
#include "qeft_common.cuh"
#include "qeft_internal.h"

namespace {

__global__ void rtn_kernel(const float* __restrict__ w, int oc, int m, int g, int bits,
                           float* __restrict__ sc, float* __restrict__ zr, uint8_t* __restrict__ codes) {
  const int ng = m > 0 ? (m + g - 1) / g : 0;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)oc * ng) return;
  const int r = (int)(idx / ng), gi = (int)(idx % ng);
  const int lo = gi * g, hi = min(lo + g, m);
  const float* row = w + (int64_t)r * m;
  float mn = row[lo], mx = row[lo];
  for (int j = lo + 1; j < hi; ++j) {
    mn = fminf(mn, row[j]);
    mx = fmaxf(mx, row[j]);
  }
  const int levels = (1 << bits) - 1;
  float s, z = mn;
  if (mx == mn)
    s = 1.f;
  else
    s = (float)(((double)mx - (double)mn) / (double)levels);
  sc[(int64_t)r * ng + gi] = s;
  zr[(int64_t)r * ng + gi] = z;
  for (int j = lo; j < hi; ++j) {
    double c = rint(((double)row[j] - (double)z) / (double)s);
    c = fmin(fmax(c, 0.0), (double)levels);
    codes[(int64_t)r * m + j] = (uint8_t)c;
  }
}

}  // namespace

namespace qeft {

int quantize_rtn(const float* w, int oc, int m, int g, int bits, float* s, float* z, uint8_t* codes,
                 cudaStream_t st) {
  QEFT_CHECK(bits == 3 || bits == 4, QEFT_ERR_SHAPE, "quantize_rtn: bits=%d", bits);
  QEFT_CHECK(g >= 1, QEFT_ERR_SHAPE, "quantize_rtn: g=%d", g);
  const int ng = m > 0 ? (m + g - 1) / g : 0;
  const int64_t n = (int64_t)oc * ng;
  if (!n) return 0;
  rtn_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(w, oc, m, g, bits, s, z, codes);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace qeft
