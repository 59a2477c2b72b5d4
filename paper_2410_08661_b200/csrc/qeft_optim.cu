// Weak-column optimizer step over the flat fp32 gradient bucket.
//
// Replaces the reference's per-layer numpy loop (pkg/src/qeft/tuning.py:226-236):
//   gnorm = sqrt(sum over ALL weak blocks of fp64 g^2); scale = max/(gnorm+1e-12)
//   if gnorm > max; then adam_step (tuning.py:148-160) on every block.
// The sum of squares is a deterministic two-pass fp64 reduction (fixed grid, fixed
// order), the clip factor is computed on device (no host sync), and Adam is
// evaluated with explicit round-to-nearest fp32 ops in the reference's order so
// the update matches numpy's float32 arithmetic bit for bit given the same
// gradient. A non-finite norm suppresses the whole update and raises a device
// flag (the reference raises DivergenceError before touching any weight).
#include <algorithm>

#include "qeft_common.cuh"
#include "qeft_internal.h"

using namespace qeft;

namespace {

constexpr int kSqBlocks = 1184;  // 8 x 148 SMs; scratch holds one double per block
constexpr int kSqThreads = 256;

// sum of (g / d)^2 in fp64, where g / d is rounded to fp32 first -- the reference divides the
// fp32 accumulators by grad_accum (tuning.py:228) before squaring them in fp64 (tuning.py:230)
__device__ __forceinline__ double sq_div(float g, float d) {
  const float q = __fdiv_rn(g, d);
  return (double)q * q;
}

__global__ void __launch_bounds__(kSqThreads) sqnorm_partial(const float* __restrict__ g, int64_t n, float d,
                                                             double* __restrict__ part) {
  __shared__ double red[kSqThreads / 32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (((uintptr_t)g & 15) == 0) {
    const int64_t n4 = n >> 2;
    for (int64_t q = i; q < n4; q += stride) {
      const float4 v = reinterpret_cast<const float4*>(g)[q];
      acc += sq_div(v.x, d) + sq_div(v.y, d) + sq_div(v.z, d) + sq_div(v.w, d);
    }
    for (int64_t q = (n4 << 2) + i; q < n; q += stride) acc += sq_div(g[q], d);
  } else {
    for (int64_t q = i; q < n; q += stride) acc += sq_div(g[q], d);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kSqThreads / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void sqnorm_final(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    *out = s;
  }
}

__global__ void div_kernel(float* __restrict__ g, int64_t n, float d) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    g[i] = __fdiv_rn(g[i], d);
}

struct AdamC {
  double max_norm;  // the reference compares and divides with the Python float (tuning.py:231-232)
  float lr, b1, omb1, b2, omb2, bc1, bc2, eps;
};

// clip factor from the global fp64 sum of squares: (float)(max / (gnorm + 1e-12)) when
// gnorm > max (the Python float scale, multiplied into the fp32 grads in fp32), else 1
__device__ __forceinline__ float clip_scale(double s2, double max_norm) {
  const double gn = sqrt(s2);
  return (max_norm > 0.0 && gn > max_norm) ? (float)(max_norm / (gn + 1e-12)) : 1.f;
}

__device__ __forceinline__ void adam_one(float& w, float& m, float& v, float g, const AdamC& c) {
  // tuning.py:154-159, float32 arithmetic in numpy's evaluation order, no FMA contraction
  m = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(c.omb1, g));
  v = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(__fmul_rn(c.omb2, g), g));
  const float mh = __fdiv_rn(m, c.bc1);
  const float vh = __fdiv_rn(v, c.bc2);
  const float up = __fdiv_rn(__fmul_rn(c.lr, mh), __fadd_rn(__fsqrt_rn(vh), c.eps));
  w = __fsub_rn(w, up);
}

__global__ void adam_kernel(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
                            const float* __restrict__ g, int64_t n, const double* __restrict__ sq,
                            AdamC c, int* __restrict__ flag) {
  const double s2 = *sq;
  if (!isfinite(s2)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 1;
    return;
  }
  // tuning.py:230-232: the scale is a Python float; numpy multiplies the float32
  // gradient by it in float32
  const float sc = clip_scale(s2, c.max_norm);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float wi = w[i], mi = m[i], vi = v[i];
    const float gi = sc == 1.f ? g[i] : __fmul_rn(g[i], sc);
    adam_one(wi, mi, vi, gi, c);
    w[i] = wi;
    m[i] = mi;
    v[i] = vi;
  }
}

template <typename T>
__device__ __forceinline__ void put(void* p, int64_t i, float v) {
  ((T*)p)[i] = from_f32<T>(v);
}

// The whole fine-tune optimizer step in ONE pass over the flat bucket (after the sum-of-squares
// pass): g / grad_accum (fp32, as tuning.py:228) -> global clip (tuning.py:229-233) -> fp32 Adam
// (tuning.py:148-160) -> the layer's fp16/bf16 kernel shadow (weak16, tile layout). One CTA row
// loop per layer (blockIdx.y), lanes along the weak columns: coalesced, no div/mod per element.
__global__ void __launch_bounds__(256) adam_step_kernel(float* __restrict__ w, float* __restrict__ m,
                                                        float* __restrict__ v, const float* __restrict__ g,
                                                        const qeft_shadow_desc_t* __restrict__ descs, float div,
                                                        const double* __restrict__ sq, AdamC c,
                                                        int* __restrict__ flag) {
  const double s2 = *sq;
  if (!isfinite(s2)) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *flag = 1;
    return;
  }
  const float sc = clip_scale(s2, c.max_norm);
  const qeft_shadow_desc_t L = descs[blockIdx.y];
  const int kw = L.k;
  for (int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < L.oc; r += gridDim.x * (blockDim.x / 32)) {
    const int64_t row = L.offset + (int64_t)r * kw;
    for (int j = threadIdx.x & 31; j < kw; j += 32) {
      const int64_t i = row + j;
      float wi = w[i], mi = m[i], vi = v[i];
      float gi = __fdiv_rn(g[i], div);
      if (sc != 1.f) gi = __fmul_rn(gi, sc);
      adam_one(wi, mi, vi, gi, c);
      w[i] = wi;
      m[i] = mi;
      v[i] = vi;
      if (L.act_dtype == QEFT_F16)
        put<__half>(L.weak16, weak_off(r, j, L.k_pad), wi);
      else
        put<__nv_bfloat16>(L.weak16, weak_off(r, j, L.k_pad), wi);
    }
  }
}

__global__ void shadow_kernel(const float* __restrict__ w32, const qeft_shadow_desc_t* __restrict__ d) {
  const qeft_shadow_desc_t L = d[blockIdx.y];
  const int64_t n = (int64_t)L.oc * L.k;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int r = (int)(i / L.k), j = (int)(i % L.k);
    const float v = w32[L.offset + i];
    if (L.act_dtype == QEFT_F16)
      put<__half>(L.weak16, weak_off(r, j, L.k_pad), v);
    else
      put<__nv_bfloat16>(L.weak16, weak_off(r, j, L.k_pad), v);
  }
}

inline unsigned grid_for(int64_t n, int threads = 256, int cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (unsigned)(b > cap ? cap : b);
}

}  // namespace

namespace qeft {

int grad_sqnorm(const float* g, int64_t n, double* scratch, double* out, cudaStream_t st, float div) {
  sqnorm_partial<<<kSqBlocks, kSqThreads, 0, st>>>(g, n, div, scratch);
  QEFT_CUDA(cudaGetLastError());
  sqnorm_final<<<1, 1024, 0, st>>>(scratch, kSqBlocks, out);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int div_scalar(float* g, int64_t n, float d, cudaStream_t st) {
  if (n <= 0) return 0;
  div_kernel<<<grid_for(n), 256, 0, st>>>(g, n, d);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int adam_step_flat(float* w, float* m, float* v, const float* g, const qeft_shadow_desc_t* descs, int n_layers,
                   int max_rows, float div, const double* sqnorm, double max_norm, float lr, float c_b1,
                   float c_1mb1, float c_b2, float c_1mb2, float bc1, float bc2, float eps, int* flag,
                   cudaStream_t st) {
  if (n_layers <= 0) return 0;
  QEFT_CHECK(n_layers <= 65535, QEFT_ERR_SHAPE, "adam_step: too many layers");
  QEFT_CHECK(div != 0.f, QEFT_ERR_SHAPE, "adam_step: zero divisor");
  AdamC c{max_norm, lr, c_b1, c_1mb1, c_b2, c_1mb2, bc1, bc2, eps};
  const int rows_per_cta = 8;  // one warp per row
  unsigned gx = (unsigned)std::min<int64_t>(((int64_t)max_rows + rows_per_cta - 1) / rows_per_cta, 148 * 4);
  adam_step_kernel<<<dim3(std::max(gx, 1u), n_layers), 256, 0, st>>>(w, m, v, g, descs, div, sqnorm, c, flag);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int adam_clip(float* w, float* m, float* v, const float* g, int64_t n, const double* sqnorm,
              double max_norm, float lr, float c_b1, float c_1mb1, float c_b2, float c_1mb2, float bc1,
              float bc2, float eps, int* flag, cudaStream_t st) {
  if (n <= 0) return 0;
  AdamC c{max_norm, lr, c_b1, c_1mb1, c_b2, c_1mb2, bc1, bc2, eps};
  adam_kernel<<<grid_for(n), 256, 0, st>>>(w, m, v, g, n, sqnorm, c, flag);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int weak_shadow(const float* w32, const qeft_shadow_desc_t* d, int n_layers, int max_elems,
                cudaStream_t st) {
  if (n_layers <= 0) return 0;
  QEFT_CHECK(n_layers <= 65535, QEFT_ERR_SHAPE, "weak_shadow: too many layers");
  shadow_kernel<<<dim3(grid_for(max_elems, 256, 64), n_layers), 256, 0, st>>>(w32, d);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace qeft
