// Offline RTN quantization on device, bit-exact with the reference's
// _minmax_params (pkg/src/qeft/quantizer.py:115-120) and _nearest_codes
// (quantizer.py:211-218): per (row, group) min/max in fp32, scale computed in
// fp64 and stored fp32, codes = clip(rint((w64 - z) / s), 0, 2^b - 1) in fp64
// (CUDA rint is round-half-to-even like np.rint).
#include <algorithm>

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

// ---------------------------------------------------------------------------
// alpha-grid parameter search (quantizer.py:144-179, grid_search_group_params), bit-exact.
// Every fp64 operation is a separately rounded IEEE op in the reference's order (no FMA
// contraction), and the squared errors are summed in numpy's pairwise order
// (np.add.reduce on a contiguous float64 array: 8 running sums over blocks of <= 128
// elements, halves split at a multiple of 8 above that), so the chosen alpha -- the last
// minimum, larger alpha on ties -- is the reference's.

struct GridCand {
  double s, lo;
};

// error of candidate (s, lo) over w[a, a+n), summed exactly like numpy's pairwise_sum
QEFT_DEV double grid_err_leaf(const double* w, int a, int n, GridCand c, double levels) {
  auto e2 = [&](int i) {
    double q = rint(__ddiv_rn(__dsub_rn(w[i], c.lo), c.s));
    q = fmin(fmax(q, 0.0), levels);
    const double d = __dsub_rn(w[i], __dadd_rn(__dmul_rn(q, c.s), c.lo));
    return __dmul_rn(d, d);
  };
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, e2(a + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = e2(a + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], e2(a + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, e2(a + i));
  return res;
}

QEFT_DEV double grid_err(const double* w, int a, int n, GridCand c, double levels) {
  if (n <= 128) return grid_err_leaf(w, a, n, c, levels);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(grid_err(w, a, n2, c, levels), grid_err(w, a + n2, n - n2, c, levels));
}

// one warp per (row, group); lanes take alphas i = lane, lane + 32, ...
__global__ void __launch_bounds__(256) grid_kernel(const float* __restrict__ wq, int oc, int m, int g, int bits,
                                                   int steps, double amin, float* __restrict__ sc,
                                                   float* __restrict__ zr) {
  extern __shared__ double wsh[];  // [8 warps][g]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ng = (m + g - 1) / g;
  const int64_t item = (int64_t)blockIdx.x * 8 + warp;
  if (item >= (int64_t)oc * ng) return;
  const int r = (int)(item / ng), gi = (int)(item % ng);
  const int a0 = gi * g, n = min(g, m - a0);
  double* w = wsh + (size_t)warp * g;
  double mn = INFINITY, mx = -INFINITY;
  for (int i = lane; i < n; i += 32) {
    const double v = (double)wq[(int64_t)r * m + a0 + i];
    w[i] = v;
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __syncwarp();
  const int64_t out = (int64_t)r * ng + gi;
  if (mx == mn) {  // constant group: scale 1, zero = wmin (quantizer.py:157-158)
    if (lane == 0) {
      sc[out] = 1.f;
      zr[out] = (float)mn;
    }
    return;
  }
  const double levels = (double)((1 << bits) - 1);
  const double mid = __dmul_rn(0.5, __dadd_rn(mn, mx));
  const double da = __dsub_rn(1.0, amin);
  double best = INFINITY;
  int bi = -1;
  GridCand bc{0.0, 0.0};
  for (int i = lane; i < steps; i += 32) {
    // alphas = alpha_min + arange(steps) * (1 - alpha_min) / (steps - 1)   (left to right)
    const double al = steps == 1 ? 1.0 : __dadd_rn(amin, __ddiv_rn(__dmul_rn((double)i, da), (double)(steps - 1)));
    double lo, hi;
    if (al == 1.0) {  // keep the min-max endpoints bit-exact
      lo = mn;
      hi = mx;
    } else {
      lo = __dsub_rn(mid, __dmul_rn(al, __dsub_rn(mid, mn)));
      hi = __dadd_rn(mid, __dmul_rn(al, __dsub_rn(mx, mid)));
    }
    const GridCand c{__ddiv_rn(__dsub_rn(hi, lo), levels), lo};
    const double e = grid_err(w, 0, n, c, levels);
    if (e <= best) {  // increasing i within the lane: later (larger) alpha wins ties
      best = e;
      bi = i;
      bc = c;
    }
  }
  // across lanes: least error, then the larger alpha index
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const double os = __shfl_xor_sync(0xffffffffu, bc.s, o);
    const double ol = __shfl_xor_sync(0xffffffffu, bc.lo, o);
    if (oi >= 0 && (bi < 0 || ob < best || (ob == best && oi > bi))) {
      best = ob;
      bi = oi;
      bc = GridCand{os, ol};
    }
  }
  if (lane == 0) {
    sc[out] = (float)bc.s;
    zr[out] = (float)bc.lo;
  }
}

// nearest codes on fixed fp32 params (quantizer.py:211-218): clip(rint((w64 - z) / s))
__global__ void nearest_kernel(const float* __restrict__ w, int oc, int m, int g, int bits,
                               const float* __restrict__ sc, const float* __restrict__ zr,
                               uint8_t* __restrict__ codes) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)oc * m) return;
  const int r = (int)(idx / m), j = (int)(idx % m);
  const int ng = (m + g - 1) / g;
  const int gi = min(j / g, ng - 1);
  const double s = (double)sc[(int64_t)r * ng + gi], z = (double)zr[(int64_t)r * ng + gi];
  double c = rint(__ddiv_rn(__dsub_rn((double)w[idx], z), s));
  c = fmin(fmax(c, 0.0), (double)((1 << bits) - 1));
  codes[idx] = (uint8_t)c;
}

// ---------------------------------------------------------------------------
// OPTQ greedy rounding (quantizer.py:221-259, optq_quantize), bit-exact given the reference's
// U = chol(inv(H_damped)).T (computed on the host by numpy, as the reference does). Every
// weight w[r][j] receives the updates w -= err[r][i] * U[i][j] for i = 0 .. j-1 in increasing
// i, each as a rounded multiply then a rounded subtract -- the reference's
// `w[:, i+1:] -= np.outer(err, u[i, i+1:])` sequence. Left-looking blocks of kOptqB columns:
//   optq_update_kernel: apply to block [j0, j0+B) the errors of all columns < j0 (in order),
//   optq_block_kernel:  one thread per row walks the block sequentially (codes, err, in-block
//                       updates).
constexpr int kOptqB = 64;

__global__ void __launch_bounds__(256) optq_update_kernel(double* __restrict__ W, const double* __restrict__ E,
                                                          const double* __restrict__ U, int oc, int m, int j0,
                                                          int j1) {
  // tile: 32 columns x 64 rows; thread -> column c, rows r0 + 8 * (t / 32) + 0..7
  __shared__ double Es[64][33];
  __shared__ double Us[32][33];
  const int t = threadIdx.x, c = t & 31, rq = t >> 5;
  const int col = j0 + blockIdx.x * 32 + c;
  const int r0 = blockIdx.y * 64;
  double w[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int r = r0 + rq * 8 + q;
    w[q] = (r < oc && col < j1) ? W[(int64_t)r * m + col] : 0.0;
  }
  for (int i0 = 0; i0 < j0; i0 += 32) {
    const int ni = min(32, j0 - i0);
    for (int e = t; e < 64 * 32; e += 256) {  // E[r0 .. r0+63][i0 .. i0+31]
      const int rr = e >> 5, ii = e & 31, r = r0 + rr;
      Es[rr][ii] = (r < oc && ii < ni) ? E[(int64_t)r * m + i0 + ii] : 0.0;
    }
    for (int e = t; e < 32 * 32; e += 256) {  // U[i0 .. i0+31][block columns]
      const int ii = e >> 5, cc = e & 31, cj = j0 + blockIdx.x * 32 + cc;
      Us[ii][cc] = (ii < ni && cj < j1) ? U[(int64_t)(i0 + ii) * m + cj] : 0.0;
    }
    __syncthreads();
    for (int ii = 0; ii < ni; ++ii) {
      const double u = Us[ii][c];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = __dsub_rn(w[q], __dmul_rn(Es[rq * 8 + q][ii], u));
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int r = r0 + rq * 8 + q;
    if (r < oc && col < j1) W[(int64_t)r * m + col] = w[q];
  }
}

__global__ void __launch_bounds__(128) optq_block_kernel(const double* __restrict__ W, double* __restrict__ E,
                                                         const double* __restrict__ U, const float* __restrict__ sc,
                                                         const float* __restrict__ zr, uint8_t* __restrict__ codes,
                                                         int oc, int m, int g, int ng, int bits, int j0) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= oc) return;
  const int nb = min(kOptqB, m - j0);
  const double levels = (double)((1 << bits) - 1);
  double w[kOptqB];
#pragma unroll
  for (int k = 0; k < kOptqB; ++k) w[k] = k < nb ? W[(int64_t)r * m + j0 + k] : 0.0;
#pragma unroll
  for (int i = 0; i < kOptqB; ++i) {
    if (i >= nb) break;
    const int col = j0 + i;
    const int gi = min(col / g, ng - 1);
    const double s = (double)sc[(int64_t)r * ng + gi], z = (double)zr[(int64_t)r * ng + gi];
    double c = rint(__ddiv_rn(__dsub_rn(w[i], z), s));
    c = fmin(fmax(c, 0.0), levels);
    codes[(int64_t)r * m + col] = (uint8_t)c;
    const double dq = __dadd_rn(__dmul_rn(c, s), z);
    const double err = __ddiv_rn(__dsub_rn(w[i], dq), U[(int64_t)col * m + col]);
    E[(int64_t)r * m + col] = err;
#pragma unroll
    for (int j = i + 1; j < kOptqB; ++j)
      if (j < nb) w[j] = __dsub_rn(w[j], __dmul_rn(err, U[(int64_t)col * m + j0 + j]));
  }
}

}  // namespace

namespace qeft {

int optq_codes(double* w, const double* u, const float* s, const float* z, int oc, int m, int g, int bits,
               double* err, uint8_t* codes, cudaStream_t st) {
  QEFT_CHECK(bits == 3 || bits == 4, QEFT_ERR_SHAPE, "optq_codes: bits=%d", bits);
  QEFT_CHECK(g >= 1, QEFT_ERR_SHAPE, "optq_codes: g=%d", g);
  if (!oc || !m) return 0;
  const int ge = std::min(g, m), ng = (m + ge - 1) / ge;
  for (int j0 = 0; j0 < m; j0 += kOptqB) {
    const int j1 = std::min(m, j0 + kOptqB);
    if (j0 > 0) {
      optq_update_kernel<<<dim3((j1 - j0 + 31) / 32, (oc + 63) / 64), 256, 0, st>>>(w, err, u, oc, m, j0, j1);
      QEFT_CUDA(cudaGetLastError());
    }
    optq_block_kernel<<<(oc + 127) / 128, 128, 0, st>>>(w, err, u, s, z, codes, oc, m, ge, ng, bits, j0);
    QEFT_CUDA(cudaGetLastError());
  }
  return 0;
}

int grid_params(const float* w, int oc, int m, int g, int bits, int steps, double amin, float* s, float* z,
                cudaStream_t st) {
  QEFT_CHECK(bits == 3 || bits == 4, QEFT_ERR_SHAPE, "grid_params: bits=%d", bits);
  QEFT_CHECK(g >= 1 && steps >= 1, QEFT_ERR_SHAPE, "grid_params: g=%d steps=%d", g, steps);
  const int ng = m > 0 ? (m + g - 1) / g : 0;
  const int64_t n = (int64_t)oc * ng;
  if (!n) return 0;
  const int gs = std::min(g, m);
  const size_t smem = (size_t)8 * gs * sizeof(double);
  QEFT_CHECK(smem <= 200 * 1024, QEFT_ERR_SHAPE, "grid_params: group size %d too large", gs);
  if (smem > 48 * 1024) QEFT_CUDA(cudaFuncSetAttribute(grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  grid_kernel<<<(unsigned)((n + 7) / 8), 256, smem, st>>>(w, oc, m, gs, bits, steps, amin, s, z);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int nearest_codes(const float* w, int oc, int m, int g, int bits, const float* s, const float* z, uint8_t* codes,
                  cudaStream_t st) {
  QEFT_CHECK(bits == 3 || bits == 4, QEFT_ERR_SHAPE, "nearest_codes: bits=%d", bits);
  QEFT_CHECK(g >= 1, QEFT_ERR_SHAPE, "nearest_codes: g=%d", g);
  const int64_t n = (int64_t)oc * m;
  if (!n) return 0;
  nearest_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, oc, m, std::min(g, m), bits, s, z, codes);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

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
