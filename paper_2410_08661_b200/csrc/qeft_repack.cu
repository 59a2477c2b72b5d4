// Format conversion between the reference's packed bytes
// (pkg/src/qeft/packing.py:24-72: row-major, LSB-first; 4-bit even column in the
// low nibble, 3-bit one bitstream per row padded to a byte) and the B200 tile
// layout documented in qeft_common.cuh; plus the group-parameter / weak-column
// packers, the input-column gather and a dequantize-to-dense debug kernel.
#include <algorithm>

#include "qeft_common.cuh"
#include "qeft_internal.h"

using namespace qeft;

namespace {

__device__ __forceinline__ int ref_code(const uint8_t* ref, int rbytes, int bits, int r, int j) {
  const uint8_t* row = ref + (int64_t)r * rbytes;
  if (bits == 4) {
    const uint8_t b = row[j >> 1];
    return (j & 1) ? (b >> 4) : (b & 15);
  }
  const int pos = 3 * j;  // LSB-first bitstream
  uint32_t w = row[pos >> 3];
  if ((pos >> 3) + 1 < rbytes) w |= (uint32_t)row[(pos >> 3) + 1] << 8;
  return (w >> (pos & 7)) & 7;
}

__device__ __forceinline__ int tile_code(const uint32_t* qw, int bits, int m_pad, int r, int j) {
  const CodeLoc L = locate_code(bits, m_pad, r, j);
  if (bits == 4) return (qw[L.lo_word] >> L.lo_shift) & 15;
  const int lo = (qw[L.lo_word] >> L.lo_shift) & 3;
  const int hi = (qw[L.hi_word] >> L.hi_shift) & 1;
  return lo | (hi << 2);
}

// one thread per code; the destination is zeroed beforehand
__global__ void ref_to_tiles_kernel(const uint8_t* __restrict__ ref, int oc, int m, int bits,
                                    int m_pad, uint32_t* __restrict__ qw) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)oc * m) return;
  const int r = (int)(idx / m), j = (int)(idx % m);
  const int rbytes = bits == 4 ? (m + 1) / 2 : (3 * m + 7) / 8;
  const int c = ref_code(ref, rbytes, bits, r, j);
  if (!c) return;
  const CodeLoc L = locate_code(bits, m_pad, r, j);
  if (bits == 4) {
    atomicOr(qw + L.lo_word, (uint32_t)c << L.lo_shift);
  } else {
    if (c & 3) atomicOr(qw + L.lo_word, (uint32_t)(c & 3) << L.lo_shift);
    if (c & 4) atomicOr(qw + L.hi_word, 1u << L.hi_shift);
  }
}

// one thread per reference output byte
__global__ void tiles_to_ref_kernel(const uint32_t* __restrict__ qw, int oc, int m, int bits,
                                    int m_pad, uint8_t* __restrict__ ref) {
  const int rbytes = bits == 4 ? (m + 1) / 2 : (3 * m + 7) / 8;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)oc * rbytes) return;
  const int r = (int)(idx / rbytes), b = (int)(idx % rbytes);
  uint32_t out = 0;
  if (bits == 4) {
    const int j = 2 * b;
    out = tile_code(qw, 4, m_pad, r, j);
    if (j + 1 < m) out |= tile_code(qw, 4, m_pad, r, j + 1) << 4;
  } else {
    for (int bit = 0; bit < 8; ++bit) {
      const int pos = 8 * b + bit, j = pos / 3;
      if (j >= m) break;
      out |= ((tile_code(qw, 3, m_pad, r, j) >> (pos % 3)) & 1u) << bit;
    }
  }
  ref[idx] = (uint8_t)out;
}

template <typename T>
__global__ void pack_sz_kernel(const float* __restrict__ scales, const float* __restrict__ zeros,
                               int oc, int oc_pad, int ng, T* __restrict__ sz) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)oc_pad * ng) return;
  const int r = (int)(idx / ng), gi = (int)(idx % ng);
  float s = 0.f, z = 0.f;
  if (r < oc) { s = scales[(int64_t)r * ng + gi]; z = zeros[(int64_t)r * ng + gi]; }
  const int64_t o = (((int64_t)(r >> 4) * ng + gi) * 16 + (r & 15)) * 2;
  sz[o] = from_f32<T>(s);
  sz[o + 1] = from_f32<T>(z);
}

// decode-GEMV copy of the group parameters: fp16 (scale, zero) half2 pairs laid out
// [oc_pad/16][ng16][8][2] (ng16 = ceil(m_pad/g), zero beyond ng): the 16 rows of a (row-block,
// group) are 64 contiguous bytes and rows r, r + 8 of the MMA fragment sit side by side.
__global__ void pack_sz16_kernel(const float* __restrict__ scales, const float* __restrict__ zeros,
                                 int oc, int oc_pad, int ng, int ng16, __half2* __restrict__ sz) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)oc_pad * ng16) return;
  const int r = (int)(idx / ng16), gi = (int)(idx % ng16);
  float s = 0.f, z = 0.f;
  if (r < oc && gi < ng) { s = scales[(int64_t)r * ng + gi]; z = zeros[(int64_t)r * ng + gi]; }
  const int rr = r & 15;
  sz[(((int64_t)(r >> 4) * ng16 + gi) * 8 + (rr & 7)) * 2 + (rr >> 3)] = __floats2half2_rn(s, z);
}

template <typename T>
__global__ void pack_weak_kernel(const float* __restrict__ weak, int oc, int k, int oc_pad,
                                 int k_pad, T* __restrict__ w16) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)oc_pad * k_pad) return;
  const int r = (int)(idx / k_pad), j = (int)(idx % k_pad);
  w16[weak_off(r, j, k_pad)] = from_f32<T>((r < oc && j < k) ? weak[(int64_t)r * k + j] : 0.f);
}

// out[r][col] (original column order, fp32) = dequantized code * s + z, weak restored
template <typename T>
__global__ void dequant_full_kernel(qeft_linear_t L, float* __restrict__ out) {
  const int kk = L.m_pad + L.k_pad;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)L.oc * kk) return;
  const int r = (int)(idx / kk), j = (int)(idx % kk);
  const int col = L.colmap[j];
  if (col < 0) return;
  float v;
  if (j < L.m_pad) {
    const int c = tile_code((const uint32_t*)L.qweight, L.bits, L.m_pad, r, j);
    const int gi = min(j / L.g, L.ng - 1);
    const float* sz = (const float*)L.sz + (((int64_t)(r >> 4) * L.ng + gi) * 16 + (r & 15)) * 2;
    v = (float)c * sz[0] + sz[1];
  } else {
    v = to_f32<T>(((const T*)L.weak16)[weak_off(r, j - L.m_pad, L.k_pad)]);
  }
  out[(int64_t)r * L.ic + col] = v;
}

// xb[t][j] = colmap[j] >= 0 ? x[t][colmap[j]] : 0   (B200 K order)
template <typename T>
__global__ void gather_cols_kernel(const T* __restrict__ x, int64_t ldx, const int* __restrict__ colmap,
                                   int kk, int rows, T* __restrict__ xb) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)rows * kk) return;
  const int t = (int)(idx / kk), j = (int)(idx % kk);
  const int c = colmap[j];
  xb[idx] = c >= 0 ? x[(int64_t)t * ldx + c] : from_f32<T>(0.f);
}

// Row-staged column gather for the GEMM's B200 K order: a CTA loads one source row (src_cols
// elements, 16-byte vectors) into shared memory, then writes the gathered row 8 elements per
// thread (colmap read as two int4, one 16-byte store). kk % 8 == 0.
template <typename T>
__global__ void __launch_bounds__(256) gather_rows_kernel(const T* __restrict__ x, int64_t ldx, int src_cols,
                                                          const int* __restrict__ colmap, int kk, int rows,
                                                          T* __restrict__ xb, int vec) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  T* row = reinterpret_cast<T*>(sm_raw);
  const T zero = from_f32<T>(0.f);
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const T* src = x + (int64_t)r * ldx;
    __syncthreads();  // previous row consumed
    if (vec) {
      for (int i = threadIdx.x; i < src_cols / 8; i += blockDim.x)
        reinterpret_cast<uint4*>(row)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {
      for (int i = threadIdx.x; i < src_cols; i += blockDim.x) row[i] = src[i];
    }
    __syncthreads();
    T* dst = xb + (int64_t)r * kk;
    for (int j8 = threadIdx.x; j8 < kk / 8; j8 += blockDim.x) {
      const int4 c0 = reinterpret_cast<const int4*>(colmap)[2 * j8];
      const int4 c1 = reinterpret_cast<const int4*>(colmap)[2 * j8 + 1];
      const int cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      uint4 o;
      T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
      for (int e = 0; e < 8; ++e) oe[e] = cs[e] >= 0 ? row[cs[e]] : zero;
      reinterpret_cast<uint4*>(dst)[j8] = o;
    }
  }
}

// Inverse: out[r][c] (+)= xb[r][j] for colmap[j] = c (the dX of a non-structured layer, written
// by the GEMM in B200 order). The CTA builds the inverse map in shared memory once, then per
// row stages the B200-order row and writes the output row 8 columns per thread.
template <typename T>
__global__ void __launch_bounds__(256) scatter_rows_kernel(const T* __restrict__ xb, int kk,
                                                           const int* __restrict__ colmap, int ic, int rows,
                                                           T* __restrict__ out, int64_t ldo, int accumulate,
                                                           int vec) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  int* inv = reinterpret_cast<int*>(sm_raw);
  T* row = reinterpret_cast<T*>(sm_raw + (size_t)((ic + 3) / 4) * 16);
  for (int c = threadIdx.x; c < ic; c += blockDim.x) inv[c] = -1;
  __syncthreads();
  for (int j = threadIdx.x; j < kk; j += blockDim.x) {
    const int c = colmap[j];
    if (c >= 0 && c < ic) inv[c] = j;
  }
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    __syncthreads();
    const uint4* src = reinterpret_cast<const uint4*>(xb + (int64_t)r * kk);
    for (int i = threadIdx.x; i < kk / 8; i += blockDim.x) reinterpret_cast<uint4*>(row)[i] = src[i];
    __syncthreads();
    T* dst = out + (int64_t)r * ldo;
    if (vec) {
      for (int c8 = threadIdx.x; c8 < ic / 8; c8 += blockDim.x) {
        uint4 o = accumulate ? reinterpret_cast<const uint4*>(dst)[c8] : make_uint4(0u, 0u, 0u, 0u);
        T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = inv[8 * c8 + e];
          const float v = j >= 0 ? to_f32<T>(row[j]) : 0.f;
          oe[e] = from_f32<T>(accumulate ? to_f32<T>(oe[e]) + v : v);
        }
        reinterpret_cast<uint4*>(dst)[c8] = o;
      }
    } else {
      for (int c = threadIdx.x; c < ic; c += blockDim.x) {
        const int j = inv[c];
        const float v = j >= 0 ? to_f32<T>(row[j]) : 0.f;
        dst[c] = from_f32<T>(accumulate ? to_f32<T>(dst[c]) + v : v);
      }
    }
  }
}

inline unsigned nblk(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

}  // namespace

namespace qeft {

int repack_ref_to_tiles(const uint8_t* ref, int oc, int m, int bits, void* qw, cudaStream_t st) {
  const int m_pad = pad_to(m, 128), oc_pad = pad_to(oc, 16);
  const size_t bytes = (size_t)(oc_pad / 16) * rowblock_bytes(bits, m_pad);
  QEFT_CUDA(cudaMemsetAsync(qw, 0, bytes, st));
  if ((int64_t)oc * m == 0) return 0;
  ref_to_tiles_kernel<<<nblk((int64_t)oc * m), 256, 0, st>>>(ref, oc, m, bits, m_pad, (uint32_t*)qw);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int repack_tiles_to_ref(const void* qw, int oc, int m, int bits, uint8_t* ref, cudaStream_t st) {
  const int m_pad = pad_to(m, 128);
  const int rbytes = bits == 4 ? (m + 1) / 2 : (3 * m + 7) / 8;
  if ((int64_t)oc * rbytes == 0) return 0;
  tiles_to_ref_kernel<<<nblk((int64_t)oc * rbytes), 256, 0, st>>>((const uint32_t*)qw, oc, m, bits,
                                                                 m_pad, ref);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int pack_sz(const float* s, const float* z, int oc, int ng, void* out, cudaStream_t st) {
  const int oc_pad = pad_to(oc, 16);
  if ((int64_t)oc_pad * ng == 0) return 0;
  pack_sz_kernel<float><<<nblk((int64_t)oc_pad * ng), 256, 0, st>>>(s, z, oc, oc_pad, ng, (float*)out);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

size_t sz16_bytes(int oc, int m, int g) {
  if (m <= 0 || g <= 0) return 0;
  return (size_t)(pad_to(oc, 16) / 16) * ((pad_to(m, 128) + g - 1) / g) * 64;
}

int pack_sz16(const float* s, const float* z, int oc, int m, int g, void* out, cudaStream_t st) {
  QEFT_CHECK(g > 0 && m >= 0, QEFT_ERR_SHAPE, "pack_sz16: g=%d m=%d", g, m);
  if (m == 0) return 0;
  const int oc_pad = pad_to(oc, 16), ng = (m + g - 1) / g, ng16 = (pad_to(m, 128) + g - 1) / g;
  pack_sz16_kernel<<<nblk((int64_t)oc_pad * ng16), 256, 0, st>>>(s, z, oc, oc_pad, ng, ng16, (__half2*)out);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int pack_weak(const float* w, int oc, int k, int dtype, void* out, cudaStream_t st) {
  const int oc_pad = pad_to(oc, 16), k_pad = pad_to(k, 64);
  if ((int64_t)oc_pad * k_pad == 0) return 0;
  if (dtype == QEFT_F16)
    pack_weak_kernel<__half><<<nblk((int64_t)oc_pad * k_pad), 256, 0, st>>>(w, oc, k, oc_pad, k_pad,
                                                                           (__half*)out);
  else
    pack_weak_kernel<__nv_bfloat16><<<nblk((int64_t)oc_pad * k_pad), 256, 0, st>>>(
        w, oc, k, oc_pad, k_pad, (__nv_bfloat16*)out);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int dequant_full(const qeft_linear_t* L, float* out, cudaStream_t st) {
  const int64_t n = (int64_t)L->oc * (L->m_pad + L->k_pad);
  if (!n) return 0;
  if (L->act_dtype == QEFT_F16)
    dequant_full_kernel<__half><<<nblk(n), 256, 0, st>>>(*L, out);
  else
    dequant_full_kernel<__nv_bfloat16><<<nblk(n), 256, 0, st>>>(*L, out);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int gather_rows(const void* x, int64_t ldx, int src_cols, const int* colmap, int kk, int rows, int dtype,
                void* xb, cudaStream_t st) {
  if ((int64_t)rows * kk == 0) return 0;
  const size_t smem = (size_t)src_cols * 2 + 16;
  if (kk % 8 != 0 || (((uintptr_t)colmap) & 15) != 0 || (((uintptr_t)xb) & 15) != 0 || smem > 200 * 1024)
    return gather_cols(x, ldx, colmap, kk, rows, dtype, xb, st);
  const int vec = ldx % 8 == 0 && src_cols % 8 == 0 && (((uintptr_t)x) & 15) == 0;
  const int grid = std::min(rows, 148 * 4);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gather_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    gather_rows_kernel<T><<<grid, 256, smem, st>>>((const T*)x, ldx, src_cols, colmap, kk, rows, (T*)xb, vec);
  };
  if (dtype == QEFT_F16) go(__half{});
  else go(__nv_bfloat16{});
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int scatter_rows(const void* xb, int kk, const int* colmap, int ic, int rows, int dtype, void* out, int64_t ldo,
                 int accumulate, cudaStream_t st) {
  if ((int64_t)rows * ic == 0) return 0;
  const size_t smem = (size_t)((ic + 3) / 4) * 16 + (size_t)kk * 2;
  QEFT_CHECK(kk % 8 == 0 && (((uintptr_t)xb) & 15) == 0 && smem <= 200 * 1024, QEFT_ERR_SHAPE,
             "scatter_rows: kk=%d ic=%d", kk, ic);
  const int vec = ic % 8 == 0 && ldo % 8 == 0 && (((uintptr_t)out) & 15) == 0;
  const int grid = std::min(rows, 148 * 4);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(scatter_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    scatter_rows_kernel<T><<<grid, 256, smem, st>>>((const T*)xb, kk, colmap, ic, rows, (T*)out, ldo, accumulate,
                                                    vec);
  };
  if (dtype == QEFT_F16) go(__half{});
  else go(__nv_bfloat16{});
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int gather_cols(const void* x, int64_t ldx, const int* colmap, int kk, int rows, int dtype, void* xb,
                cudaStream_t st) {
  const int64_t n = (int64_t)rows * kk;
  if (!n) return 0;
  if (dtype == QEFT_F16)
    gather_cols_kernel<__half><<<nblk(n), 256, 0, st>>>((const __half*)x, ldx, colmap, kk, rows,
                                                        (__half*)xb);
  else
    gather_cols_kernel<__nv_bfloat16><<<nblk(n), 256, 0, st>>>(
        (const __nv_bfloat16*)x, ldx, colmap, kk, rows, (__nv_bfloat16*)xb);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace qeft
