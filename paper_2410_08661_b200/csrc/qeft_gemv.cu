// Decode GEMV for the QEFT mixed-precision layer, N = 1..16 activation columns.
//
// Replaces the reference's matvec paths (pkg/src/qeft/kernels.py:66-157,
// `_grouped_accumulate`): y = sum_g s_g * (c_g . x_g) + z_g * sum(x_g) + W_weak . x_weak.
//
// HBM-bound design (B200):
//   * grid = (K slices, 64-row groups); CTA = 4 warps, warp w streams row-block
//     4*rg + w over the CTA's K slice. Every lane issues ALL of its 128-bit
//     weight loads (ld.global.nc.L1::no_allocate) before touching x, so each
//     CTA has its whole slice (8-32 KB) in flight while x is staged.
//   * x (gathered through colmap: structured / irregular / online-reorder are
//     the same kernel) is staged once per CTA into padded shared memory, plus
//     fp32 group sums for the zero-point fold.
//   * codes become mma A fragments straight from the 128-bit load: one LOP3 per
//     fragment yields (magic + code) halves; mma.sync m16n8k16 accumulates
//     sum (magic + c) * x in fp32 and the group fold removes the magic:
//       y += s' * acc + (z - magic * s') * sum(x)          (s' = s, or s/16 for
//     the fp16 hi-nibble trick), so per code the kernel spends ~0.7 issue slots.
//   * the fp16 weak block rides the same warp loop as plain mma tiles.
//   * K slices are combined deterministically: partials go to a workspace and
//     the last CTA of a row group (atomic ticket) sums them in slice order.
#include "qeft_common.cuh"
#include "qeft_internal.h"

using namespace qeft;

namespace {

constexpr int kWarps = 4;
constexpr int kMaxKS = 1024;           // max K slice (codes)
constexpr int kMaxT4 = kMaxKS / 64;    // 4-bit tiles per warp per slice
constexpr int kMaxT3 = kMaxKS / 128;   // 3-bit tiles
constexpr int kMaxWeakT = 4;           // k_pad <= 256
constexpr int kMaxGrp = kMaxKS / 64;   // groups per slice (g >= 64 in FOLD mode)

struct GemvArgs {
  const uint8_t* qw;
  const void* sz;
  const void* weak16;
  const int* colmap;
  const void* x;
  int64_t ldx;
  void* y;
  int64_t ldy;
  int y_f32;
  int oc, ic, m, m_pad, k, k_pad, g, ng, n;
  int ks, s_quant, s_total, fast_x, xs_stride;
  float* ws;
  int* counters;
};

template <typename T>
__device__ __forceinline__ void store_out(const GemvArgs& a, int n, int row, float v) {
  if (a.y_f32)
    ((float*)a.y)[(int64_t)n * a.ldy + row] = v;
  else
    ((T*)a.y)[(int64_t)n * a.ldy + row] = from_f32<T>(v);
}

// BITS: 3/4 (quant slices); FOLD: g % 64 == 0 (group fold) else per-element dequant.
template <int BITS, int NT, typename T, bool FOLD>
__global__ void __launch_bounds__(kWarps * 32)
gemv_kernel(const GemvArgs a) {
  using T2 = typename DTraits<T>::T2;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ float xsum_s[kMaxGrp][16];
  __shared__ int last_flag;

  const int s = blockIdx.x, rg = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int rb = rg * kWarps + warp;
  const bool rb_ok = rb * 16 < a.oc;
  const bool weak = s == a.s_quant;
  const int j0 = weak ? a.m_pad : s * a.ks;
  const int jlen = weak ? a.k_pad : min(a.ks, a.m_pad - j0);
  const int xs_stride = a.xs_stride;  // halves; stride bytes == 16 mod 32 -> conflict-free LDS.128
  T* xs = reinterpret_cast<T*>(smem);

  // ---- 1. put the whole weight slice of this warp in flight ----
  uint4 wq[(BITS == 4) ? kMaxT4 : kMaxT3];
  uint2 wh[(BITS == 3) ? kMaxT3 : 1];
  uint4 ww[kMaxWeakT][4];
  int ntile;
  if (!weak) {
    if constexpr (BITS == 4) {
      ntile = jlen >> 6;
      const uint8_t* base = a.qw + ((int64_t)rb * (a.m_pad >> 6) + (j0 >> 6)) * 512 + lane * 16;
#pragma unroll
      for (int i = 0; i < kMaxT4; ++i)
        if (i < ntile && rb_ok) wq[i] = ldg_stream(base + i * 512);
    } else {
      ntile = jlen >> 7;
      const uint8_t* base = a.qw + ((int64_t)rb * (a.m_pad >> 7) + (j0 >> 7)) * 768;
#pragma unroll
      for (int i = 0; i < kMaxT3; ++i)
        if (i < ntile && rb_ok) {
          wq[i] = ldg_stream(base + i * 768 + lane * 16);
          wh[i] = ldg_stream64(base + i * 768 + 512 + lane * 8);
        }
    }
  } else {
    ntile = jlen >> 6;
    const T* w0 = (const T*)a.weak16 + (int64_t)(rb * 16 + g8) * a.k_pad + 16 * t4;
    const T* w1 = w0 + 8 * (int64_t)a.k_pad;
#pragma unroll
    for (int i = 0; i < kMaxWeakT; ++i)
      if (i < ntile && rb_ok) {
        ww[i][0] = ldg_stream(w0 + 64 * i);
        ww[i][1] = ldg_stream(w0 + 64 * i + 8);
        ww[i][2] = ldg_stream(w1 + 64 * i);
        ww[i][3] = ldg_stream(w1 + 64 * i + 8);
      }
  }

  // ---- 2. stage x[n][j0 .. j0+jlen) (B200 K order) into shared memory ----
  const T* x = (const T*)a.x;
  if (a.fast_x) {
    const int nch = jlen >> 3;
    for (int e = threadIdx.x; e < a.n * nch; e += blockDim.x) {
      const int n = e / nch, c = e % nch;
      const int j = j0 + 8 * c;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (!weak) {
        if (j < a.m) v = *reinterpret_cast<const uint4*>(x + (int64_t)n * a.ldx + j);
      } else if (j - a.m_pad < a.k) {
        v = *reinterpret_cast<const uint4*>(x + (int64_t)n * a.ldx + a.m + (j - a.m_pad));
      }
      *reinterpret_cast<uint4*>(xs + n * xs_stride + 8 * c) = v;
    }
  } else {
    for (int e = threadIdx.x; e < a.n * jlen; e += blockDim.x) {
      const int n = e / jlen, jj = e % jlen;
      const int col = a.colmap[j0 + jj];
      xs[n * xs_stride + jj] = col >= 0 ? x[(int64_t)n * a.ldx + col] : from_f32<T>(0.f);
    }
  }
  __syncthreads();

  // group sums for the zero-point fold
  int ga = 0;
  if constexpr (FOLD) {
    if (!weak) {
      ga = j0 / a.g;
      const int gb = (j0 + jlen - 1) / a.g;
      const int npair = (gb - ga + 1) * a.n;
      for (int p = warp; p < npair; p += kWarps) {
        const int gl = p / a.n, n = p % a.n;
        const int lo = max((ga + gl) * a.g, j0) - j0, hi = min((ga + gl + 1) * a.g, j0 + jlen) - j0;
        float acc = 0.f;
        for (int jj = lo + lane; jj < hi; jj += 32) acc += to_f32<T>(xs[n * xs_stride + jj]);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) xsum_s[gl][n] = acc;
      }
      __syncthreads();
    }
  }

  // ---- 3. tensor-core dot products ----
  float acc[NT][4];
  float accg[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = accg[nt][e] = 0.f;

  const T* xrow[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xrow[nt] = xs + min(g8 + 8 * nt, a.n - 1) * xs_stride + 16 * t4;

  auto fold = [&](int grp) {
    const T2* sz = (const T2*)a.sz + ((int64_t)rb * a.ng + grp) * 16;
    const float2 p0 = t2_to_f2<T2>(sz[g8]);
    const float2 p1 = t2_to_f2<T2>(sz[g8 + 8]);
    constexpr float M = DTraits<T>::kMagicF;
    const float s0 = p0.x;
    const float s1 = (BITS == 4 && DTraits<T>::kHiTrick) ? p1.x * (1.f / 16.f) : p1.x;
    const float z0 = p0.y - M * s0, z1 = p1.y - M * s1;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c0 = 8 * nt + 2 * t4;
      const float xa = c0 < a.n ? xsum_s[grp - ga][c0] : 0.f;
      const float xb = c0 + 1 < a.n ? xsum_s[grp - ga][c0 + 1] : 0.f;
      acc[nt][0] += s0 * accg[nt][0] + z0 * xa;
      acc[nt][1] += s0 * accg[nt][1] + z0 * xb;
      acc[nt][2] += s1 * accg[nt][2] + z1 * xa;
      acc[nt][3] += s1 * accg[nt][3] + z1 * xb;
#pragma unroll
      for (int e = 0; e < 4; ++e) accg[nt][e] = 0.f;
    }
  };

  // per-element dequant for group sizes that are not a multiple of 64
  auto dq_frag = [&](uint32_t mag, bool hi16, int row_local, int col) -> uint32_t {
    T2 c = magic_to_code<T>(mag, hi16);
    const float2 cf = t2_to_f2<T2>(c);
    const int g0 = min(col / a.g, a.ng - 1), g1 = min((col + 1) / a.g, a.ng - 1);
    const T2* sz = (const T2*)a.sz + (int64_t)rb * a.ng * 16;
    const float2 p0 = t2_to_f2<T2>(sz[g0 * 16 + row_local]);
    const float2 p1 = t2_to_f2<T2>(sz[g1 * 16 + row_local]);
    T lo = from_f32<T>(cf.x * p0.x + p0.y), hi = from_f32<T>(cf.y * p1.x + p1.y);
    T2 r;
    r.x = lo;
    r.y = hi;
    return *reinterpret_cast<uint32_t*>(&r);
  };

  if (rb_ok) {
    if (!weak) {
      int cur = FOLD ? (j0 / a.g) : 0;
      if constexpr (BITS == 4) {
#pragma unroll
        for (int i = 0; i < kMaxT4; ++i) {
          if (i < ntile) {
            if constexpr (FOLD) {
              const int grp = (j0 + 64 * i) / a.g;
              if (grp != cur) { fold(cur); cur = grp; }
            }
            const uint32_t q[4] = {wq[i].x, wq[i].y, wq[i].z, wq[i].w};
            uint4 xa[NT], xb[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              xa[nt] = *reinterpret_cast<const uint4*>(xrow[nt] + 64 * i);
              xb[nt] = *reinterpret_cast<const uint4*>(xrow[nt] + 64 * i + 8);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t f[4];
              decode4<T>(q[j], f);
              if constexpr (!FOLD) {
                const int c = j0 + 64 * i + 16 * t4 + 4 * j;
                const bool h16 = DTraits<T>::kHiTrick;
                f[0] = dq_frag(f[0], false, g8, c);
                f[1] = dq_frag(f[1], h16, g8 + 8, c);
                f[2] = dq_frag(f[2], false, g8, c + 2);
                f[3] = dq_frag(f[3], h16, g8 + 8, c + 2);
              }
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                const uint32_t b0 = (j == 0) ? xa[nt].x : (j == 1) ? xa[nt].z : (j == 2) ? xb[nt].x : xb[nt].z;
                const uint32_t b1 = (j == 0) ? xa[nt].y : (j == 1) ? xa[nt].w : (j == 2) ? xb[nt].y : xb[nt].w;
                mma16816<T>(FOLD ? accg[nt] : acc[nt], f, b0, b1);
              }
            }
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < kMaxT3; ++i) {
          if (i < ntile) {
            const uint32_t w2[4] = {wq[i].x, wq[i].y, wq[i].z, wq[i].w};
            const uint32_t hb[2] = {wh[i].x, wh[i].y};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if constexpr (FOLD) {
                const int grp = (j0 + 128 * i + 64 * h) / a.g;
                if (grp != cur) { fold(cur); cur = grp; }
              }
              uint4 xa[NT], xb[NT];
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                xa[nt] = *reinterpret_cast<const uint4*>(xrow[nt] + 128 * i + 64 * h);
                xb[nt] = *reinterpret_cast<const uint4*>(xrow[nt] + 128 * i + 64 * h + 8);
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int wwi = j >> 1;
                uint32_t f[4];
#pragma unroll
                for (int pp = 0; pp < 4; ++pp)
                  f[pp] = decode3_pair<T>(w2[2 * h + wwi], hb[h], 4 * (j & 1) + pp, wwi);
                if constexpr (!FOLD) {
                  const int c = j0 + 128 * i + 64 * h + 16 * t4 + 4 * j;
                  f[0] = dq_frag(f[0], false, g8, c);
                  f[1] = dq_frag(f[1], false, g8 + 8, c);
                  f[2] = dq_frag(f[2], false, g8, c + 2);
                  f[3] = dq_frag(f[3], false, g8 + 8, c + 2);
                }
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                  const uint32_t b0 = (j == 0) ? xa[nt].x : (j == 1) ? xa[nt].z : (j == 2) ? xb[nt].x : xb[nt].z;
                  const uint32_t b1 = (j == 0) ? xa[nt].y : (j == 1) ? xa[nt].w : (j == 2) ? xb[nt].y : xb[nt].w;
                  mma16816<T>(FOLD ? accg[nt] : acc[nt], f, b0, b1);
                }
              }
            }
          }
        }
      }
      if constexpr (FOLD) fold(cur);
    } else {
#pragma unroll
      for (int i = 0; i < kMaxWeakT; ++i) {
        if (i < ntile) {
          uint4 xa[NT], xb[NT];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            xa[nt] = *reinterpret_cast<const uint4*>(xrow[nt] + 64 * i);
            xb[nt] = *reinterpret_cast<const uint4*>(xrow[nt] + 64 * i + 8);
          }
          const uint32_t r0[8] = {ww[i][0].x, ww[i][0].y, ww[i][0].z, ww[i][0].w,
                                  ww[i][1].x, ww[i][1].y, ww[i][1].z, ww[i][1].w};
          const uint32_t r1[8] = {ww[i][2].x, ww[i][2].y, ww[i][2].z, ww[i][2].w,
                                  ww[i][3].x, ww[i][3].y, ww[i][3].z, ww[i][3].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t f[4] = {r0[2 * j], r1[2 * j], r0[2 * j + 1], r1[2 * j + 1]};
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const uint32_t b0 = (j == 0) ? xa[nt].x : (j == 1) ? xa[nt].z : (j == 2) ? xb[nt].x : xb[nt].z;
              const uint32_t b1 = (j == 0) ? xa[nt].y : (j == 1) ? xa[nt].w : (j == 2) ? xb[nt].y : xb[nt].w;
              mma16816<T>(acc[nt], f, b0, b1);
            }
          }
        }
      }
    }
  }

  // ---- 4. output: direct, or deterministic split-K combine ----
  const int row0 = rb * 16 + g8, row1 = row0 + 8;
  if (a.s_total == 1) {
    if (rb_ok) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c0 = 8 * nt + 2 * t4;
        if (c0 < a.n) {
          if (row0 < a.oc) store_out<T>(a, c0, row0, acc[nt][0]);
          if (row1 < a.oc) store_out<T>(a, c0, row1, acc[nt][2]);
        }
        if (c0 + 1 < a.n) {
          if (row0 < a.oc) store_out<T>(a, c0 + 1, row0, acc[nt][1]);
          if (row1 < a.oc) store_out<T>(a, c0 + 1, row1, acc[nt][3]);
        }
      }
    }
    return;
  }
  float* part = a.ws + ((int64_t)rg * a.s_total + s) * (16 * 64);
  const int rl0 = warp * 16 + g8, rl1 = rl0 + 8;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c0 = 8 * nt + 2 * t4;
    if (c0 < a.n) { part[c0 * 64 + rl0] = acc[nt][0]; part[c0 * 64 + rl1] = acc[nt][2]; }
    if (c0 + 1 < a.n) { part[(c0 + 1) * 64 + rl0] = acc[nt][1]; part[(c0 + 1) * 64 + rl1] = acc[nt][3]; }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last_flag = (atomicAdd(a.counters + rg, 1) == a.s_total - 1);
  __syncthreads();
  if (!last_flag) return;
  __threadfence();
  const float* pbase = a.ws + (int64_t)rg * a.s_total * (16 * 64);
  for (int e = threadIdx.x; e < a.n * 64; e += blockDim.x) {
    const int c = e >> 6, rl = e & 63;
    const int row = rg * 64 + rl;
    float v = 0.f;
    for (int ss = 0; ss < a.s_total; ++ss) v += __ldcg(pbase + ss * (16 * 64) + c * 64 + rl);
    if (row < a.oc) store_out<T>(a, c, row, v);
  }
  if (threadIdx.x == 0) a.counters[rg] = 0;
}

struct Plan {
  int ks, s_quant, s_total, n_rg;
};

Plan make_plan(const qeft_linear_t* L) {
  Plan p;
  p.n_rg = (L->oc_pad + 63) / 64;
  p.ks = kMaxKS;
  // shrink the slice until the grid covers the chip twice
  while (p.ks > 128 && (int64_t)p.n_rg * ((L->m_pad + p.ks - 1) / p.ks) < 2 * 148) p.ks >>= 1;
  p.s_quant = L->m_pad ? (L->m_pad + p.ks - 1) / p.ks : 0;
  p.s_total = p.s_quant + (L->k_pad ? 1 : 0);
  return p;
}

template <int BITS, int NT, typename T, bool FOLD>
int launch(const GemvArgs& a, int n_rg, cudaStream_t st) {
  const size_t smem = (size_t)a.n * a.xs_stride * sizeof(T);
  auto kern = gemv_kernel<BITS, NT, T, FOLD>;
  if (smem > 48 * 1024) QEFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<dim3(a.s_total, n_rg), kWarps * 32, smem, st>>>(a);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

template <typename T>
int dispatch(const GemvArgs& a, int bits, int n_rg, bool fold, cudaStream_t st) {
  const bool nt2 = a.n > 8;
#define QEFT_GEMV_CASE(B, NT, F) \
  if (bits == B && (NT == 2) == nt2 && fold == F) return launch<B, NT, T, F>(a, n_rg, st);
  QEFT_GEMV_CASE(4, 1, true) QEFT_GEMV_CASE(4, 2, true) QEFT_GEMV_CASE(4, 1, false)
  QEFT_GEMV_CASE(4, 2, false) QEFT_GEMV_CASE(3, 1, true) QEFT_GEMV_CASE(3, 2, true)
  QEFT_GEMV_CASE(3, 1, false) QEFT_GEMV_CASE(3, 2, false)
#undef QEFT_GEMV_CASE
  set_error("gemv: unsupported bits=%d", bits);
  return QEFT_ERR_LAYOUT;
}

}  // namespace

namespace qeft {

size_t gemv_workspace_bytes(const qeft_linear_t* L, int n) {
  (void)n;
  const Plan p = make_plan(L);
  return (size_t)p.n_rg * p.s_total * 16 * 64 * sizeof(float) + (size_t)p.n_rg * sizeof(int) + 256;
}

int gemv(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int y_f32, int n,
         void* ws, size_t ws_bytes, cudaStream_t st) {
  QEFT_CHECK(n >= 1 && n <= 16, QEFT_ERR_SHAPE, "gemv: n_cols=%d outside 1..16", n);
  QEFT_CHECK(L->bits == 3 || L->bits == 4, QEFT_ERR_SHAPE, "gemv: bits=%d", L->bits);
  QEFT_CHECK(L->k_pad <= 64 * kMaxWeakT, QEFT_ERR_LAYOUT, "gemv: k_pad=%d > 256", L->k_pad);
  QEFT_CHECK(ldx >= L->ic && ldy >= L->oc, QEFT_ERR_SHAPE, "gemv: ld too small");
  const Plan p = make_plan(L);
  if (p.s_total == 0) return 0;
  QEFT_CHECK(p.s_total == 1 || ws_bytes >= gemv_workspace_bytes(L, n), QEFT_ERR_SHAPE,
             "gemv: workspace %zu < %zu bytes", ws_bytes, gemv_workspace_bytes(L, n));
  GemvArgs a;
  a.qw = (const uint8_t*)L->qweight;
  a.sz = L->sz;
  a.weak16 = L->weak16;
  a.colmap = L->colmap;
  a.x = x;
  a.ldx = ldx;
  a.y = y;
  a.ldy = ldy;
  a.y_f32 = y_f32;
  a.oc = L->oc; a.ic = L->ic; a.m = L->m; a.m_pad = L->m_pad; a.k = L->k; a.k_pad = L->k_pad;
  a.g = L->g; a.ng = L->ng; a.n = n;
  a.ks = p.ks; a.s_quant = p.s_quant; a.s_total = p.s_total;
  a.xs_stride = (p.ks > L->k_pad ? p.ks : L->k_pad) + 8;
  a.fast_x = (L->flags & QEFT_FLAG_STRUCTURED_FAST) && (ldx % 8 == 0) &&
             (((uintptr_t)x & 15) == 0);
  a.ws = (float*)ws;
  a.counters = (int*)((char*)ws + (size_t)p.n_rg * p.s_total * 16 * 64 * sizeof(float));
  const bool fold = (L->g % 64) == 0;
  if (L->act_dtype == QEFT_F16) return dispatch<__half>(a, L->bits, p.n_rg, fold, st);
  return dispatch<__nv_bfloat16>(a, L->bits, p.n_rg, fold, st);
}

}  // namespace qeft
