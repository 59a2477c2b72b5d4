// Decode GEMV for the QEFT mixed-precision layer, N = 1..16 activation columns.
//
// Replaces the reference's matvec paths (pkg/src/qeft/kernels.py:66-157,
// `_grouped_accumulate`): y = sum_g s_g * (c_g . x_g) + z_g * sum(x_g) + W_weak . x_weak.
//
// HBM-bound design for B200 (one pass over the packed weights, nothing else):
//   * The tile layout (qeft_common.cuh) hands every lane exactly the 16 bytes of
//     a 16 x 64 tile that form its mma.m16n8k16 A fragments, so codes go
//     straight from HBM into registers with coalesced 128-bit streaming loads
//     (ld.global.nc.L1::no_allocate) -- no shared-memory staging. Measured on
//     B200 (scripts/micro/stream_bench.cu): register streaming with >= 16
//     warps/SM reaches 6.5-7 TB/s, while cp.async.bulk saturates at ~4 copies
//     in flight per CTA (2-4 KB copies: 1.2-2.3 TB/s).
//   * CTA = 8 warps on one row-block (16 output rows); the warps split the K
//     range in whole groups, so every CTA owns complete output rows and the
//     K-partials are summed in a fixed order through shared memory: no
//     cross-CTA reduction, deterministic results.
//   * Each warp software-pipelines its K range in batches of kU 64-column
//     steps with incremental pointers and no bounds checks in the steady state:
//     the next batch's codes and (scale, zero) pairs are in flight while the
//     current batch is decoded and multiplied. The first batch is issued BEFORE
//     the programmatic-dependent-launch wait, so a layer's weight stream
//     overlaps the previous kernel; only x (staged once into shared memory in
//     the B200 K order, zero padded) and the trainable weak block wait for it.
//   * Codes become (magic + code) half2 A fragments with one LOP3 each and the
//     per-group fold is
//       y += s' * acc + (z - magic * s') * sum(x)   (s' = s, or s/16 for the
//     fp16 hi-nibble trick). For N <= 8 the group sums of x are formed while x is
//     staged (segmented warp shuffles) and read from shared memory; for N > 8 an
//     all-ones MMA per step accumulates them in the accumulator layout. GT (64-column steps
//     per group) is a template constant; GT = 0 is the generic per-element
//     dequant path for group sizes that are not 64 * {1, 2, 4}.
#include <algorithm>
#include <cstdlib>

#include "qeft_common.cuh"
#include "qeft_internal.h"

using namespace qeft;

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kU = 4;                 // 64-column steps per pipelined batch
constexpr int kR = 4;                 // per-warp cp.async ring depth (batches); 3 when a batched x
                                      // (N > 1) would otherwise cost the second CTA per SM
constexpr int kXSmemMax = 32 * 1024;  // stage x in smem up to this size, else read via L1

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

constexpr int kMaxLayers = 3;  // layers sharing x in one launch (q/k/v, gate/up)

struct GemvArgs {
  // per layer (rows concatenated in launch order): codes, group params, weak tiles, output
  const uint8_t* qw[kMaxLayers];
  const float2* sz[kMaxLayers];
  const uint8_t* weak16[kMaxLayers];
  void* ys[kMaxLayers];
  int ocs[kMaxLayers];
  int rb_end[kMaxLayers];  // cumulative row-block counts
  int nl;
  const uint8_t* x;  // fast: original columns; else pre-gathered B200 order [n][m_pad + k_pad]
  int64_t ldx;       // elements
  int64_t ldy;
  int y_f32;  // bit 0: fp32 output; bit 1: accumulate (y += W x, e.g. a residual stream)
  int m, m_pad, k, k_pad, g, ng, n, n_rb;
  int gathered;
  int nsq;      // quantized 64-column steps (m_pad / 64)
  int spw;      // quantized steps per warp (multiple of the group's steps)
  int xs_ld;    // smem x row stride (elements), 0 = x read through L1
  int64_t rbb;  // qweight bytes per row-block
  int dbg;      // tuning only: 1 = skip the weight stream (compute-only timing)
};

template <typename T>
__device__ __forceinline__ void store_out(const GemvArgs& a, void* y, int n, int row, float v) {
  const int64_t i = (int64_t)n * a.ldy + row;
  if (a.y_f32 & 1) {
    float* p = (float*)y + i;
    *p = (a.y_f32 & 2) ? *p + v : v;
  } else {
    T* p = (T*)y + i;
    *p = from_f32<T>((a.y_f32 & 2) ? to_f32<T>(*p) + v : v);  // one rounding of y + Wx
  }
}

// global row-block -> (layer, layer-local row-block)
QEFT_DEV int layer_of(const GemvArgs& a, int grb, int& rb) {
  int l = 0;
  while (l + 1 < a.nl && grb >= a.rb_end[l]) ++l;
  rb = grb - (l ? a.rb_end[l - 1] : 0);
  return l;
}

QEFT_DEV uint4 ldg_l1(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
QEFT_DEV float2 ldg_f2(const float2* p) {
  float2 r;
  asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];\n" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
QEFT_DEV uint32_t ldg_stream32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];\n" : "=r"(r) : "l"(p));
  return r;
}

// x element (n, j) of the B200 K order (quantized [0, m_pad), weak [m_pad, m_pad + k_pad)),
// 8 consecutive columns starting at j (j % 8 == 0); zero for padding
template <typename T>
QEFT_DEV uint4 x_chunk(const GemvArgs& a, int n, int j) {
  if (a.gathered) return ldg_l1(reinterpret_cast<const T*>(a.x) + (int64_t)n * a.ldx + j);
  int col;
  if (j < a.m_pad) {
    if (j >= a.m) return make_uint4(0, 0, 0, 0);
    col = j;
  } else {
    const int w = j - a.m_pad;
    if (w >= a.k) return make_uint4(0, 0, 0, 0);
    col = a.m + w;
  }
  return ldg_l1(reinterpret_cast<const T*>(a.x) + (int64_t)n * a.ldx + col);
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

__host__ __device__ inline size_t xsum_bytes(int ng, int nt) {
  return ((size_t)ng * nt * 8 * sizeof(float) + 127) & ~(size_t)127;
}

template <int GT>
struct Ring {
  static constexpr int G = GT > 0 ? GT : 1;
  static constexpr int kSP = kU / G;                   // group-param slots per batch
  static constexpr int kSlot = kU * 512 + kSP * 128;   // bytes per warp per batch
};

template <int BITS, int NT, int GT, typename T, bool XS, int R = kR>
__global__ void __launch_bounds__(kThreads, (NT == 1 || !XS) ? 2 : 1)  // NT = 2, x resident: 1 CTA/SM anyway
gemv_kernel(const GemvArgs a) {
  // dynamic smem: [x (XS only): n x xs_ld][weak tiles: 2 x wbytes][rings: kWarps x kR x kSlot]
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float part[2][kWarps][16][NT * 8];
  __shared__ __align__(8) uint64_t wbar[2];
  constexpr bool FOLD = GT > 0;
  constexpr int G = Ring<GT>::G, kSP = Ring<GT>::kSP, kSlot = Ring<GT>::kSlot;
  // sum(x) per group: from the x staging for one n-tile (N <= 8), else an all-ones MMA per step
  constexpr bool kXsum = FOLD && NT == 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int s_beg = min(warp * a.spw, a.nsq), s_end = min(s_beg + a.spw, a.nsq);
  const int nsteps = s_end - s_beg;
  const int nb = (nsteps + kU - 1) / kU;  // batches per row-block (last may be partial)
  // persistent: this CTA's row-blocks are blockIdx.x + j * gridDim.x
  const int nrbc = (a.n_rb - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int nwt = a.k_pad >> 6;
  const uint32_t wbytes = (uint32_t)nwt * 2048u;
  // per-(group, column) sums of x: the zero-point term of the fold, shared by every row
  float* xsum = reinterpret_cast<float*>(smem + (XS ? (size_t)a.n * a.xs_ld * sizeof(T) : 0));
  uint8_t* wsm = reinterpret_cast<uint8_t*>(xsum) + xsum_bytes(a.ng, NT);
  uint8_t* ring = wsm + 2 * wbytes + (size_t)warp * R * kSlot;

  auto rb_of = [&](int j) { return (int)blockIdx.x + j * (int)gridDim.x; };

  float acc[NT][4], accg[NT][4], accx[NT][4];
  auto zero_acc = [&]() {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = accg[nt][e] = accx[nt][e] = 0.f;
  };
  zero_acc();
  int xrow[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xrow[nt] = min(g8 + 8 * nt, a.n - 1);
  const uint32_t ones[4] = {DTraits<T>::kOne2, DTraits<T>::kOne2, DTraits<T>::kOne2, DTraits<T>::kOne2};

  auto bsel = [](const uint4& xa, const uint4& xb, int j, uint32_t& b0, uint32_t& b1) {
    b0 = (j == 0) ? xa.x : (j == 1) ? xa.z : (j == 2) ? xb.x : xb.z;
    b1 = (j == 0) ? xa.y : (j == 1) ? xa.w : (j == 2) ? xb.y : xb.w;
  };
  // B fragments of the 64-column step starting at B200 K position j
  auto x_frag = [&](int j, uint4 xa[NT], uint4 xb[NT]) {
    const int c0 = j + 16 * t4;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      if constexpr (XS) {
        const T* xp = reinterpret_cast<const T*>(smem) + xrow[nt] * a.xs_ld + c0;
        xa[nt] = *reinterpret_cast<const uint4*>(xp);
        xb[nt] = *reinterpret_cast<const uint4*>(xp + 8);
      } else {
        xa[nt] = x_chunk<T>(a, xrow[nt], c0);
        xb[nt] = x_chunk<T>(a, xrow[nt], c0 + 8);
      }
    }
  };
  // per-element dequant for group sizes that are not 64 * {1, 2, 4}
  auto dq_frag = [&](int rb, uint32_t mag, bool hi16, int row_local, int col) -> uint32_t {
    using T2 = typename DTraits<T>::T2;
    const float2 cf = t2_to_f2<T2>(magic_to_code<T>(mag, hi16));
    const int gA = min(col / a.g, a.ng - 1), gB = min((col + 1) / a.g, a.ng - 1);
    int lrb;
    const int l = layer_of(a, rb, lrb);
    const float2* sz = a.sz[l] + (int64_t)lrb * a.ng * 16;
    const float2 pA = sz[gA * 16 + row_local];
    const float2 pB = sz[gB * 16 + row_local];
    T2 r;
    r.x = from_f32<T>(cf.x * pA.x + pA.y);
    r.y = from_f32<T>(cf.y * pB.x + pB.y);
    return *reinterpret_cast<uint32_t*>(&r);
  };

  // fold group `grp`: acc += s' * g + (z - magic * s') * sum(x of the group)
  // fold group `grp`: acc += s' * g + (z - magic * s') * sum(x); the sums come from the
  // staging table (kXsum) or from the all-ones MMA accumulators `xs`
  auto fold = [&](const float2* szs, int grp, const float (&g)[NT][4], const float (&xs)[NT][4]) {
    constexpr float M = DTraits<T>::kMagicF;
    const float2 p0 = szs[g8], p1 = szs[g8 + 8];
    const float s0 = p0.x;
    const float s1 = (BITS == 4 && DTraits<T>::kHiTrick) ? p1.x * (1.f / 16.f) : p1.x;
    const float z0 = p0.y - M * s0, z1 = p1.y - M * s1;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float2 sx0, sx1;
      if constexpr (kXsum) {
        sx0 = sx1 = *reinterpret_cast<const float2*>(xsum + grp * (NT * 8) + 8 * nt + 2 * t4);
      } else {
        sx0 = make_float2(xs[nt][0], xs[nt][1]);
        sx1 = make_float2(xs[nt][2], xs[nt][3]);
      }
      acc[nt][0] += s0 * g[nt][0] + z0 * sx0.x;
      acc[nt][1] += s0 * g[nt][1] + z0 * sx0.y;
      acc[nt][2] += s1 * g[nt][2] + z1 * sx1.x;
      acc[nt][3] += s1 * g[nt][3] + z1 * sx1.y;
    }
  };

  // one 64-column step: decode + MMA (+ fold with params p0/p1 when `fold_now`)
  auto step = [&](int rb, int st, const uint4& q, const float2* szs, bool fold_now) {
    const int col = st * 64;
    uint4 xa[NT], xb[NT];
    x_frag(col, xa, xb);
    if constexpr (FOLD && !kXsum) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          uint32_t b0_, b1_;
          bsel(xa[nt], xb[nt], j, b0_, b1_);
          mma16816<T>(accx[nt], ones, b0_, b1_);
        }
    }
    uint32_t f[4][4];
    if constexpr (BITS == 4) {
      const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) decode4<T>(qq[j], f[j]);
    } else {
      const uint32_t ww2[2] = {q.x, q.y};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) f[j][pp] = decode3_pair<T>(ww2[j >> 1], q.z, 4 * (j & 1) + pp, j >> 1);
    }
    if constexpr (!FOLD) {
      constexpr bool h16 = (BITS == 4) && DTraits<T>::kHiTrick;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cc = col + 16 * t4 + 4 * j;
        f[j][0] = dq_frag(rb, f[j][0], false, g8, cc);
        f[j][1] = dq_frag(rb, f[j][1], h16, g8 + 8, cc);
        f[j][2] = dq_frag(rb, f[j][2], false, g8, cc + 2);
        f[j][3] = dq_frag(rb, f[j][3], h16, g8 + 8, cc + 2);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t b0_, b1_;
        bsel(xa[nt], xb[nt], j, b0_, b1_);
        mma16816<T>(FOLD ? accg[nt] : acc[nt], f[j], b0_, b1_);
      }
    if constexpr (FOLD) {
      // steps past the last group (g = 64 with an odd group count) carry only padding
      if (fold_now && st / G < a.ng) {
        fold(szs, st / G, accg, accx);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) accg[nt][e] = accx[nt][e] = 0.f;
      }
    }
  };

  // ---- the warp's batch stream through its private cp.async ring ----
  // batch (row-block j, batch b) = kU 64-column steps; every step of a group slot
  // shares its group (batches start at group boundaries)
  const int TB = nb * nrbc;
  int ij = 0, ib = 0;
  auto issue_next = [&](int t) {
    if (t < TB && !a.dbg) {
      uint8_t* slot = ring + (t % R) * kSlot;
      int rb;
      const int l = layer_of(a, rb_of(ij), rb);
      const int b0 = s_beg + ib * kU;
      const uint8_t* base = a.qw[l] + rb * a.rbb;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int st = b0 + u;
        if (st < s_end) {
          if constexpr (BITS == 4) {
            cp_async16(slot + u * 512 + lane * 16, base + (int64_t)st * 512 + lane * 16);
          } else {
            const uint8_t* tb = base + (int64_t)(st >> 1) * 768;
            const int h = st & 1;
            cp_async8(slot + u * 512 + lane * 16, tb + lane * 16 + 8 * h);
            cp_async4(slot + u * 512 + lane * 16 + 8, tb + 512 + lane * 8 + 4 * h);
          }
        }
      }
      if (FOLD && lane < 16) {
        const float2* szp = a.sz[l] + ((int64_t)rb * a.ng) * 16 + lane;
#pragma unroll
        for (int i = 0; i < kSP; ++i) {
          if (b0 + i * G < s_end) {
            const int grp = min(b0 / G + i, a.ng - 1);
            cp_async8(slot + kU * 512 + i * 128 + lane * 8, szp + grp * 16);
          }
        }
      }
      if (++ib == nb) { ib = 0; ++ij; }
    }
    cp_async_commit();  // one group per batch (possibly empty) keeps the wait count uniform
  };
  // decode the step's codes into mma A fragments ((magic + code) halves, or dequantized
  // values on the generic path)
  auto decode = [&](int rb, int st, const uint4& q, uint32_t (&f)[4][4]) {
    if constexpr (BITS == 4) {
      const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) decode4<T>(qq[j], f[j]);
    } else {
      const uint32_t ww2[2] = {q.x, q.y};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) f[j][pp] = decode3_pair<T>(ww2[j >> 1], q.z, 4 * (j & 1) + pp, j >> 1);
    }
    if constexpr (!FOLD) {
      constexpr bool h16 = (BITS == 4) && DTraits<T>::kHiTrick;
      const int col = st * 64;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cc = col + 16 * t4 + 4 * j;
        f[j][0] = dq_frag(rb, f[j][0], false, g8, cc);
        f[j][1] = dq_frag(rb, f[j][1], h16, g8 + 8, cc);
        f[j][2] = dq_frag(rb, f[j][2], false, g8, cc + 2);
        f[j][3] = dq_frag(rb, f[j][3], h16, g8 + 8, cc + 2);
      }
    }
  };
  auto compute = [&](int t, int j, int b) {
    const uint8_t* slot = ring + (t % R) * kSlot;
    const int rb = rb_of(j);
    const int b0 = s_beg + b * kU;
    if (b0 + kU <= s_end) {
      // full batch: every step gets its own accumulators, so the kU steps' MMA chains
      // are independent
      float ag[kU][NT][4], ax[kU][NT][4];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int st = b0 + u;
        const uint4 q = *reinterpret_cast<const uint4*>(slot + u * 512 + lane * 16);
        uint4 xa[NT], xb[NT];
        x_frag(st * 64, xa, xb);
        uint32_t f[4][4];
        decode(rb, st, q, f);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) ag[u][nt][e] = ax[u][nt][e] = 0.f;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            uint32_t b0_, b1_;
            bsel(xa[nt], xb[nt], jj, b0_, b1_);
            if constexpr (FOLD && !kXsum) mma16816<T>(ax[u][nt], ones, b0_, b1_);
            mma16816<T>(ag[u][nt], f[jj], b0_, b1_);
          }
      }
#pragma unroll
      for (int i = 0; i < kSP; ++i) {
        float g[NT][4], xs[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            g[nt][e] = ag[i * G][nt][e];
            xs[nt][e] = ax[i * G][nt][e];
#pragma unroll
            for (int u = 1; u < G; ++u) {
              g[nt][e] += ag[i * G + u][nt][e];
              if constexpr (!kXsum) xs[nt][e] += ax[i * G + u][nt][e];
            }
          }
        if constexpr (FOLD) {
          const int grp = (b0 + i * G) / G;
          if (grp < a.ng) fold(reinterpret_cast<const float2*>(slot + kU * 512 + i * 128), grp, g, xs);
        } else {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[nt][e] += g[nt][e];
        }
      }
      return;
    }
    // partial batch (end of a warp's range): one step at a time
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int st = b0 + u;
      if (st < s_end) {
        const uint4 q = *reinterpret_cast<const uint4*>(slot + u * 512 + lane * 16);
        const float2* szs = reinterpret_cast<const float2*>(slot + kU * 512 + (u / G) * 128);
        step(rb, st, q, szs, (u % G) == G - 1 || st + 1 == s_end);
      }
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    fence_mbar_init();
  }
#pragma unroll
  for (int t = 0; t < R - 1; ++t) issue_next(t);
  // Programmatic dependent launch: the next layer may start streaming its weights
  // now; x (the previous kernel's output) and the trainable weak block are read
  // after the wait.
  pdl_launch_dependents();
  pdl_wait();
  if (a.dbg == 2) return;  // tuning only: launch + PDL overhead
  __syncthreads();  // barrier init visible
  auto issue_weak = [&](int j) {
    if (nwt > 0 && j < nrbc) {
      mbar_expect_tx(&wbar[j & 1], wbytes);
      int rb;
      const int l = layer_of(a, rb_of(j), rb);
      bulk_g2s(wsm + (j & 1) * wbytes, a.weak16[l] + (int64_t)rb * wbytes, wbytes, &wbar[j & 1]);
    }
  };
  if (threadIdx.x == 0) {
    issue_weak(0);
    issue_weak(1);
  }
  if constexpr (kXsum) {
    // Stage x once per CTA (B200 K order, zero padded) and form the per-(group, column) sums
    // of x on the way: the quantized columns are walked in 8-column chunks (all n <= 8 columns'
    // loads in flight together); a group's 8 * G chunks are consecutive lanes of one warp, so a
    // segmented shuffle reduction gives its fp32 sum without another pass over x.
    constexpr int kCG = 8 * G;  // chunks per group (<= 32)
    const int qchunks = a.m_pad >> 3, row_chunks = (a.m_pad + a.k_pad) >> 3;
    using T2 = typename DTraits<T>::T2;
    for (int c0 = 0; c0 < row_chunks; c0 += kThreads) {
      const int c = c0 + (int)threadIdx.x;
      uint4 v[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        v[n] = make_uint4(0, 0, 0, 0);
        if (n < a.n && c < row_chunks) v[n] = x_chunk<T>(a, n, c << 3);
      }
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        if (n >= a.n) break;
        if (XS && c < row_chunks) *reinterpret_cast<uint4*>(reinterpret_cast<T*>(smem) + n * a.xs_ld + (c << 3)) = v[n];
        if (c0 < qchunks) {  // warp-uniform: qchunks is a multiple of 16, kThreads of 32
          const T2* h = reinterpret_cast<const T2*>(&v[n]);
          float sum = 0.f;
          if (c < qchunks) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f2 = t2_to_f2<T2>(h[q]);
              sum += f2.x + f2.y;
            }
          }
#pragma unroll
          for (int o = 1; o < kCG; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
          const int grp = c / kCG;
          if ((c % kCG) == 0 && c < qchunks && grp < a.ng) xsum[grp * (NT * 8) + n] = sum;
        }
      }
    }
    __syncthreads();
  } else if constexpr (XS) {
    const int row_chunks = (a.m_pad + a.k_pad) >> 3;
    for (int e = threadIdx.x; e < a.n * row_chunks; e += kThreads) {
      const int n = e / row_chunks, jj = (e - n * row_chunks) << 3;
      *reinterpret_cast<uint4*>(reinterpret_cast<T*>(smem) + n * a.xs_ld + jj) = x_chunk<T>(a, n, jj);
    }
    __syncthreads();
  }
  // weak tiles + fixed-order sum of the warps' K-partials for row-block j
  // (part is double-buffered: one barrier per row-block)
  auto finish = [&](int j) {
    const int rb = rb_of(j);
    if (warp < nwt) mbar_wait(&wbar[j & 1], (j >> 1) & 1);
    for (int wt = warp; wt < nwt; wt += kWarps) {
      const T* w16 = reinterpret_cast<const T*>(wsm + (j & 1) * wbytes) + wt * 1024;
      const uint4 r0a = *reinterpret_cast<const uint4*>(w16 + g8 * 64 + 16 * t4);
      const uint4 r0b = *reinterpret_cast<const uint4*>(w16 + g8 * 64 + 16 * t4 + 8);
      const uint4 r1a = *reinterpret_cast<const uint4*>(w16 + (g8 + 8) * 64 + 16 * t4);
      const uint4 r1b = *reinterpret_cast<const uint4*>(w16 + (g8 + 8) * 64 + 16 * t4 + 8);
      uint4 xa[NT], xb[NT];
      x_frag(a.m_pad + wt * 64, xa, xb);
      const uint32_t f[4][4] = {{r0a.x, r1a.x, r0a.y, r1a.y}, {r0a.z, r1a.z, r0a.w, r1a.w},
                                {r0b.x, r1b.x, r0b.y, r1b.y}, {r0b.z, r1b.z, r0b.w, r1b.w}};
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          uint32_t b0_, b1_;
          bsel(xa[nt], xb[nt], jj, b0_, b1_);
          mma16816<T>(acc[nt], f[jj], b0_, b1_);
        }
    }
    float (*pp)[16][NT * 8] = part[j & 1];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int cA = 8 * nt + 2 * t4;
      pp[warp][g8][cA] = acc[nt][0];
      pp[warp][g8][cA + 1] = acc[nt][1];
      pp[warp][g8 + 8][cA] = acc[nt][2];
      pp[warp][g8 + 8][cA + 1] = acc[nt][3];
    }
    zero_acc();
    __syncthreads();
    // every warp is past row-block j's weak tiles: refill that buffer for j + 2
    if (threadIdx.x == 0) issue_weak(j + 2);
    for (int e = threadIdx.x; e < 16 * a.n; e += kThreads) {
      const int rl = e & 15, n = e >> 4;
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += pp[w][rl][n];
      int lrb;
      const int l = layer_of(a, rb, lrb);
      const int row = lrb * 16 + rl;
      if (row < a.ocs[l]) store_out<T>(a, a.ys[l], n, row, v);
    }
  };

  if (nb == 0) {
    for (int j = 0; j < nrbc; ++j) finish(j);
    return;
  }
  int cj = 0, cb = 0;
  for (int t = 0; t < TB; ++t) {
    cp_async_wait<R - 2>();  // batch t has landed (this lane's copies)
    __syncwarp();             // ... and every lane's (group params are shared)
    compute(t, cj, cb);
    issue_next(t + R - 1);   // refills the slot consumed at t - 1
    if (++cb == nb) {
      finish(cj);
      cb = 0;
      ++cj;
    }
  }
}

template <int BITS, int NT, int GT, typename T, bool XS, int R>
int launch_kernel(const GemvArgs& a, size_t smem, int per_sm, cudaStream_t st) {
  auto kern = gemv_kernel<BITS, NT, GT, T, XS, R>;
  static size_t max_dyn = 0;
  if (!max_dyn) {  // all the dynamic smem the SM leaves next to this kernel's static smem
    cudaFuncAttributes fa{};
    QEFT_CUDA(cudaFuncGetAttributes(&fa, kern));
    max_dyn = std::min<size_t>(227 * 1024 - fa.sharedSizeBytes, (size_t)env_int("QEFT_GEMV_MAXDYN", 227 * 1024));
    QEFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn));
  }
  QEFT_CHECK(smem <= max_dyn, QEFT_ERR_LAYOUT, "gemv: %zu B of shared memory (k_pad=%d, n=%d) too large", smem,
             a.k_pad, a.n);
  // persistent CTAs, equal row-block counts per CTA
  const int slots = per_sm * num_sms();
  const int per = (a.n_rb + slots - 1) / slots;
  const int grid = (a.n_rb + per - 1) / per;
  QEFT_CUDA(launch_pdl(kern, dim3(grid), dim3(kThreads), smem, st, a));
  return 0;
}

template <int BITS, int NT, int GT, typename T>
int launch(const GemvArgs& a0, cudaStream_t st) {
  GemvArgs a = a0;
  const size_t xs_bytes = (size_t)a.n * (a.m_pad + a.k_pad + 8) * sizeof(T);
  const size_t w_bytes = (size_t)2 * (a.k_pad / 64) * 2048;
  const size_t fixed = xsum_bytes(a.ng, NT) + w_bytes;
  const size_t ring4 = (size_t)kWarps * kR * Ring<GT>::kSlot, ring3 = (size_t)kWarps * 3 * Ring<GT>::kSlot;
  static const size_t xs_max = (size_t)env_int("QEFT_GEMV_XSMAX", 200 * 1024);  // tuning
  constexpr size_t kStatic = 9 * 1024;  // per-CTA static smem + reserve (what every launch so far fit)
  auto fits2 = [&](size_t dyn) { return 2 * (dyn + kStatic) <= 227 * 1024; };
  // x staged in smem whenever it fits; prefer two CTAs per SM (a 3-batch ring if that is what
  // keeps the second CTA), else one CTA per SM with the whole x resident
  const bool xs = xs_bytes <= xs_max && fixed + ring4 + xs_bytes + kStatic <= 227 * 1024;
  a.xs_ld = xs ? a.m_pad + a.k_pad + 8 : 0;  // 16 B skew between rows: conflict-free LDS.128
  const size_t xb = xs ? xs_bytes : 0;
  int per_sm = fits2(fixed + ring4 + xb) ? 2 : 1;
  // (x of more than 8 columns never fits two CTAs: the 3-batch form exists for NT == 1 only)
  const bool r3 = NT == 1 && per_sm == 1 && fits2(fixed + ring3 + xb);
  if (r3) per_sm = 2;
  per_sm = std::min(per_sm, env_int("QEFT_GEMV_CPS", per_sm));
  if constexpr (NT == 1) {
    if (r3) {
      if (xs) return launch_kernel<BITS, NT, GT, T, true, 3>(a, fixed + ring3 + xb, per_sm, st);
      return launch_kernel<BITS, NT, GT, T, false, 3>(a, fixed + ring3, per_sm, st);
    }
  }
  if (xs) return launch_kernel<BITS, NT, GT, T, true, kR>(a, fixed + ring4 + xb, per_sm, st);
  return launch_kernel<BITS, NT, GT, T, false, kR>(a, fixed + ring4, per_sm, st);
}

template <int BITS, typename T>
int dispatch_gt(const GemvArgs& a, int gt, cudaStream_t st) {
  const bool nt2 = a.n > 8;
#define QEFT_GT(NT)                                      \
  switch (gt) {                                          \
    case 1: return launch<BITS, NT, 1, T>(a, st);        \
    case 2: return launch<BITS, NT, 2, T>(a, st);        \
    case 4: return launch<BITS, NT, 4, T>(a, st);        \
    default: return launch<BITS, NT, 0, T>(a, st);       \
  }
  if (nt2) {
    QEFT_GT(2)
  } else {
    QEFT_GT(1)
  }
#undef QEFT_GT
}

}  // namespace

namespace qeft {

// Workspace = [64 KB of row-block counters for the bulk-copy path (zero between calls)]
//             [split-K partials (bulk-copy path) | x gather buffer (generic path)].
constexpr size_t kWsHead = 64 * 1024;

// (+ the fused RMS-norm's fallback: normalized x [n][ic] and rstd [n] behind the gather buffer)
static size_t norm_ws_bytes(const qeft_linear_t* L, int n) { return (size_t)n * L->ic * 2 + (size_t)n * 4 + 512; }
static size_t gather_ws_bytes(const qeft_linear_t* L, int n) {
  return ((size_t)n * (L->m_pad + L->k_pad) * 2 + 256 + 255) & ~(size_t)255;
}

size_t gemv_workspace_bytes(const qeft_linear_t* L, int n) {
  return std::max(gemv2_workspace_bytes(L, n), kWsHead + gather_ws_bytes(L, n) + norm_ws_bytes(L, n));
}

int gemv_multi(const qeft_linear_t* const* Ls, int nl, const void* x, int64_t ldx, void* const* ys, int64_t ldy,
               int y_f32, int n, void* ws, size_t ws_bytes, cudaStream_t st, const float* ngain, const void* xu) {
  QEFT_CHECK(nl >= 1 && nl <= kMaxLayers, QEFT_ERR_SHAPE, "gemv: %d layers per launch (1..%d)", nl, kMaxLayers);
  const qeft_linear_t* L = Ls[0];
  QEFT_CHECK(n >= 1 && n <= 16, QEFT_ERR_SHAPE, "gemv: n_cols=%d outside 1..16", n);
  QEFT_CHECK(L->bits == 3 || L->bits == 4, QEFT_ERR_SHAPE, "gemv: bits=%d", L->bits);
  bool v2 = true;
  GemvArgs a{};
  a.nl = nl;
  int rb_total = 0;
  for (int l = 0; l < nl; ++l) {
    const qeft_linear_t* Li = Ls[l];
    // layers of one launch share x: identical K geometry, dtype and column map
    QEFT_CHECK(Li->ic == L->ic && Li->k == L->k && Li->bits == L->bits && Li->g == L->g &&
                   Li->act_dtype == L->act_dtype && Li->flags == L->flags &&
                   (Li->colmap == L->colmap || (L->flags & QEFT_FLAG_STRUCTURED_FAST)),
               QEFT_ERR_SHAPE, "gemv: layer %d does not share the first layer's input geometry", l);
    QEFT_CHECK(ldx >= Li->ic && ldy >= Li->oc, QEFT_ERR_SHAPE, "gemv: ld too small");
    v2 = v2 && gemv2_supported(Li, n);
    a.qw[l] = (const uint8_t*)Li->qweight;
    a.sz[l] = (const float2*)Li->sz;
    a.weak16[l] = (const uint8_t*)Li->weak16;
    a.ys[l] = ys[l];
    a.ocs[l] = Li->oc;
    rb_total += Li->oc_pad / 16;
    a.rb_end[l] = rb_total;
  }
  // bulk-copy warp-ring kernel (qeft_gemv2.cu) for group sizes that are multiples of 64;
  // the per-element-dequant kernel below otherwise
  if (v2) {
    const int r = gemv2_multi(Ls, nl, x, ldx, ys, ldy, y_f32, n, ws, ws_bytes, st, ngain, xu);
    if (r != -1) return r;
  }
  if (xu) {
    // the fused SwiGLU did not fit this launch: the stand-alone kernel, then the plain GEMV
    const size_t off = kWsHead + gather_ws_bytes(L, n);
    QEFT_CHECK(ws_bytes >= off + norm_ws_bytes(L, n) && ldx == L->ic, QEFT_ERR_SHAPE,
               "gemv: workspace too small for the SwiGLU (or ldx != ic)");
    uint8_t* f = (uint8_t*)ws + off;
    if (int r = silu_mul_fwd(x, xu, f, (int64_t)n * L->ic, L->act_dtype, st)) return r;
    return gemv_multi(Ls, nl, f, L->ic, ys, ldy, y_f32, n, ws, ws_bytes, st, ngain, nullptr);
  }
  if (ngain) {
    // the fused norm did not fit this launch: the stand-alone kernel, then the plain GEMV
    const size_t off = kWsHead + gather_ws_bytes(L, n);
    QEFT_CHECK(ws_bytes >= off + norm_ws_bytes(L, n) && ldx == L->ic, QEFT_ERR_SHAPE,
               "gemv: workspace too small for the RMS-norm (or ldx != ic)");
    uint8_t* xn = (uint8_t*)ws + off;
    float* rstd = (float*)(xn + (((size_t)n * L->ic * 2 + 255) & ~(size_t)255));
    if (int r = rmsnorm_fwd(x, ngain, xn, rstd, n, L->ic, L->act_dtype, st)) return r;
    return gemv_multi(Ls, nl, xn, L->ic, ys, ldy, y_f32, n, ws, ws_bytes, st, nullptr);
  }
  QEFT_CHECK(ws_bytes >= kWsHead, QEFT_ERR_SHAPE, "gemv: workspace too small");
  ws = (uint8_t*)ws + kWsHead;  // never touch the bulk-copy path's counters
  ws_bytes -= kWsHead;
  a.ldy = ldy;
  a.y_f32 = y_f32;
  a.m = L->m; a.m_pad = L->m_pad; a.k = L->k; a.k_pad = L->k_pad;
  a.g = L->g; a.ng = L->ng; a.n = n;
  a.n_rb = rb_total;
  a.rbb = rowblock_bytes(L->bits, L->m_pad);
  a.nsq = L->m_pad / 64;
  a.dbg = env_int("QEFT_GEMV_DEBUG", 0);
  int gt = (L->g % 64) == 0 ? L->g / 64 : 0;
  if (gt != 1 && gt != 2 && gt != 4) gt = 0;  // generic per-element dequant
  // warps split the quantized steps in whole groups (and whole 3-bit tiles)
  int unit = std::max(gt, 1);
  if (L->bits == 3 && unit == 1) unit = 2;
  int spw = (a.nsq + kWarps - 1) / kWarps;
  spw = (spw + unit - 1) / unit * unit;
  a.spw = std::max(spw, unit);
  const bool fast = (L->flags & QEFT_FLAG_STRUCTURED_FAST) && (ldx % 8 == 0) &&
                    (((uintptr_t)x & 15) == 0);
  if (fast) {
    a.x = (const uint8_t*)x;
    a.ldx = ldx;
    a.gathered = 0;
  } else {
    const int kk = L->m_pad + L->k_pad;
    QEFT_CHECK(ws_bytes >= (size_t)n * kk * 2, QEFT_ERR_SHAPE, "gemv: workspace %zu too small",
               ws_bytes);
    if (int r = gather_cols(x, ldx, L->colmap, kk, n, L->act_dtype, ws, st)) return r;
    a.x = (const uint8_t*)ws;
    a.ldx = kk;
    a.gathered = 1;
  }
  const bool bf = L->act_dtype == QEFT_BF16;
  if (L->bits == 4) return bf ? dispatch_gt<4, __nv_bfloat16>(a, gt, st) : dispatch_gt<4, __half>(a, gt, st);
  return bf ? dispatch_gt<3, __nv_bfloat16>(a, gt, st) : dispatch_gt<3, __half>(a, gt, st);
}

int gemv(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int y_f32, int n,
         void* ws, size_t ws_bytes, cudaStream_t st) {
  return gemv_multi(&L, 1, x, ldx, &y, ldy, y_f32, n, ws, ws_bytes, st);
}

}  // namespace qeft
