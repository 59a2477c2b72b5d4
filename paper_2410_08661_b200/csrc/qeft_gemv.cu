// Decode GEMV for the QEFT mixed-precision layer, N = 1..16 activation columns.
//
// Replaces the reference's matvec paths (pkg/src/qeft/kernels.py:66-157,
// `_grouped_accumulate`): y = sum_g s_g * (c_g . x_g) + z_g * sum(x_g) + W_weak . x_weak.
//
// HBM-bound design for B200:
//   * Each 16-row block of the layer is a list of equal "chunks": the quantized
//     part (256 K columns of codes per chunk, contiguous in the tile layout)
//     followed by the weak block (64 fp16 columns per chunk, row-block tiles).
//     grid = (S ranks, 128-row groups) launched as clusters of the S ranks of
//     one row group; rank s takes an equal contiguous share of the chunk list,
//     so quantized and weak work are balanced across the cluster.
//   * CTA = 4 warps; warp w owns TWO row-blocks (32 rows) so every x fragment,
//     every sum(x) MMA and all per-chunk bookkeeping is shared by 32 rows.
//   * Chunks stream through shared memory with TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx) into a private ring per warp; a
//     quantized chunk's group (scale, zero) pairs ride in the same slot. One lane
//     refills a slot as soon as the warp consumed it. The first ring-full is
//     issued before the programmatic-dependent-launch wait, so a kernel's weight
//     stream overlaps the previous kernel in the stream.
//   * x is staged per chunk into a double-buffered smem tile by the whole CTA,
//     prefetched one chunk ahead in registers.
//   * codes become mma.m16n8k16 A fragments with one LOP3 per fragment
//     ((magic + code) halves); the MMA accumulates sum (magic + c) x in fp32 and a
//     second MMA with an all-ones A fragment accumulates sum(x) in the same
//     fragment layout, so the per-group fold
//       y += s' * acc + (z - magic * s') * sum(x)   (s' = s, or s/16 for the
//     fp16 hi-nibble trick) needs no separate pass over x.
//   * Ranks are combined deterministically through distributed shared memory:
//     each CTA leaves its fp32 partial in its own smem, the cluster syncs, and
//     rank 0 sums the ranks in order.
#include <algorithm>

#include "qeft_common.cuh"
#include "qeft_internal.h"

using namespace qeft;

namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kRB = 2;                // row-blocks per warp
constexpr int kRows = kWarps * kRB * 16;  // rows per CTA
constexpr int kSlots = 2;             // ring depth per warp (2 x 4 KB of codes in flight)
constexpr int kQCols = 256;           // K columns per quantized chunk
constexpr int kWCols = 64;            // K columns per weak chunk
constexpr int kQBytes4 = 2048;        // 16 rows x 256 codes x 4 bit
constexpr int kQBytes3 = 1536;        // 16 rows x 256 codes x 3 bit
constexpr int kWBytes = 2048;         // 16 rows x 64 x 16 bit
constexpr int kPart = 2560;           // per row-block: chunk bytes (<= 2 KB) + (s, z) of <= 4 groups
constexpr int kSzOff = 2048;
constexpr int kSlotBytes = kRB * kPart;
constexpr int kMaxCluster = 8;
constexpr int kXStride = kQCols + 8;  // halves; 528 B == 16 mod 32 -> conflict-free LDS.128

struct GemvArgs {
  const uint8_t* qw;
  const float2* sz;
  const void* weak16;
  const void* x;      // [n][ldx]; fast: original columns; else pre-gathered B200 order
  int64_t ldx;
  void* y;
  int64_t ldy;
  int y_f32;
  int oc, m, m_pad, k, k_pad, g, ng, n;
  int nq, nw, ranks, gathered;  // chunks per row-block: nq quantized + nw weak
  int gt;                       // 64-column steps per group (FOLD: g % 64 == 0)
  uint32_t mgt;                 // ceil(2^32 / gt): ti / gt == umulhi(ti, mgt) for gt > 1
};

template <typename T>
__device__ __forceinline__ void store_out(const GemvArgs& a, int n, int row, float v) {
  if (a.y_f32)
    ((float*)a.y)[(int64_t)n * a.ldy + row] = v;
  else
    ((T*)a.y)[(int64_t)n * a.ldy + row] = from_f32<T>(v);
}

template <int BITS, int NT, typename T, bool FOLD>
__global__ void __launch_bounds__(kThreads)
gemv_kernel(const GemvArgs a) {
  using T2 = typename DTraits<T>::T2;
  constexpr int kXPer = NT * 2;  // uint4 of x per thread per chunk: (8*NT rows x 256 cols / 8) / 128
  constexpr int kQBytes = BITS == 4 ? kQBytes4 : kQBytes3;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kWarps][kSlots];
  __shared__ __align__(16) float xsum_s[2][kQCols / 64][16];
  float (*part)[kRows] = reinterpret_cast<float (*)[kRows]>(smem);  // reuses the rings at the end

  const int s = blockIdx.x, rg = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int rb0 = (rg * kWarps + warp) * kRB;           // first of this warp's row-blocks
  const int nrb = min(kRB, max(0, (a.oc - rb0 * 16 + 15) / 16));  // valid row-blocks (0..2)
  const int ntot = a.nq + a.nw;
  const int c0 = (int)((int64_t)s * ntot / a.ranks), c1 = (int)((int64_t)(s + 1) * ntot / a.ranks);
  const int nchunk = c1 - c0;
  uint8_t* ring = smem + warp * (kSlots * kSlotBytes);
  T* xs = reinterpret_cast<T*>(smem + kWarps * kSlots * kSlotBytes);  // [2][8*NT][kXStride]
  uint64_t* bar = bars[warp];
  const int64_t rbb = rowblock_bytes(BITS, a.m_pad);

  // ti / gt without a hardware-emulated division (exact for ti * gt < 2^32)
  auto div_gt = [&](int ti) -> int { return a.gt == 1 ? ti : (int)__umulhi((uint32_t)ti, a.mgt); };

  // ---- 1. producer: lane 0 of each warp fills its private ring ----
  auto issue = [&](int c, int slot) {
    uint8_t* dst = ring + slot * kSlotBytes;
    if (c >= a.nq) {
      mbar_expect_tx(&bar[slot], nrb * kWBytes);
      for (int r = 0; r < nrb; ++r)
        bulk_g2s(dst + r * kPart,
                 (const uint8_t*)a.weak16 + ((int64_t)(rb0 + r) * (a.k_pad >> 6) + (c - a.nq)) * kWBytes,
                 kWBytes, &bar[slot]);
      return;
    }
    const int tiles = min(kQCols, a.m_pad - c * kQCols) >> 6;
    const uint32_t nb = (uint32_t)(tiles * 64 * 2 * BITS);  // 16 rows * bits / 8 per column
    int gf = 0;
    uint32_t nsz = 0;
    if (FOLD) {
      gf = min(div_gt(c * (kQCols / 64)), a.ng - 1);
      const int gl = min(div_gt(c * (kQCols / 64) + tiles - 1), a.ng - 1);
      nsz = (uint32_t)(gl - gf + 1) * 16 * sizeof(float2);
    }
    mbar_expect_tx(&bar[slot], nrb * (nb + nsz));
    for (int r = 0; r < nrb; ++r) {
      bulk_g2s(dst + r * kPart, a.qw + (int64_t)(rb0 + r) * rbb + (int64_t)c * kQBytes, nb, &bar[slot]);
      if (FOLD)
        bulk_g2s(dst + r * kPart + kSzOff, a.sz + ((int64_t)(rb0 + r) * a.ng + gf) * 16, nsz, &bar[slot]);
    }
  };
  if (lane == 0) {
    for (int i = 0; i < kSlots; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0 && nrb > 0) {
    for (int i = 0; i < min(nchunk, kSlots); ++i) issue(c0 + i, i);
  }

  // Programmatic dependent launch: the next kernel may start streaming its own
  // weights now; x (the previous kernel's output) is read only after the wait.
  pdl_launch_dependents();
  pdl_wait();

  // x chunk staging: thread -> (row xn, 8-column piece xp) pairs, kXPer per thread
  auto cbase = [&](int c) { return c < a.nq ? c * kQCols : a.m_pad + (c - a.nq) * kWCols; };
  const T* xg = (const T*)a.x;
  uint4 xr[kXPer];
  auto x_load = [&](int c) {
    const int base = cbase(c);
    const int lim = c < a.nq ? a.m : a.m_pad + a.k;  // valid B200 columns of this region
#pragma unroll
    for (int i = 0; i < kXPer; ++i) {
      const int e = threadIdx.x + i * kThreads;
      const int n = e >> 5, j = base + 8 * (e & 31);
      const int col = (a.gathered || j < a.m_pad) ? j : a.m + (j - a.m_pad);
      const bool ok = n < a.n && (a.gathered ? (j < a.m_pad + a.k_pad) : (j < lim)) &&
                      (c >= a.nq ? (8 * (e & 31) < kWCols) : true);
      xr[i] = ok ? *reinterpret_cast<const uint4*>(xg + (int64_t)n * a.ldx + col) : make_uint4(0, 0, 0, 0);
    }
  };
  // also leaves fp32 sums of every 64-column segment: xsum_s[buf][seg][row] (zero-point fold)
  auto x_store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < kXPer; ++i) {
      const int e = threadIdx.x + i * kThreads;
      *reinterpret_cast<uint4*>(xs + (buf * 8 * NT + (e >> 5)) * kXStride + 8 * (e & 31)) = xr[i];
      if constexpr (FOLD) {
        const T2* h = reinterpret_cast<const T2*>(&xr[i]);
        float sum = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f2 = t2_to_f2<T2>(h[q]);
          sum += f2.x + f2.y;
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        if ((lane & 7) == 0) xsum_s[buf][(e & 31) >> 3][e >> 5] = sum;
      }
    }
  };
  if (nchunk > 0) {
    x_load(c0);
    x_store(0);
  }
  __syncthreads();

  float acc[kRB][NT][4], accg[kRB][NT][4], accx[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      accx[nt][e] = 0.f;
#pragma unroll
      for (int r = 0; r < kRB; ++r) acc[r][nt][e] = accg[r][nt][e] = 0.f;
    }
  const uint32_t ones[4] = {DTraits<T>::kOne2, DTraits<T>::kOne2, DTraits<T>::kOne2, DTraits<T>::kOne2};
  int xrow[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xrow[nt] = min(g8 + 8 * nt, a.n - 1);

  // fold group grp of row-block r; its params are in the current slot (starting at group gf)
  auto fold = [&](int grp, const uint8_t* buf, int gf) {
    constexpr float M = DTraits<T>::kMagicF;
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      const float2* sz = reinterpret_cast<const float2*>(buf + r * kPart + kSzOff) + (grp - gf) * 16;
      const float2 p0 = sz[g8];
      const float2 p1 = sz[g8 + 8];
      const float s0 = p0.x;
      const float s1 = (BITS == 4 && DTraits<T>::kHiTrick) ? p1.x * (1.f / 16.f) : p1.x;
      const float z0 = p0.y - M * s0, z1 = p1.y - M * s1;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        acc[r][nt][0] += s0 * accg[r][nt][0] + z0 * accx[nt][0];
        acc[r][nt][1] += s0 * accg[r][nt][1] + z0 * accx[nt][1];
        acc[r][nt][2] += s1 * accg[r][nt][2] + z1 * accx[nt][2];
        acc[r][nt][3] += s1 * accg[r][nt][3] + z1 * accx[nt][3];
#pragma unroll
        for (int e = 0; e < 4; ++e) accg[r][nt][e] = 0.f;
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) accx[nt][e] = 0.f;
  };

  // per-element dequant (group sizes that are not a multiple of 64)
  auto dq_frag = [&](uint32_t mag, bool hi16, int rb, int row_local, int col) -> uint32_t {
    const float2 cf = t2_to_f2<T2>(magic_to_code<T>(mag, hi16));
    const int gA = min(col / a.g, a.ng - 1), gB = min((col + 1) / a.g, a.ng - 1);
    const float2* sz = a.sz + (int64_t)rb * a.ng * 16;
    const float2 pA = sz[gA * 16 + row_local];
    const float2 pB = sz[gB * 16 + row_local];
    T2 r;
    r.x = from_f32<T>(cf.x * pA.x + pA.y);
    r.y = from_f32<T>(cf.y * pB.x + pB.y);
    return *reinterpret_cast<uint32_t*>(&r);
  };

  // B fragments of one 64-column step at chunk-local column xc
  auto x_frag = [&](const T* xbuf, int xc, uint4 xa[NT], uint4 xb[NT]) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const T* xp = xbuf + xrow[nt] * kXStride + xc + 16 * t4;
      xa[nt] = *reinterpret_cast<const uint4*>(xp);
      xb[nt] = *reinterpret_cast<const uint4*>(xp + 8);
    }
  };
  auto bsel = [](const uint4& xa, const uint4& xb, int j, uint32_t& b0, uint32_t& b1) {
    b0 = (j == 0) ? xa.x : (j == 1) ? xa.z : (j == 2) ? xb.x : xb.z;
    b1 = (j == 0) ? xa.y : (j == 1) ? xa.w : (j == 2) ? xb.y : xb.w;
  };

  // last quantized column this rank covers (a group is folded at its end or here)
  const int qend = min(min(c1, a.nq) * kQCols, a.m_pad);

  // ---- 2. consumer: the CTA walks its chunks in lockstep (x is shared) ----
  for (int i = 0; i < nchunk; ++i) {
    const int c = c0 + i;
    if (i + 1 < nchunk) x_load(c + 1);  // next x chunk in flight during this chunk's math
    const T* xbuf = xs + (i & 1) * 8 * NT * kXStride;
    if (nrb > 0) {
      const int slot = i % kSlots;
      mbar_wait(&bar[slot], (i / kSlots) & 1);
      const uint8_t* buf = ring + slot * kSlotBytes;
      if (c >= a.nq) {
        // weak tile: 16 rows x 64 fp16, row-major; lane reads rows g8, g8+8, cols 16t..16t+15
        uint4 xa[NT], xb[NT];
        x_frag(xbuf, 0, xa, xb);
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
          const T* w16 = (const T*)(buf + r * kPart);
          const uint4 r0a = *reinterpret_cast<const uint4*>(w16 + g8 * 64 + 16 * t4);
          const uint4 r0b = *reinterpret_cast<const uint4*>(w16 + g8 * 64 + 16 * t4 + 8);
          const uint4 r1a = *reinterpret_cast<const uint4*>(w16 + (g8 + 8) * 64 + 16 * t4);
          const uint4 r1b = *reinterpret_cast<const uint4*>(w16 + (g8 + 8) * 64 + 16 * t4 + 8);
          const uint32_t f[4][4] = {{r0a.x, r1a.x, r0a.y, r1a.y}, {r0a.z, r1a.z, r0a.w, r1a.w},
                                    {r0b.x, r1b.x, r0b.y, r1b.y}, {r0b.z, r1b.z, r0b.w, r1b.w}};
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              uint32_t b0, b1;
              bsel(xa[nt], xb[nt], j, b0, b1);
              mma16816<T>(acc[r][nt], f[j], b0, b1);
            }
        }
      } else {
        const int jc0 = c * kQCols;
        const int tiles = min(kQCols, a.m_pad - jc0) >> 6;
        // group bookkeeping without per-step division
        const int t0 = c * (kQCols / 64);
        int grp = FOLD ? div_gt(t0) : 0;
        const int gf = FOLD ? min(grp, a.ng - 1) : 0;
        int left = FOLD ? a.gt - (t0 - grp * a.gt) : 0;
#pragma unroll
        for (int st = 0; st < kQCols / 64; ++st) {
          if (st < tiles) {
            const int jc = jc0 + 64 * st;
            uint4 xa[NT], xb[NT];
            x_frag(xbuf, 64 * st, xa, xb);
            // sum(x) of this step for this lane's output columns (2t, 2t+1 [+8])
            if constexpr (FOLD) {
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                const float2 sx = *reinterpret_cast<const float2*>(&xsum_s[i & 1][st][8 * nt + 2 * t4]);
                accx[nt][0] += sx.x;
                accx[nt][1] += sx.y;
                accx[nt][2] += sx.x;
                accx[nt][3] += sx.y;
              }
            }
#pragma unroll
            for (int r = 0; r < kRB; ++r) {
              uint32_t f[4][4];
              if constexpr (BITS == 4) {
                const uint4 q = *reinterpret_cast<const uint4*>(buf + r * kPart + st * 512 + lane * 16);
                const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) decode4<T>(qq[j], f[j]);
              } else {
                const uint8_t* tb = buf + r * kPart + (st >> 1) * 768;
                const int h = st & 1;
                const uint2 w2 = *reinterpret_cast<const uint2*>(tb + lane * 16 + 8 * h);
                const uint32_t hb = *reinterpret_cast<const uint32_t*>(tb + 512 + lane * 8 + 4 * h);
                const uint32_t ww2[2] = {w2.x, w2.y};
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                  for (int pp = 0; pp < 4; ++pp)
                    f[j][pp] = decode3_pair<T>(ww2[j >> 1], hb, 4 * (j & 1) + pp, j >> 1);
              }
              if constexpr (!FOLD) {
                constexpr bool h16 = (BITS == 4) && DTraits<T>::kHiTrick;
                const int rb = rb0 + r;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int cc = jc + 16 * t4 + 4 * j;
                  f[j][0] = dq_frag(f[j][0], false, rb, g8, cc);
                  f[j][1] = dq_frag(f[j][1], h16, rb, g8 + 8, cc);
                  f[j][2] = dq_frag(f[j][2], false, rb, g8, cc + 2);
                  f[j][3] = dq_frag(f[j][3], h16, rb, g8 + 8, cc + 2);
                }
              }
#pragma unroll
              for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                  uint32_t b0, b1;
                  bsel(xa[nt], xb[nt], j, b0, b1);
                  mma16816<T>(FOLD ? accg[r][nt] : acc[r][nt], f[j], b0, b1);
                }
            }
            if constexpr (FOLD) {
              // a group is folded right after its last step, while its params are in this slot
              if (--left == 0 || jc + 64 >= qend) {
                fold(min(grp, a.ng - 1), buf, gf);
                ++grp;
                left = a.gt;
              }
            }
          }
        }
      }
      // slot consumed by the whole warp -> refill it
      __syncwarp();
      if (lane == 0 && i + kSlots < nchunk) issue(c + kSlots, slot);
    }
    if (i + 1 < nchunk) x_store((i + 1) & 1);
    __syncthreads();
  }

  // ---- 3. output ----
  if (a.ranks == 1) {
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      const int row0 = (rb0 + r) * 16 + g8, row1 = row0 + 8;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int cA = 8 * nt + 2 * t4;
        if (cA < a.n) {
          if (row0 < a.oc) store_out<T>(a, cA, row0, acc[r][nt][0]);
          if (row1 < a.oc) store_out<T>(a, cA, row1, acc[r][nt][2]);
        }
        if (cA + 1 < a.n) {
          if (row0 < a.oc) store_out<T>(a, cA + 1, row0, acc[r][nt][1]);
          if (row1 < a.oc) store_out<T>(a, cA + 1, row1, acc[r][nt][3]);
        }
      }
    }
    return;
  }
  __syncthreads();  // every warp is done with its ring before partials overwrite it
#pragma unroll
  for (int r = 0; r < kRB; ++r) {
    const int rl0 = (warp * kRB + r) * 16 + g8, rl1 = rl0 + 8;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int cA = 8 * nt + 2 * t4;
      part[cA][rl0] = acc[r][nt][0];
      part[cA][rl1] = acc[r][nt][2];
      part[cA + 1][rl0] = acc[r][nt][1];
      part[cA + 1][rl1] = acc[r][nt][3];
    }
  }
  cluster_sync();  // partials of every rank are visible cluster-wide
  if (cluster_ctarank() == 0) {
    const uint32_t local = smem_u32(&part[0][0]);
    for (int e = threadIdx.x; e < a.n * kRows; e += blockDim.x) {
      const int cc = e / kRows, rl = e % kRows;
      float v = 0.f;
      for (int r = 0; r < a.ranks; ++r) v += ld_dsmem_f32(local + (uint32_t)(cc * kRows + rl) * 4, r);
      const int row = rg * kRows + rl;
      if (row < a.oc) store_out<T>(a, cc, row, v);
    }
  }
  cluster_sync();  // keep every rank's smem alive until rank 0 has read it
}

template <int BITS, int NT, typename T, bool FOLD>
int launch(const GemvArgs& a, int n_rg, cudaStream_t st) {
  auto kern = gemv_kernel<BITS, NT, T, FOLD>;
  const size_t smem = (size_t)kWarps * kSlots * kSlotBytes + (size_t)2 * 8 * NT * kXStride * sizeof(T);
  static bool attr_done = false;
  if (!attr_done) {
    QEFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done = true;
  }
  QEFT_CUDA(launch_pdl_cluster(kern, dim3(a.ranks, n_rg), dim3(kThreads), smem, st, a.ranks, a));
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
  // gather buffer for layouts whose x cannot be read in place
  return (size_t)n * (L->m_pad + L->k_pad) * 2 + 256;
}

int gemv(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int y_f32, int n,
         void* ws, size_t ws_bytes, cudaStream_t st) {
  QEFT_CHECK(n >= 1 && n <= 16, QEFT_ERR_SHAPE, "gemv: n_cols=%d outside 1..16", n);
  QEFT_CHECK(L->bits == 3 || L->bits == 4, QEFT_ERR_SHAPE, "gemv: bits=%d", L->bits);
  QEFT_CHECK(ldx >= L->ic && ldy >= L->oc, QEFT_ERR_SHAPE, "gemv: ld too small");
  GemvArgs a;
  a.qw = (const uint8_t*)L->qweight;
  a.sz = (const float2*)L->sz;
  a.weak16 = L->weak16;
  a.x = x;
  a.ldx = ldx;
  a.y = y;
  a.ldy = ldy;
  a.y_f32 = y_f32;
  a.oc = L->oc; a.m = L->m; a.m_pad = L->m_pad; a.k = L->k; a.k_pad = L->k_pad;
  a.g = L->g; a.ng = L->ng; a.n = n;
  a.nq = (L->m_pad + kQCols - 1) / kQCols;
  a.nw = L->k_pad / kWCols;
  a.gt = std::max(1, L->g / 64);
  a.mgt = a.gt > 1 ? (uint32_t)((0x100000000ull + a.gt - 1) / a.gt) : 0u;
  const int n_rg = (L->oc_pad + kRows - 1) / kRows;
  // ranks per row group: cover the chip ~2x, <= one portable cluster, >= 2 chunks each
  int ranks = (2 * 148 + n_rg - 1) / n_rg;
  ranks = std::min(ranks, kMaxCluster);
  ranks = std::min(ranks, std::max(1, (a.nq + a.nw) / 2));
  a.ranks = std::max(ranks, 1);
  const bool fast = (L->flags & QEFT_FLAG_STRUCTURED_FAST) && (ldx % 8 == 0) &&
                    (((uintptr_t)x & 15) == 0);
  a.gathered = fast ? 0 : 1;
  if (!fast) {
    const int kk = L->m_pad + L->k_pad;
    QEFT_CHECK(ws_bytes >= (size_t)n * kk * 2, QEFT_ERR_SHAPE, "gemv: workspace %zu too small",
               ws_bytes);
    if (int r = gather_cols(x, ldx, L->colmap, kk, n, L->act_dtype, ws, st)) return r;
    a.x = ws;
    a.ldx = kk;
  }
  const bool fold = (L->g % 64) == 0;
  if (L->act_dtype == QEFT_F16) return dispatch<__half>(a, L->bits, n_rg, fold, st);
  return dispatch<__nv_bfloat16>(a, L->bits, n_rg, fold, st);
}

}  // namespace qeft
