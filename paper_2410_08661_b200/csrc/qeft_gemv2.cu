// Decode GEMV, bulk-copy warp rings: the HBM-bound hot kernel of the decode path.
//
// Replaces the reference's matvec paths (pkg/src/qeft/kernels.py:66-157,
// `_grouped_accumulate`): y = sum_g s_g * (c_g . x_g) + z_g * sum(x_g) + W_weak . x_weak,
// for 1..16 activation columns and up to 3 layers that read the same x (q/k/v, gate/up).
//
// Why this shape (measured on B200, scripts/micro/bulk_warp_bench.cu, profiles/r02):
//   * every warp owns a private ring of R stages fed by its OWN lane 0 with 1-D bulk copies
//     (cp.async.bulk, the TMA engine) completing on an mbarrier: 8 warps x 3 x 4 KB per SM
//     streams 6.9-7.0 TB/s. No per-lane address arithmetic, no producer/consumer handshake
//     across warps: a warp waits on its own barrier, decodes, multiplies, and refills.
//   * work split: a thread-block cluster of S CTAs owns a contiguous run of row-blocks (16
//     output rows each); CTA rank r streams K slice r of every one of them (slices are whole
//     groups, balanced by bytes). Inside a CTA the run's stages (4 KB each) are dealt to the
//     8 warps round-robin, so every warp streams the same number of bytes. Partials go to
//     shared memory; at the end the 8 warp partials and then the S slice partials (over
//     DSMEM) are summed in a fixed order: deterministic, no atomics, no global scratch.
//   * x is staged once per CTA for its K slice only (gathered through the column map for
//     irregular / online layouts, so no separate gather launch), with the per-(group,
//     column) sums of x that the zero-point fold needs.
//   * codes become (magic + code) half2 A fragments with one LOP3 each (qeft_common.cuh
//     decode4 / decode3_pair) for mma.sync m16n8k16 (x is the B operand: 8 columns per MMA
//     at no extra cost), and every group is folded as
//       acc += s' * sum(c' x) + (z - magic * s') * sum(x)     (fp32)
//     with (scale, zero) read as an fp16 pair (sz16, 4 B per row and group: SURVEY 7.3).
//   * programmatic dependent launch: each warp issues its first weight stages BEFORE
//     griddepcontrol.wait, so a layer's weight stream overlaps the previous kernel's tail;
//     x and the trainable weak block are read only after the wait.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "qeft_common.cuh"
#include "qeft_internal.h"

using namespace qeft;

namespace {

// Launch shape (template): NW warps per CTA, CPS 128-column chunks per codes stage (a stage
// holds CPS * 1 KB of 4-bit codes + their sz16 pairs, or CPS / 2 weak tiles), R stages per ring.
constexpr int kMaxS = 4;            // K slices = cluster size
constexpr int kMaxL = 3;            // layers per launch
constexpr int kMaxJ = 48;           // row-blocks per cluster (partials live in shared memory)

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

struct G2Args {
  const uint8_t* qw[kMaxL];
  const uint8_t* sz[kMaxL];
  const uint8_t* wk[kMaxL];
  void* ys[kMaxL];
  int ocs[kMaxL];
  int rb_end[kMaxL];
  int nl;
  const void* x;
  int64_t ldx;
  const int* colmap;
  int fast;  // x read in place (structured layout): B200 K order = [0, m) then [m, ic)
  int64_t ldy;
  int yflags;  // QEFT_Y_F32 | QEFT_Y_ACCUMULATE
  int m, m_pad, k, k_pad, g, n, n_rb;
  int nch;   // m_pad / 128 chunks
  int U;     // chunks per slicing unit (whole groups)
  int nuc;   // codes units
  int ng16;  // sz16 groups per row-block
  int S;     // K slices (cluster size)
  int ub[kMaxS + 1];
  int J;        // row-blocks per cluster
  int xs_ld;    // staged x row stride (elements)
  int64_t rbb;  // qweight bytes per row-block
};

struct Slice {
  int c0, c1, w0, w1;
};

QEFT_DEV Slice slice_of(const G2Args& a, int s) {
  const int u0 = a.ub[s], u1 = a.ub[s + 1];
  Slice r;
  r.c0 = min(min(u0, a.nuc) * a.U, a.nch);
  r.c1 = min(min(u1, a.nuc) * a.U, a.nch);
  r.w0 = max(u0, a.nuc) - a.nuc;
  r.w1 = max(u1, a.nuc) - a.nuc;
  return r;
}

// B200 K position where unit boundary u starts
QEFT_DEV int kpos(const G2Args& a, int u) {
  return u <= a.nuc ? min(u * a.U, a.nch) * 128 : a.m_pad + (u - a.nuc) * 64;
}

QEFT_DEV int layer_of(const G2Args& a, int j, int& lrb) {
  int l = 0;
  while (l + 1 < a.nl && j >= a.rb_end[l]) ++l;
  lrb = j - (l ? a.rb_end[l - 1] : 0);
  return l;
}

QEFT_DEV uint4 lds128(const void* p) { return *reinterpret_cast<const uint4*>(p); }
QEFT_DEV uint2 lds64(const void* p) { return *reinterpret_cast<const uint2*>(p); }

template <int BITS, int NT, int GT, typename T, int R, int NW, int CPS>
__global__ void __launch_bounds__(NW * 32, 1) gemv2_kernel(const G2Args a) {
  constexpr int kNW = NW, kCPS = CPS, kWPS = CPS / 2;
  constexpr int kSzOff = CPS * 1024, kStage = CPS * 1152;  // codes, then sz16 pairs
  constexpr int NTS = NT * 8;                 // x-sum column stride
  constexpr int CB = BITS == 4 ? 1024 : 768;  // bytes per 128-column chunk of 16 rows
  constexpr int HG = GT >= 2 ? GT / 2 : 1;    // chunks per group (GT >= 2)
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kNW][R];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int rank = a.S > 1 ? (int)cluster_ctarank() : 0;
  const int clu = blockIdx.x / a.S;

  // shared memory: [rings][partials red: J x kNW x 16 x n floats][x: n x xs_ld][x sums]
  uint8_t* ring = smem + (size_t)warp * R * kStage;
  float* red = reinterpret_cast<float*>(smem + (size_t)kNW * R * kStage);
  const int redn = 16 * a.n;  // floats per (row-block, warp)
  T* xs = reinterpret_cast<T*>(red + (size_t)a.J * kNW * redn);
  float* xsum = reinterpret_cast<float*>(xs + (size_t)a.n * a.xs_ld);

  // this CTA: row-blocks [j0, j1) of the cluster, K slice `rank`; stages of row-block jl are
  // jl * nst .. jl * nst + nst - 1 (codes stages, then weak stages); warp w takes w, w + 8, ...
  const int j0 = clu * a.J, j1 = min(j0 + a.J, a.n_rb), nj = max(j1 - j0, 0);
  const Slice sl = slice_of(a, rank);
  const int ncs = (sl.c1 - sl.c0 + kCPS - 1) / kCPS;
  const int nst = ncs + (sl.w1 - sl.w0 + kWPS - 1) / kWPS;
  const int total = nj * nst;
  const int my_n = warp < total ? (total - warp + kNW - 1) / kNW : 0;

  // ---- lane 0: bulk-copy issue (stage i of this warp = global stage warp + i * kNW) ----
  int issued = 0;
  int is_jl = warp / max(nst, 1), is_t = warp - is_jl * nst;
  const uint8_t *pq = nullptr, *ps = nullptr, *pw = nullptr;  // row-block is_jl's streams
  auto rb_ptrs = [&]() {
    int lrb;
    const int l = layer_of(a, j0 + is_jl, lrb);
    pq = a.qw[l] + lrb * a.rbb;
    ps = a.sz[l] + (int64_t)lrb * a.ng16 * 64;
    pw = a.wk[l] + (int64_t)lrb * (a.k_pad >> 6) * 2048;
  };
  if (lane == 0 && my_n > 0) rb_ptrs();
  auto issue = [&](bool codes_only) -> bool {
    if (issued >= my_n) return false;
    if (codes_only && is_t >= ncs) return false;
    const int slot = issued % R;
    uint8_t* dst = ring + slot * kStage;
    uint64_t* bar = &full[warp][slot];
    if (is_t < ncs) {
      const int ca = sl.c0 + is_t * kCPS, cb = min(ca + kCPS, sl.c1);
      const int ga = GT == 1 ? 2 * ca : ca / HG;
      const int gb = GT == 1 ? 2 * cb : (cb + HG - 1) / HG;
      const uint32_t cbytes = (uint32_t)(cb - ca) * CB, sbytes = (uint32_t)(gb - ga) * 64;
      mbar_expect_tx(bar, cbytes + sbytes);
      bulk_g2s(dst, pq + ca * CB, cbytes, bar);
      bulk_g2s(dst + kSzOff, ps + ga * 64, sbytes, bar);
    } else {
      const int wa = sl.w0 + (is_t - ncs) * kWPS, wb = min(wa + kWPS, sl.w1);
      const uint32_t bytes = (uint32_t)(wb - wa) * 2048;
      mbar_expect_tx(bar, bytes);
      bulk_g2s(dst, pw + wa * 2048, bytes, bar);
    }
    ++issued;
    is_t += kNW;
    if (is_t >= nst) {
      do {
        is_t -= nst;
        ++is_jl;
      } while (is_t >= nst);
      if (issued < my_n) rb_ptrs();
    }
    return true;
  };

  if (lane == 0) {
    for (int i = 0; i < R; ++i) mbar_init(&full[warp][i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  // weight stages (codes + group params: never written by a preceding kernel) go out first
  if (lane == 0)
    while (issued < R && issue(true)) {
    }
  pdl_launch_dependents();
  pdl_wait();

  // ---- stage x (B200 K order) for this CTA's K slice; zero the partials ----
  const int kb = kpos(a, a.ub[rank]), ke = kpos(a, a.ub[rank + 1]);
  const int ncols = ke - kb;
  for (int e = threadIdx.x; e < nj * kNW * redn; e += kNW * 32) red[e] = 0.f;
  {
    const T zero = from_f32<T>(0.f);
    const T* x = reinterpret_cast<const T*>(a.x);
    if (a.fast) {
      const int n8 = ncols >> 3;
      for (int e = threadIdx.x; e < a.n * n8; e += kNW * 32) {
        const int n = e / n8, c = (e - n * n8) << 3, kk = kb + c;
        uint4 v = make_uint4(0, 0, 0, 0);
        int col = -1;
        if (kk < a.m_pad) {
          if (kk < a.m) col = kk;
        } else if (kk - a.m_pad < a.k) {
          col = a.m + kk - a.m_pad;
        }
        if (col >= 0) v = *reinterpret_cast<const uint4*>(x + n * a.ldx + col);
        *reinterpret_cast<uint4*>(xs + n * a.xs_ld + c) = v;
      }
    } else {
      for (int e = threadIdx.x; e < a.n * ncols; e += kNW * 32) {
        const int n = e / ncols, c = e - n * ncols;
        const int col = a.colmap[kb + c];
        xs[n * a.xs_ld + c] = col >= 0 ? x[n * a.ldx + col] : zero;
      }
    }
  }
  __syncthreads();
  // per-(group, column) sums of x over the staged quantized columns: 16 lanes per pair,
  // fixed-order tree reduction (deterministic)
  const int gx0 = kb < a.m_pad ? kb / a.g : 0;
  const int qend = min(ke, a.m_pad);
  const int ngx = kb < a.m_pad ? (qend - gx0 * a.g + a.g - 1) / a.g : 0;
  {
    using T2 = typename DTraits<T>::T2;
    const int half = lane >> 4, l16 = lane & 15;
    // warp-uniform trip count (the shuffles need all 32 lanes); an odd tail half idles
    for (int p0 = warp * 2; p0 < ngx * a.n; p0 += kNW * 2) {
      const int p = p0 + half;
      const bool live = p < ngx * a.n;
      const int gi = live ? p / a.n : 0, n = live ? p - gi * a.n : 0;
      const int c_beg = (gx0 + gi) * a.g, c_end = live ? min(c_beg + a.g, qend) : c_beg;
      float sum = 0.f;
      for (int c = c_beg + l16 * 8; c < c_end; c += 128) {
        const uint4 v = lds128(xs + n * a.xs_ld + (c - kb));
        const T2* h = reinterpret_cast<const T2*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = t2_to_f2<T2>(h[q]);
          sum += f.x + f.y;
        }
      }
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (l16 == 0 && live) xsum[gi * NTS + n] = sum;
    }
  }
  __syncthreads();

  // ---- consume ----
  if (lane == 0)
    while (issued < R && issue(false)) {
    }
  int xrow[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xrow[nt] = min(g8 + 8 * nt, a.n - 1);
  const T* xlane[NT];  // this lane's staged x row, at its 16-column offset inside a step
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xlane[nt] = xs + xrow[nt] * a.xs_ld + 16 * t4 - kb;
  float acc[NT][4];
  auto zero4 = [](float (&v)[NT][4]) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) v[nt][e] = 0.f;
  };
  zero4(acc);

  auto bsel = [](const uint4& xa, const uint4& xb, int jj, uint32_t& b0, uint32_t& b1) {
    b0 = (jj == 0) ? xa.x : (jj == 1) ? xa.z : (jj == 2) ? xb.x : xb.z;
    b1 = (jj == 0) ? xa.y : (jj == 1) ? xa.w : (jj == 2) ? xb.y : xb.w;
  };
  // d += A fragments (one 64-column step) x the lane's 16 staged x columns at B200 column k
  auto mma_step = [&](const uint32_t (&f)[4][4], int k, float (&d)[NT][4]) {
    uint4 xa[NT], xb[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      xa[nt] = lds128(xlane[nt] + k);
      xb[nt] = lds128(xlane[nt] + k + 8);
    }
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t b0, b1;
        bsel(xa[nt], xb[nt], jj, b0, b1);
        mma16816<T>(d[nt], f[jj], b0, b1);
      }
  };
  // decode the 64-column step h (0/1) of the chunk at cp into (magic + code) A fragments
  auto decode_step = [&](const uint8_t* cp, int h, uint32_t (&f)[4][4]) {
    if constexpr (BITS == 4) {
      const uint4 qv = lds128(cp + h * 512 + lane * 16);
      decode4<T>(qv.x, f[0]);
      decode4<T>(qv.y, f[1]);
      decode4<T>(qv.z, f[2]);
      decode4<T>(qv.w, f[3]);
    } else {
      const uint2 q2 = lds64(cp + lane * 16 + h * 8);
      const uint32_t hbits = *reinterpret_cast<const uint32_t*>(cp + 512 + lane * 8 + h * 4);
      const uint32_t ww2[2] = {q2.x, q2.y};
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) f[jj][pp] = decode3_pair<T>(ww2[jj >> 1], hbits, 4 * (jj & 1) + pp, jj >> 1);
    }
  };
  // acc += s' * sum(c' x) + (z - magic s') * sum(x) for one group (sz16 pair at szp)
  auto fold = [&](const uint8_t* szp, int gx, const float (&gsum)[NT][4]) {
    constexpr float M = DTraits<T>::kMagicF;
    const uint2 p = lds64(szp + g8 * 8);
    const float2 r0 = __half22float2(*reinterpret_cast<const __half2*>(&p.x));
    const float2 r1 = __half22float2(*reinterpret_cast<const __half2*>(&p.y));
    const float s0 = r0.x;
    const float s1 = (BITS == 4 && DTraits<T>::kHiTrick) ? r1.x * (1.f / 16.f) : r1.x;
    const float z0 = fmaf(-M, s0, r0.y), z1 = fmaf(-M, s1, r1.y);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float2 sx = *reinterpret_cast<const float2*>(xsum + gx * NTS + 8 * nt + 2 * t4);
      acc[nt][0] = fmaf(s0, gsum[nt][0], fmaf(z0, sx.x, acc[nt][0]));
      acc[nt][1] = fmaf(s0, gsum[nt][1], fmaf(z0, sx.y, acc[nt][1]));
      acc[nt][2] = fmaf(s1, gsum[nt][2], fmaf(z1, sx.x, acc[nt][2]));
      acc[nt][3] = fmaf(s1, gsum[nt][3], fmaf(z1, sx.y, acc[nt][3]));
    }
  };
  auto park = [&](int jl) {  // this warp's partial of row-block jl -> shared memory
    float* rp = red + ((size_t)jl * kNW + warp) * redn;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = g8 + 8 * (e >> 1), col = 8 * nt + 2 * t4 + (e & 1);
        if (col < a.n) rp[row * a.n + col] = acc[nt][e];
      }
  };

  // steps per group (64-column steps): full codes stages hold 8 steps = 8 / GT groups
  constexpr int kSteps = 2 * kCPS;
  constexpr int kGPS = GT <= kSteps ? kSteps / GT : 1;
  int jl = warp / max(nst, 1), t = warp - jl * nst;  // stage (row-block, index) under this warp
  int cur_jl = jl;
  int slot = 0;
  uint32_t phase = 0;
  for (int i = 0; i < my_n; ++i) {
    if (jl != cur_jl) {  // this warp is done with row-block cur_jl
      park(cur_jl);
      zero4(acc);
      cur_jl = jl;
    }
    mbar_wait(&full[warp][slot], phase);
    const uint8_t* st = ring + slot * kStage;
    if (t < ncs) {
      const int ca = sl.c0 + t * kCPS, nck = min(kCPS, sl.c1 - ca);
      const int ga = GT == 1 ? 2 * ca : ca / HG;
      const int kc = ca * 128;  // B200 column of the stage's first code
      if (nck == kCPS && (GT <= kSteps)) {
        // full stage: 8 steps, one MMA chain per group, folded after the chain
        float d[kGPS][NT][4];
#pragma unroll
        for (int q = 0; q < kGPS; ++q) zero4(d[q]);
#pragma unroll
        for (int sidx = 0; sidx < kSteps; ++sidx) {
          uint32_t f[4][4];
          decode_step(st + (sidx >> 1) * CB, sidx & 1, f);
          mma_step(f, kc + sidx * 64, d[sidx / (GT <= kSteps ? GT : 1)]);
        }
#pragma unroll
        for (int q = 0; q < kGPS; ++q) {
          const int grp = (GT == 1 ? 2 * ca : ca / HG) + q;
          fold(st + kSzOff + (grp - ga) * 64, grp - gx0, d[q]);
        }
      } else {
        // partial stage (end of a slice) or very large groups: step by step
        float d[NT][4];
        zero4(d);
        for (int sidx = 0; sidx < 2 * nck; ++sidx) {
          uint32_t f[4][4];
          decode_step(st + (sidx >> 1) * CB, sidx & 1, f);
          mma_step(f, kc + sidx * 64, d);
          const int step = 2 * ca + sidx;  // global 64-column step
          if ((step % GT) == GT - 1 || step == 2 * a.nch - 1) {
            const int grp = step / GT;
            fold(st + kSzOff + (grp - ga) * 64, grp - gx0, d);
            zero4(d);
          }
        }
      }
    } else {
      const int wa = sl.w0 + (t - ncs) * kWPS, nwt = min(kWPS, sl.w1 - wa);
#pragma unroll
      for (int wt = 0; wt < kWPS; ++wt) {
        if (wt < nwt) {
          const T* w16 = reinterpret_cast<const T*>(st + wt * 2048);
          const uint4 r0a = lds128(w16 + g8 * 64 + 16 * t4);
          const uint4 r0b = lds128(w16 + g8 * 64 + 16 * t4 + 8);
          const uint4 r1a = lds128(w16 + (g8 + 8) * 64 + 16 * t4);
          const uint4 r1b = lds128(w16 + (g8 + 8) * 64 + 16 * t4 + 8);
          const uint32_t f[4][4] = {{r0a.x, r1a.x, r0a.y, r1a.y}, {r0a.z, r1a.z, r0a.w, r1a.w},
                                    {r0b.x, r1b.x, r0b.y, r1b.y}, {r0b.z, r1b.z, r0b.w, r1b.w}};
          mma_step(f, a.m_pad + (wa + wt) * 64, acc);
        }
      }
    }
    __syncwarp();  // every lane is done with the slot
    if (lane == 0)
      while (issued < i + 1 + R && issue(false)) {
      }
    if (++slot == R) {
      slot = 0;
      phase ^= 1u;
    }
    t += kNW;
    while (t >= nst) {
      t -= nst;
      ++jl;
    }
  }
  if (my_n > 0) park(cur_jl);
  __syncthreads();
  // ---- this CTA's slice partial of every row-block: sum the warps in order (into slot 0) ----
  for (int e = threadIdx.x; e < nj * redn; e += kNW * 32) {
    const int jl = e / redn, r = e - jl * redn;
    const float* p = red + (size_t)jl * kNW * redn + r;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kNW; ++w) v += p[w * redn];
    red[(size_t)jl * kNW * redn + r] = v;
  }
  // ---- sum the S slices (ranks in order, over DSMEM) and store y ----
  if (a.S > 1) cluster_sync();
  else __syncthreads();
  for (int e = threadIdx.x; e < nj * redn; e += kNW * 32) {
    const int jl = e / redn, r = e - jl * redn;
    if (a.S > 1 && (jl % a.S) != rank) continue;
    const uint32_t off = smem_u32(red + (size_t)jl * kNW * redn + r);
    float v = 0.f;
    for (int q = 0; q < a.S; ++q) v += a.S > 1 ? ld_dsmem_f32(off, q) : red[(size_t)jl * kNW * redn + r];
    const int row16 = r / a.n, col = r - row16 * a.n;
    int lrb;
    const int l = layer_of(a, j0 + jl, lrb);
    const int row = lrb * 16 + row16;
    if (row < a.ocs[l]) {
      const int64_t idx = (int64_t)col * a.ldy + row;
      if (a.yflags & QEFT_Y_F32) {
        float* py = (float*)a.ys[l] + idx;
        *py = (a.yflags & QEFT_Y_ACCUMULATE) ? *py + v : v;
      } else {
        T* py = (T*)a.ys[l] + idx;
        *py = from_f32<T>((a.yflags & QEFT_Y_ACCUMULATE) ? to_f32<T>(*py) + v : v);
      }
    }
  }
  if (a.S > 1) cluster_sync();  // keep this CTA's partials alive until every rank has read them
}

// ---------------------------------------------------------------------------
// host: slicing and launch

// balance units (codes units then weak tiles) into S contiguous slices by bytes
void slice_units(int nuc, int U, int nch, int nwt, int cb, int szb, int S, int* ub) {
  const int nu = nuc + nwt;
  auto ubytes = [&](int u) -> double {
    if (u < nuc) {
      const int ch = std::min(U, nch - u * U);
      return (double)ch * cb + szb;
    }
    return 2048.0;
  };
  double total = 0;
  for (int u = 0; u < nu; ++u) total += ubytes(u);
  ub[0] = 0;
  double accb = 0;
  int u = 0;
  for (int s = 1; s < S; ++s) {
    const double target = total * s / S;
    while (u < nu && accb + 0.5 * ubytes(u) < target) accb += ubytes(u++);
    ub[s] = std::max(u, ub[s - 1]);
  }
  ub[S] = nu;
}

int kpos_host(int u, int nuc, int U, int nch, int m_pad) {
  return u <= nuc ? std::min(u * U, nch) * 128 : m_pad + (u - nuc) * 64;
}

template <int BITS, int NT, int GT, typename T, int R, int NW, int CPS>
int launch2(G2Args a, const qeft_linear_t* L, cudaStream_t st) {
  constexpr int kNW = NW, kStage = CPS * 1152;
  auto kern = gemv2_kernel<BITS, NT, GT, T, R, NW, CPS>;
  constexpr int kSmemMax = 227 * 1024 - 1024;
  static bool attr = false;
  if (!attr) {
    QEFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
    QEFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    QEFT_CUDA(cudaGetDevice(&dev));
    QEFT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int cb = BITS == 4 ? 1024 : 768;
  const int szb = 64 * std::max(1, a.U * 128 / a.g);
  const int nwt = a.k_pad / 64;
  const int rings = kNW * R * kStage;
  const int force_s = env_int("QEFT_GEMV2_S", 0);
  // choose the cluster size S (= K slices): the busiest CTA streams J row-blocks of its slice
  double best = 1e300;
  G2Args bestA = a;
  int best_grid = 0;
  size_t best_smem = 0;
  for (int S = 1; S <= kMaxS; ++S) {
    if (force_s && S != force_s) continue;
    if (S > a.nuc + nwt) break;
    G2Args b = a;
    b.S = S;
    slice_units(a.nuc, a.U, a.nch, nwt, cb, szb, S, b.ub);
    bool empty = false;
    double smax = 0;
    int xc = 0, xg = 0;
    for (int s = 0; s < S; ++s) {
      empty |= b.ub[s + 1] == b.ub[s];
      const int kb = kpos_host(b.ub[s], a.nuc, a.U, a.nch, a.m_pad), ke = kpos_host(b.ub[s + 1], a.nuc, a.U, a.nch, a.m_pad);
      xc = std::max(xc, ke - kb);
      if (kb < a.m_pad) xg = std::max(xg, (std::min(ke, a.m_pad) - kb / a.g * a.g + a.g - 1) / a.g);
      const int c0 = std::min(std::min(b.ub[s], a.nuc) * a.U, a.nch), c1 = std::min(std::min(b.ub[s + 1], a.nuc) * a.U, a.nch);
      const int w0 = std::max(b.ub[s], a.nuc) - a.nuc, w1 = std::max(b.ub[s + 1], a.nuc) - a.nuc;
      smax = std::max(smax, (double)(c1 - c0) * cb + (double)(c1 - c0) * 128 / a.g * 64 + (w1 - w0) * 2048.0);
    }
    if (empty) continue;
    b.xs_ld = xc + 8;  // 16 B skew between staged x rows
    // clusters that fit on the GPU at once (persistent: one wave)
    int nclu = sms / S;
    size_t smem = 0;
    for (int it = 0; it < 3; ++it) {
      b.J = (a.n_rb + nclu - 1) / nclu;
      if (b.J > kMaxJ) break;
      smem = (size_t)rings + (size_t)b.J * kNW * 16 * a.n * 4 + (size_t)a.n * b.xs_ld * 2 + (size_t)xg * NT * 8 * 4;
      if (smem > (size_t)kSmemMax) break;
      if (S > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nclu * S);
        cfg.blockDim = dim3(kNW * 32);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = S;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int maxc = 0;
        if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) != cudaSuccess || maxc <= 0) {
          cudaGetLastError();
          smem = 0;
          break;
        }
        if (maxc >= nclu) break;
        nclu = maxc;
      } else {
        break;
      }
    }
    if (b.J > kMaxJ || smem == 0 || smem > (size_t)kSmemMax) continue;
    const int ncl = (a.n_rb + b.J - 1) / b.J;
    const double cost = b.J * smax + (S > 1 ? 8192.0 : 0.0);  // + the DSMEM reduction
    if (cost < best * 0.98) {
      best = cost;
      bestA = b;
      best_grid = ncl * S;
      best_smem = smem;
    }
  }
  if (best_grid == 0) return -1;  // partials do not fit shared memory: the generic kernel serves it
  if (bestA.S > 1) {
    QEFT_CUDA(launch_pdl_cluster(kern, dim3(best_grid), dim3(kNW * 32), best_smem, st, bestA.S, bestA));
  } else {
    QEFT_CUDA(launch_pdl(kern, dim3(best_grid), dim3(kNW * 32), best_smem, st, bestA));
  }
  return 0;
}

template <int BITS, typename T>
int dispatch2(const G2Args& a, const qeft_linear_t* L, int gt, cudaStream_t st) {
  const bool nt2 = a.n > 8;
  if constexpr (BITS == 4 && std::is_same<T, __half>::value) {
    // tuning variants of the 7B decode path (4-bit, g = 128, <= 8 columns)
    static const int var = env_int("QEFT_GEMV2_VAR", 0);
    if (!nt2 && gt == 2 && var) {
      switch (var) {
        case 1: return launch2<4, 1, 2, T, 2, 16, 4>(a, L, st);
        case 2: return launch2<4, 1, 2, T, 2, 8, 8>(a, L, st);
        case 3: return launch2<4, 1, 2, T, 2, 12, 4>(a, L, st);
        default: break;
      }
    }
  }
#define QEFT_G2(NT)                                                  \
  switch (gt) {                                                      \
    case 1: return launch2<BITS, NT, 1, T, 3, 8, 4>(a, L, st);       \
    case 2: return launch2<BITS, NT, 2, T, 3, 8, 4>(a, L, st);       \
    case 4: return launch2<BITS, NT, 4, T, 3, 8, 4>(a, L, st);       \
    default: return launch2<BITS, NT, 8, T, 3, 8, 4>(a, L, st);      \
  }
  if (nt2) {
    QEFT_G2(2)
  } else {
    QEFT_G2(1)
  }
#undef QEFT_G2
}

}  // namespace

namespace qeft {

bool gemv2_supported(const qeft_linear_t* L, int n) {
  if (L->sz16 == nullptr || env_int("QEFT_GEMV_V1", 0)) return false;
  if (L->g % 64 != 0) return false;
  const int gt = L->g / 64;
  return (gt == 1 || gt == 2 || gt == 4 || gt == 8) && n >= 1 && n <= 16 && L->m > 0;
}

size_t gemv2_workspace_bytes(const qeft_linear_t*, int) { return 0; }

int gemv2_multi(const qeft_linear_t* const* Ls, int nl, const void* x, int64_t ldx, void* const* ys, int64_t ldy,
                int y_f32, int n, void*, size_t, cudaStream_t st) {
  const qeft_linear_t* L = Ls[0];
  G2Args a{};
  a.nl = nl;
  int rb_total = 0;
  for (int l = 0; l < nl; ++l) {
    const qeft_linear_t* Li = Ls[l];
    QEFT_CHECK(Li->sz16 != nullptr, QEFT_ERR_LAYOUT, "gemv: layer %d has no sz16", l);
    a.qw[l] = (const uint8_t*)Li->qweight;
    a.sz[l] = (const uint8_t*)Li->sz16;
    a.wk[l] = (const uint8_t*)Li->weak16;
    a.ys[l] = ys[l];
    a.ocs[l] = Li->oc;
    rb_total += Li->oc_pad / 16;
    a.rb_end[l] = rb_total;
  }
  a.x = x;
  a.ldx = ldx;
  a.colmap = L->colmap;
  a.fast = (L->flags & QEFT_FLAG_STRUCTURED_FAST) && (ldx % 8 == 0) && (((uintptr_t)x & 15) == 0);
  a.ldy = ldy;
  a.yflags = y_f32;
  a.m = L->m;
  a.m_pad = L->m_pad;
  a.k = L->k;
  a.k_pad = L->k_pad;
  a.g = L->g;
  a.n = n;
  a.n_rb = rb_total;
  a.nch = L->m_pad / 128;
  a.U = std::max(1, L->g / 128);
  a.nuc = (a.nch + a.U - 1) / a.U;
  a.ng16 = (L->m_pad + L->g - 1) / L->g;
  a.rbb = rowblock_bytes(L->bits, L->m_pad);
  const int gt = L->g / 64;
  const bool bf = L->act_dtype == QEFT_BF16;
  if (L->bits == 4) return bf ? dispatch2<4, __nv_bfloat16>(a, L, gt, st) : dispatch2<4, __half>(a, L, gt, st);
  return bf ? dispatch2<3, __nv_bfloat16>(a, L, gt, st) : dispatch2<3, __half>(a, L, gt, st);
}

}  // namespace qeft
