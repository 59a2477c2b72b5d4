#pragma once
// Decode GEMV, bulk-copy warp rings: the HBM-bound hot kernel of the decode path.
//
// Replaces the reference's matvec paths (pkg/src/qeft/kernels.py:66-157,
// `_grouped_accumulate`): y = sum_g s_g * (c_g . x_g) + z_g * sum(x_g) + W_weak . x_weak,
// for 1..16 activation columns and up to 3 layers that read the same x (q/k/v, gate/up).
//
// Why this shape (measured on B200, scripts/micro/bulk_warp_bench.cu, profiles/r02):
//   * every warp owns a private ring of R stages fed by its OWN lane 0 with 1-D bulk copies
//     (cp.async.bulk, the TMA engine) completing on an mbarrier: 8-16 warps x 2-3 x 4 KB per
//     SM stream 6.9-7.0 TB/s. No per-lane address arithmetic, no producer/consumer handshake
//     across warps: a warp waits on its own barrier, decodes, multiplies, and refills.
//   * work split: a thread-block cluster of S CTAs owns a contiguous run of row-blocks (16
//     output rows each); CTA rank r streams K slice r of every one of them (slices are whole
//     groups, balanced by bytes; S = 1 unless the row-blocks do not spread evenly over the
//     SMs). Inside a CTA the run's stages (4 KB each) are dealt to the warps round-robin.
//     Partials go to shared memory; at the end the warp partials and then the S slice
//     partials (over DSMEM) are summed in a fixed order: deterministic, no atomics, no
//     global scratch.
//   * x is staged once per CTA for its K slice only (gathered through the column map for
//     irregular / online layouts, so no separate gather launch), with the per-(group,
//     column) sums of x that the zero-point fold needs.
//   * codes become (magic + code) half2 A fragments with one LOP3 each (qeft_common.cuh
//     decode4 / decode3_pair) for mma.sync m16n8k16 (x is the B operand: 8 columns per MMA
//     at no extra cost); one MMA chain per group, then the group is folded as
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


namespace qeft {
namespace g2 {

constexpr int kMaxS = 4;   // K slices = cluster size
constexpr int kMaxL = 3;   // layers per launch
constexpr int kMaxJ = 48;  // row-blocks per cluster (partials live in shared memory)

inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// one K slice, precomputed on the host: codes chunks [c0, c1), weak tiles [w0, w1), staged
// B200 columns [kb, ke), x-sum groups [gx0, gx0 + ngx), codes / total stages per row-block
struct SliceGeo {
  int c0, c1, w0, w1, kb, ke, gx0, ngx, ncs, nst;
};

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
  int ng16;  // sz16 groups per row-block
  int S;     // K slices (cluster size)
  SliceGeo geo[kMaxS];
  int J;        // row-blocks per cluster
  int xs_ld;    // staged x row stride (elements)
  int64_t rbb;  // qweight bytes per row-block
  int ic;        // input columns (the raw x row staged for column-map gathers)
  int l2pf;      // L2-prefetch each warp's first codes stage before the PDL wait
  const void* xu;      // fused SwiGLU input (model.py:389-391): x = silu(x) * xu (structured layers)
  int xu_off;          // byte offset of the staged xu rows in shared memory
  const float* ngain;  // fused RMS-norm of x (model.py:249-256): gain [ic] fp32, or null
  int nthr;            // the stand-alone rmsnorm kernel's block size (its reduction order is kept)
  int xraw_off;  // byte offset of the raw x rows in shared memory (0: gather from global memory)
  int contig;   // stages dealt to warps as contiguous runs (partials: J + NW slots) instead of
                // round-robin (J x NW slots)
  unsigned long long* trace;  // profiling only (qeft_gemv_trace): per-CTA timestamps, or null
};

// per (bits, activation dtype) launchers, one translation unit each (qeft_gemv2_{4,3}{h,b}.cu)
int dispatch_4h(const G2Args& a, int gt, cudaStream_t st);
int dispatch_4b(const G2Args& a, int gt, cudaStream_t st);
int dispatch_3h(const G2Args& a, int gt, cudaStream_t st);
int dispatch_3b(const G2Args& a, int gt, cudaStream_t st);
}  // namespace g2
}  // namespace qeft

#ifdef QEFT_GEMV2_KERNELS
namespace {
using namespace qeft::g2;

QEFT_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

QEFT_DEV int layer_of(const G2Args& a, int j, int& lrb) {
  int l = 0;
  while (l + 1 < a.nl && j >= a.rb_end[l]) ++l;
  lrb = j - (l ? a.rb_end[l - 1] : 0);
  return l;
}

// contiguous dealing: warp w streams stages [w * total / NW, (w + 1) * total / NW); the warp
// holding stage s is the last one starting at or before s
QEFT_DEV int run_start(int w, int total, int nw) { return (int)((int64_t)w * total / nw); }
QEFT_DEV int warp_of_stage(int s, int total, int nw) {
  int w = (int)(((int64_t)s * nw) / max(total, 1));
  while (w > 0 && run_start(w, total, nw) > s) --w;
  while (w + 1 < nw && run_start(w + 1, total, nw) <= s) ++w;
  return w;
}

QEFT_DEV uint4 lds128(const void* p) { return *reinterpret_cast<const uint4*>(p); }
QEFT_DEV uint2 lds64(const void* p) { return *reinterpret_cast<const uint2*>(p); }

// Launch shape (template): NW warps per CTA, CPS 128-column chunks per codes stage (a stage
// holds CPS KB of 4-bit codes + their sz16 pairs, or CPS / 2 weak tiles), R stages per ring.
// ONE: a single activation column (batch-1 decode): only column 0 of the MMA output is live.
// FUSED: the decode step's RMS-norm / SwiGLU in the x staging (separate instantiations, so the
// plain kernel carries none of it)
template <int BITS, int NT, int GT, typename T, int R, int NW, int CPS, bool ONE, int MINB, int PRE, bool CONTIG,
          bool FUSED = false>
__global__ void __launch_bounds__(NW * 32, MINB) gemv2_kernel(const G2Args a) {
  constexpr int kWPS = CPS / 2;
  constexpr int kSzOff = CPS * 1024, kStage = CPS * 1152;  // codes, then sz16 pairs
  constexpr int NTS = NT * 8;                               // x-sum column stride
  constexpr int CB = BITS == 4 ? 1024 : 768;                // bytes per 128-column chunk
  constexpr int HG = GT >= 2 ? GT / 2 : 1;                  // chunks per group (GT >= 2)
  static_assert(GT <= 2 * CPS && (2 * CPS) % GT == 0, "a full stage must hold whole groups");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[NW][R];
  __shared__ __align__(8) uint64_t xbar;  // x staging (bulk copies)
  __shared__ __align__(8) uint64_t xsbar;  // the per-group x sums are complete
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int rank = a.S > 1 ? (int)cluster_ctarank() : 0;
  const int clu = a.S > 1 ? blockIdx.x / a.S : blockIdx.x;
  const int n = ONE ? 1 : a.n;
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtime();

  // shared memory: [rings][partials red: J x NW x 16 x n floats][x: n x xs_ld][x sums]
  uint8_t* ring = smem + (size_t)warp * R * kStage;
  float* red = reinterpret_cast<float*>(smem + (size_t)NW * R * kStage);
  const int redn = 16 * n;  // floats per (row-block, warp)
  T* xs = reinterpret_cast<T*>(red + (size_t)(CONTIG ? a.J + NW : a.J * NW) * redn);
  float* xsum = reinterpret_cast<float*>(xs + (size_t)n * a.xs_ld);

  // this CTA: row-blocks [j0, j0 + nj) of the cluster, K slice `rank`; stages of row-block jl
  // are jl * nst .. jl * nst + nst - 1 (codes stages, then weak stages); warp w takes w, w + NW..
  const SliceGeo sg = a.geo[rank];
  const int j0 = clu * a.J, nj = max(min(a.J, a.n_rb - j0), 0);
  const int ncs = sg.ncs, nst = sg.nst;
  const int total = nj * nst;
  const int s_beg = CONTIG ? run_start(warp, total, NW) : warp;
  const int my_n = CONTIG ? run_start(warp + 1, total, NW) - s_beg
                            : (warp < total ? (total - warp + NW - 1) / NW : 0);
  const int sstep = CONTIG ? 1 : NW;
  const int nslot = CONTIG ? nj + NW : nj * NW;  // partial slots (redn floats each)

  // ---- lane 0: bulk-copy issue (stage i of this warp = global stage warp + i * NW) ----
  int issued = 0;
  int is_jl = s_beg / nst, is_t = s_beg - is_jl * nst;
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
      const int ca = sg.c0 + is_t * CPS, cb = min(ca + CPS, sg.c1);
      const int ga = GT == 1 ? 2 * ca : ca / HG;
      const int gb = GT == 1 ? 2 * cb : (cb + HG - 1) / HG;
      const uint32_t cbytes = (uint32_t)(cb - ca) * CB, sbytes = (uint32_t)(gb - ga) * 64;
      mbar_expect_tx(bar, cbytes + sbytes);
      bulk_g2s(dst, pq + ca * CB, cbytes, bar);
      bulk_g2s(dst + kSzOff, ps + ga * 64, sbytes, bar);
    } else {
      const int wa = sg.w0 + (is_t - ncs) * kWPS, wb = min(wa + kWPS, sg.w1);
      const uint32_t bytes = (uint32_t)(wb - wa) * 2048;
      mbar_expect_tx(bar, bytes);
      bulk_g2s(dst, pw + wa * 2048, bytes, bar);
    }
    ++issued;
    is_t += sstep;
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
    if (warp == 0) {
      mbar_init(&xbar, 1);
      mbar_init(&xsbar, NW);  // every warp computes a share of the x sums
    }
    fence_mbar_init();
  }
  __syncwarp();
  // PRE > 0: weight stages (codes + group params, never written by a preceding kernel) go out
  // before the PDL wait -- worth it only when this CTA can start beside the previous kernel's
  pdl_launch_dependents();
  if constexpr (PRE > 0) {
    if (lane == 0)
      while (issued < PRE && issue(true)) {
      }
  } else {
    // the first codes stage of this warp toward L2 (frozen data; the smem copy and the x copy
    // are issued after the wait)
    if (lane == 0)
      for (int i = 0; i < a.l2pf && i < my_n; ++i) {
        const int sidx = s_beg + i * sstep, jl_i = sidx / nst, t_i = sidx - jl_i * nst;
        if (t_i >= ncs) continue;
        int lrb;
        const int l = layer_of(a, j0 + jl_i, lrb);
        const int ca = sg.c0 + t_i * CPS, cb = min(ca + CPS, sg.c1);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.qw[l] + lrb * a.rbb + ca * CB),
                     "r"((uint32_t)(cb - ca) * CB)
                     : "memory");
      }
  }
  if (tr && threadIdx.x == 0) tr[7] = gtime();
  pdl_wait();  // (xbar is initialised and armed by thread 0 itself; the others touch it only after
               // the staging barrier below)
  if (tr && threadIdx.x == 0) tr[1] = gtime();

  // ---- stage x (B200 K order) for this CTA's K slice; zero the partials ----
  const int kb = sg.kb, ncols = sg.ke - sg.kb;
  for (int e = threadIdx.x; e < nslot * redn; e += NW * 32) red[e] = 0.f;
  {
    const T zero = from_f32<T>(0.f);
    const T* x = reinterpret_cast<const T*>(a.x);
    if (a.fast) {
      // structured layout: the slice's x is (at most) two contiguous runs per row -- quantized
      // columns [kb, min(ke, m)) and weak columns -- moved by bulk copies; padding zeroed here
      const int q1 = min(sg.ke, a.m);
      const int w_beg = max(kb, a.m_pad), w_end = min(sg.ke, a.m_pad + a.k);
      if (threadIdx.x == 0) {
        const uint32_t bytes =
            (uint32_t)n * 2u * (uint32_t)(max(q1 - kb, 0) + max(w_end - w_beg, 0));
        if (bytes) {
          T* xus = reinterpret_cast<T*>(smem + a.xu_off);
          const T* xu = reinterpret_cast<const T*>(a.xu);
          mbar_expect_tx(&xbar, (FUSED && a.xu) ? 2 * bytes : bytes);
          for (int r = 0; r < n; ++r) {
            if (q1 > kb) bulk_g2s(xs + r * a.xs_ld, x + r * a.ldx + kb, (uint32_t)(q1 - kb) * 2u, &xbar);
            if (w_end > w_beg)
              bulk_g2s(xs + r * a.xs_ld + (w_beg - kb), x + r * a.ldx + a.m + (w_beg - a.m_pad),
                       (uint32_t)(w_end - w_beg) * 2u, &xbar);
            if (FUSED && a.xu) {
              if (q1 > kb) bulk_g2s(xus + r * a.xs_ld, xu + r * a.ldx + kb, (uint32_t)(q1 - kb) * 2u, &xbar);
              if (w_end > w_beg)
                bulk_g2s(xus + r * a.xs_ld + (w_beg - kb), xu + r * a.ldx + a.m + (w_beg - a.m_pad),
                         (uint32_t)(w_end - w_beg) * 2u, &xbar);
            }
          }
        } else {
          mbar_arrive(&xbar);
        }
      }
      __syncthreads();  // x goes into the copy queue ahead of the weight stream
      if (lane == 0)
        while (issued < R && issue(false)) {
        }
      // zero padding: quantized [m, m_pad) and weak [m_pad + k, m_pad + k_pad) inside the slice
      const int z0a = max(kb, a.m), z0b = min(sg.ke, a.m_pad);
      const int z1a = max(kb, a.m_pad + a.k), z1b = sg.ke;
      const int nz0 = max(z0b - z0a, 0), nz1 = max(z1b - z1a, 0);
      for (int e = threadIdx.x; e < n * (nz0 + nz1); e += NW * 32) {
        const int r = ONE ? 0 : e / (nz0 + nz1), c = e - r * (nz0 + nz1);
        xs[r * a.xs_ld + (c < nz0 ? z0a + c : z1a + c - nz0) - kb] = zero;
      }
      mbar_wait(&xbar, 0);
      if (FUSED && a.xu) {
        // SwiGLU in place, the stand-alone kernel's expression (bit-identical): x = silu(g) * u
        const T* xus = reinterpret_cast<const T*>(smem + a.xu_off);
        const int nq = max(q1 - kb, 0), nw = max(w_end - w_beg, 0);
        for (int e = threadIdx.x; e < n * (nq + nw); e += NW * 32) {
          const int r = ONE ? 0 : e / (nq + nw), c = e - r * (nq + nw);
          const int o = r * a.xs_ld + (c < nq ? c : (w_beg - kb) + (c - nq));
          const float gv = to_f32<T>(xs[o]);
          xs[o] = from_f32<T>(gv / (1.f + __expf(-gv)) * to_f32<T>(xus[o]));
        }
      }
      if (tr && threadIdx.x == 0) tr[5] = gtime();
    } else if (a.xraw_off) {
      // column map (irregular / online layouts): the raw x rows land in shared memory by bulk
      // copy (ahead of the weight stream), the column map is read meanwhile, then the gather
      // runs shared -> shared
      T* xraw = reinterpret_cast<T*>(smem + a.xraw_off);
      const int icp = (a.ic + 7) & ~7;
      if (threadIdx.x == 0) {
        mbar_expect_tx(&xbar, (uint32_t)n * a.ic * 2u);
        for (int r = 0; r < n; ++r) bulk_g2s(xraw + r * icp, x + r * a.ldx, (uint32_t)a.ic * 2u, &xbar);
      }
      __syncthreads();  // x goes into the copy queue ahead of the weight stream
      if (lane == 0)
        while (issued < R && issue(false)) {
        }
      constexpr int kPer = 12;  // columns per thread held in registers while x lands
      const int nthr = NW * 32;
      int cols[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int c = threadIdx.x + u * nthr;
        cols[u] = c < ncols ? a.colmap[kb + c] : -1;
      }
      mbar_wait(&xbar, 0);
      for (int r = 0; r < n; ++r) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int c = threadIdx.x + u * nthr;
          if (c < ncols) xs[r * a.xs_ld + c] = cols[u] >= 0 ? xraw[r * icp + cols[u]] : zero;
        }
        for (int c = threadIdx.x + kPer * nthr; c < ncols; c += nthr) {
          const int col = a.colmap[kb + c];
          xs[r * a.xs_ld + c] = col >= 0 ? xraw[r * icp + col] : zero;
        }
      }
    } else {
      if (lane == 0)
        while (issued < R && issue(false)) {
        }
      // column map (irregular / online layouts): gather, 4 loads in flight per thread
      const int tot = n * ncols;
      for (int e0 = threadIdx.x; e0 < tot; e0 += 4 * NW * 32) {
        int col[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * NW * 32;
          const int r = ONE ? 0 : e / ncols, c = e - r * ncols;
          col[u] = e < tot ? a.colmap[kb + c] : -1;
        }
        T v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * NW * 32;
          const int r = ONE ? 0 : e / ncols;
          v[u] = col[u] >= 0 ? x[r * a.ldx + col[u]] : zero;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * NW * 32;
          const int r = ONE ? 0 : e / ncols, c = e - r * ncols;
          if (e < tot) xs[r * a.xs_ld + c] = v[u];
        }
      }
    }
  }
  __syncthreads();
  if (FUSED && a.ngain) {
    // fused RMS-norm of the staged x, bit-identical to qeft_rmsnorm_fwd: the first nthr threads
    // sum x^2 in that kernel's order (8 consecutive columns per thread, stride nthr * 8, warp
    // shuffles, then across warps), read from the staged row when it holds every column
    // (structured, one K slice), else from the raw row / global x; then y = gain * x * rstd.
    __shared__ float s_nred[32];
    __shared__ float s_rstd[16];
    const T* xg = reinterpret_cast<const T*>(a.x);
    const T* xraw = reinterpret_cast<const T*>(smem + a.xraw_off);
    const int icp = (a.ic + 7) & ~7;
    const bool from_xs = a.fast && a.S == 1;
    for (int r = 0; r < n; ++r) {
      float ss = 0.f;
      if ((int)threadIdx.x < a.nthr) {
        for (int c = threadIdx.x * 8; c < a.ic; c += a.nthr * 8) {
          uint4 v;
          if (from_xs) v = lds128(xs + r * a.xs_ld + (c < a.m ? c : a.m_pad + (c - a.m)) - kb);
          else if (a.xraw_off) v = lds128(xraw + r * icp + c);
          else v = *reinterpret_cast<const uint4*>(xg + r * a.ldx + c);
          const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float f = to_f32<T>(e[i]);
            ss += f * f;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) s_nred[warp] = ss;
      __syncthreads();
      if (threadIdx.x < 32) {
        float v = (int)threadIdx.x < (a.nthr >> 5) ? s_nred[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) s_rstd[r] = rsqrtf(v / (float)a.ic + 1e-5f);
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < n * ncols; e += NW * 32) {
      const int r = ONE ? 0 : e / ncols, c = e - r * ncols, p = kb + c;
      int col;
      if (a.fast) col = p < a.m ? p : ((p >= a.m_pad && p < a.m_pad + a.k) ? a.m + (p - a.m_pad) : -1);
      else col = a.colmap[p];
      if (col >= 0) xs[r * a.xs_ld + c] = from_f32<T>(a.ngain[col] * to_f32<T>(xs[r * a.xs_ld + c]) * s_rstd[r]);
    }
    __syncthreads();
  }
  // per-(group, column) sums of x over the staged quantized columns: 16 lanes per pair,
  // fixed-order tree reduction (deterministic)
  const int gx0 = sg.gx0, ngx = sg.ngx;
  {
    using T2 = typename DTraits<T>::T2;
    const int half = lane >> 4, l16 = lane & 15;
    const int qend = min(sg.ke, a.m_pad);
    // warp-uniform trip count (the shuffles need all 32 lanes); an odd tail half idles. No CTA
    // barrier after it: each warp arrives on xsbar and waits for it only before its first fold
    // (so it refills its ring and starts its first MMA chain meanwhile). (4 summing warps for
    // one column measured 4 % slower: the sums then arrive later than the first folds.)
    constexpr int XW = NW;
    for (int p0 = warp * 2; warp < XW && p0 < ngx * n; p0 += XW * 2) {
      const int p = p0 + half;
      const bool live = p < ngx * n;
      const int gi = !live ? 0 : ONE ? p : p / n, r = live && !ONE ? p - gi * n : 0;
      const int c_beg = (gx0 + gi) * a.g, c_end = live ? min(c_beg + a.g, qend) : c_beg;
      float sum = 0.f;
      for (int c = c_beg + l16 * 8; c < c_end; c += 128) {
        const uint4 v = lds128(xs + r * a.xs_ld + (c - kb));
        const T2* h = reinterpret_cast<const T2*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = t2_to_f2<T2>(h[q]);
          sum += f.x + f.y;
        }
      }
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (l16 == 0 && live) xsum[gi * NTS + r] = sum;
    }
    if (warp < XW) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&xsbar);
    }
  }
  bool xs_ready = false;
  if (tr && threadIdx.x == 0) tr[2] = gtime();

  // ---- consume ----
  if (lane == 0)
    while (issued < R && issue(false)) {
    }
  const T* xlane[NT];  // this lane's staged x row, at its 16-column offset inside a step
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xlane[nt] = xs + min(g8 + 8 * nt, n - 1) * a.xs_ld + 16 * t4 - kb;
  const float* xsl = xsum + 2 * t4 - gx0 * NTS;  // this lane's x-sum columns, by group
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
  // acc += s' * sum(c' x) + (z - magic s') * sum(x) for group grp (sz16 pair at szp)
  auto fold = [&](const uint8_t* szp, int grp, const float (&gsum)[NT][4]) {
    constexpr float M = DTraits<T>::kMagicF;
    if (!xs_ready) {
      mbar_wait(&xsbar, 0);
      xs_ready = true;
    }
    const uint2 p = lds64(szp + g8 * 8);
    const float2 r0 = __half22float2(*reinterpret_cast<const __half2*>(&p.x));
    const float2 r1 = __half22float2(*reinterpret_cast<const __half2*>(&p.y));
    const float s0 = r0.x;
    const float s1 = (BITS == 4 && DTraits<T>::kHiTrick) ? r1.x * (1.f / 16.f) : r1.x;
    const float z0 = fmaf(-M, s0, r0.y), z1 = fmaf(-M, s1, r1.y);
    if constexpr (ONE) {  // column 0 only (lanes t4 == 0 carry it; the others are discarded)
      const float sx = xsl[grp * NTS];
      acc[0][0] = fmaf(s0, gsum[0][0], fmaf(z0, sx, acc[0][0]));
      acc[0][2] = fmaf(s1, gsum[0][2], fmaf(z1, sx, acc[0][2]));
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float2 sx = *reinterpret_cast<const float2*>(xsl + grp * NTS + 8 * nt);
        acc[nt][0] = fmaf(s0, gsum[nt][0], fmaf(z0, sx.x, acc[nt][0]));
        acc[nt][1] = fmaf(s0, gsum[nt][1], fmaf(z0, sx.y, acc[nt][1]));
        acc[nt][2] = fmaf(s1, gsum[nt][2], fmaf(z1, sx.x, acc[nt][2]));
        acc[nt][3] = fmaf(s1, gsum[nt][3], fmaf(z1, sx.y, acc[nt][3]));
      }
    }
  };
  // NCK whole chunks starting at chunk ca, straight-line: one MMA chain per group, then folds
  auto codes_stage = [&](auto nck_c, const uint8_t* st, int ca) {
    constexpr int NCK = decltype(nck_c)::value;
    constexpr int NG = 2 * NCK / GT;
    const int ga = GT == 1 ? 2 * ca : ca / HG;
    float d[NG][NT][4];
#pragma unroll
    for (int q = 0; q < NG; ++q) zero4(d[q]);
#pragma unroll
    for (int s = 0; s < 2 * NCK; ++s) {
      uint32_t f[4][4];
      decode_step(st + (s >> 1) * CB, s & 1, f);
      mma_step(f, ca * 128 + s * 64, d[s / GT]);
    }
#pragma unroll
    for (int q = 0; q < NG; ++q) fold(st + kSzOff + q * 64, ga + q, d[q]);
  };
  auto park = [&](int jl) {  // this warp's partial of row-block jl -> shared memory
    float* rp = red + (size_t)(CONTIG ? jl + warp : jl * NW + warp) * redn;
    if constexpr (ONE) {
      if (t4 == 0) {
        rp[g8] = acc[0][0];
        rp[g8 + 8] = acc[0][2];
      }
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = g8 + 8 * (e >> 1), col = 8 * nt + 2 * t4 + (e & 1);
          if (col < n) rp[row * n + col] = acc[nt][e];
        }
    }
  };

  int jl = s_beg / nst, t = s_beg - jl * nst;  // stage (row-block, index) under this warp
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
    if (tr && threadIdx.x == 0 && i == 0) tr[3] = gtime();
    const uint8_t* st = ring + slot * kStage;
    if (t < ncs) {
      const int ca = sg.c0 + t * CPS, nck = min(CPS, sg.c1 - ca);
      if (nck == CPS) {
        codes_stage(std::integral_constant<int, CPS>{}, st, ca);
      } else if (GT <= 2 || (nck % HG) == 0) {
        // end of a slice (whole groups): straight-line code per chunk count
        switch (nck) {
          case 1: if constexpr (GT <= 2) codes_stage(std::integral_constant<int, 1>{}, st, ca); break;
          case 2: if constexpr (GT <= 4 && 2 < CPS) codes_stage(std::integral_constant<int, 2>{}, st, ca); break;
          case 3: if constexpr (GT <= 2 && 3 < CPS) codes_stage(std::integral_constant<int, 3>{}, st, ca); break;
          case 4: if constexpr (4 < CPS) codes_stage(std::integral_constant<int, (4 < CPS ? 4 : 1)>{}, st, ca); break;
          case 5: if constexpr (GT <= 2 && 5 < CPS) codes_stage(std::integral_constant<int, (5 < CPS ? 5 : 1)>{}, st, ca); break;
          case 6: if constexpr (GT <= 4 && 6 < CPS) codes_stage(std::integral_constant<int, (6 < CPS ? 6 : 1)>{}, st, ca); break;
          case 7: if constexpr (GT <= 2 && 7 < CPS) codes_stage(std::integral_constant<int, (7 < CPS ? 7 : 1)>{}, st, ca); break;
          default: break;
        }
      } else {
        // the ragged last group of a layer (m_pad / 128 not a multiple of g / 128): by step
        const int ga = ca / HG;
        float d[NT][4];
        zero4(d);
        for (int s = 0; s < 2 * nck; ++s) {
          uint32_t f[4][4];
          decode_step(st + (s >> 1) * CB, s & 1, f);
          mma_step(f, ca * 128 + s * 64, d);
          const int step = 2 * ca + s;
          if ((step % GT) == GT - 1 || step == 2 * a.nch - 1) {
            fold(st + kSzOff + (step / GT - ga) * 64, step / GT, d);
            zero4(d);
          }
        }
      }
    } else {
      const int wa = sg.w0 + (t - ncs) * kWPS, nwt = min(kWPS, sg.w1 - wa);
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
    t += sstep;
    while (t >= nst) {
      t -= nst;
      ++jl;
    }
  }
  if (my_n > 0) park(cur_jl);
  if (tr && threadIdx.x == 0) tr[4] = gtime();
  __syncthreads();
  // ---- this CTA's slice partial of every row-block: sum the warps in order (into the slot
  // of the first contributing warp: fslot) ----
  auto fslot = [&](int jq, int nst_r) {
    return CONTIG ? jq + warp_of_stage(jq * nst_r, nj * nst_r, NW) : jq * NW;
  };
  auto store = [&](int jq, int r, float v) {
    const int row16 = ONE ? r : r / n, col = ONE ? 0 : r - row16 * n;
    int lrb;
    const int l = layer_of(a, j0 + jq, lrb);
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
  };
  // one K slice: the warp sum is the output (stored straight away, no second pass)
  for (int e = threadIdx.x; e < nj * redn; e += NW * 32) {
    const int jq = e / redn, r = e - jq * redn;
    float v = 0.f;
    float* dst;
    if (CONTIG) {
      const int wa = warp_of_stage(jq * nst, total, NW), wb = warp_of_stage(jq * nst + nst - 1, total, NW);
      float* p = red + (size_t)jq * redn + r;
      for (int w = wa; w <= wb; ++w) v += p[w * redn];
      dst = p + wa * redn;
    } else {
      float* p = red + (size_t)jq * NW * redn + r;
#pragma unroll
      for (int w = 0; w < NW; ++w) v += p[w * redn];
      dst = p;
    }
    if (a.S > 1) *dst = v;
    else store(jq, r, v);
  }
  // ---- K slices of a cluster: sum them (ranks in order, over DSMEM) and store y ----
  if (a.S > 1) {
    cluster_sync();
    for (int e = threadIdx.x; e < nj * redn; e += NW * 32) {
      const int jq = e / redn, r = e - jq * redn;
      if ((jq % a.S) != rank) continue;
      // rank q's slot of row-block jq follows from its own slice geometry
      float v = 0.f;
      for (int q = 0; q < a.S; ++q)
        v += ld_dsmem_f32(smem_u32(red + (size_t)fslot(jq, a.geo[q].nst) * redn + r), q);
      store(jq, r, v);
    }
  }
  if (a.S > 1) cluster_sync();  // keep this CTA's partials alive until every rank has read them
  if (tr && threadIdx.x == 0) tr[6] = gtime();
}

// ---------------------------------------------------------------------------
// host: slicing and launch

struct Geom {
  int nch, U, nuc, nwt, cb, szb, m_pad, g, CPS;
};

// balance units (codes units of U chunks, then weak tiles) into S contiguous slices by bytes
void slice_units(const Geom& G, int S, int* ub) {
  const int nu = G.nuc + G.nwt;
  auto ubytes = [&](int u) -> double {
    if (u < G.nuc) return (double)std::min(G.U, G.nch - u * G.U) * G.cb + G.szb;
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

SliceGeo slice_geo(const Geom& G, int u0, int u1) {
  SliceGeo s{};
  auto kpos = [&](int u) { return u <= G.nuc ? std::min(u * G.U, G.nch) * 128 : G.m_pad + (u - G.nuc) * 64; };
  s.c0 = std::min(std::min(u0, G.nuc) * G.U, G.nch);
  s.c1 = std::min(std::min(u1, G.nuc) * G.U, G.nch);
  s.w0 = std::max(u0, G.nuc) - G.nuc;
  s.w1 = std::max(u1, G.nuc) - G.nuc;
  s.kb = kpos(u0);
  s.ke = kpos(u1);
  s.gx0 = s.kb < G.m_pad ? s.kb / G.g : 0;
  s.ngx = s.kb < G.m_pad ? (std::min(s.ke, G.m_pad) - s.gx0 * G.g + G.g - 1) / G.g : 0;
  s.ncs = (s.c1 - s.c0 + G.CPS - 1) / G.CPS;
  s.nst = s.ncs + (s.w1 - s.w0 + G.CPS / 2 - 1) / (G.CPS / 2);
  return s;
}

// MINB CTAs per SM (2: a CTA of the next launch can start -- and prefetch its weights --
// beside a CTA of this one)
template <int BITS, int NT, int GT, typename T, int R, int NW, int CPS, bool CONTIG = false, int MINB = 1,
          int GPS = MINB>
int launch2(G2Args a, cudaStream_t st) {
  a.contig = CONTIG;
  if (a.ngain && NW * 32 < a.nthr) return -1;  // the fused norm needs the rmsnorm block size
  constexpr int kStage = CPS * 1152;
  constexpr int kSmemMax = (MINB == 1 ? 227 * 1024 : 113 * 1024) - 1024;
  constexpr int PRE = MINB > 1 ? R : 0;  // pre-wait weight prefetch only when CTAs can overlap
  auto kern1 = gemv2_kernel<BITS, NT, GT, T, R, NW, CPS, true, MINB, PRE, CONTIG>;
  auto kernN = gemv2_kernel<BITS, NT, GT, T, R, NW, CPS, false, MINB, PRE, CONTIG>;
  const bool one = a.n == 1 && NT == 1;
  auto kern = one ? kern1 : kernN;
  const bool fused = a.ngain || a.xu;
  if constexpr (NT == 1 && NW == 16 && CPS == 4 && !CONTIG && MINB == 1) {
    if (fused) {
      static bool fattr = false;
      auto f1 = gemv2_kernel<BITS, NT, GT, T, R, NW, CPS, true, MINB, PRE, CONTIG, true>;
      auto fN = gemv2_kernel<BITS, NT, GT, T, R, NW, CPS, false, MINB, PRE, CONTIG, true>;
      if (!fattr) {
        for (auto kk : {f1, fN}) {
          QEFT_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
          QEFT_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        fattr = true;
      }
      kern = one ? f1 : fN;
    }
  } else {
    if (fused) return -1;  // the decode plans host the fusions; others use the stand-alone kernels
  }
  static bool attr = false;
  if (!attr) {
    for (auto kk : {kern1, kernN}) {
      QEFT_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
      QEFT_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    QEFT_CUDA(cudaGetDevice(&dev));
    QEFT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  Geom G;
  G.nch = a.nch;
  G.U = std::max(1, a.g / 128);
  G.nuc = (G.nch + G.U - 1) / G.U;
  G.nwt = a.k_pad / 64;
  G.cb = BITS == 4 ? 1024 : 768;
  G.szb = 64 * std::max(1, G.U * 128 / a.g);
  G.m_pad = a.m_pad;
  G.g = a.g;
  G.CPS = CPS;
  const int rings = NW * R * kStage;
  const int force_s = env_int("QEFT_GEMV2_S", 0);
  // choose the cluster size S (= K slices): the busiest CTA streams J row-blocks of its slice
  double best = 1e300;
  G2Args bestA = a;
  int best_grid = 0;
  size_t best_smem = 0;
  for (int S = 1; S <= kMaxS; ++S) {
    if (force_s && S != force_s) continue;
    if (S > G.nuc + G.nwt) break;
    G2Args b = a;
    b.S = S;
    int ub[kMaxS + 1];
    slice_units(G, S, ub);
    bool empty = false;
    double smax = 0;
    int xc = 0, xg = 0;
    for (int s = 0; s < S; ++s) {
      empty |= ub[s + 1] == ub[s];
      b.geo[s] = slice_geo(G, ub[s], ub[s + 1]);
      const SliceGeo& q = b.geo[s];
      xc = std::max(xc, q.ke - q.kb);
      xg = std::max(xg, q.ngx);
      smax = std::max(smax, (double)(q.c1 - q.c0) * G.cb + (double)(q.c1 - q.c0) * 128 / a.g * 64 +
                                (q.w1 - q.w0) * 2048.0);
    }
    if (empty) continue;
    b.xs_ld = xc + 8;  // 16 B skew between staged x rows
    // clusters that fit on the GPU at once (persistent: one wave)
    int nclu = sms * GPS / S;
    size_t smem = 0;
    for (int it = 0; it < 3; ++it) {
      b.J = (a.n_rb + nclu - 1) / nclu;
      if (b.J > kMaxJ) break;
      const int slots = a.contig ? b.J + NW : b.J * NW;
      smem = (size_t)rings + (size_t)slots * 16 * a.n * 4 + (size_t)a.n * b.xs_ld * 2 + (size_t)xg * NT * 8 * 4;
      if (a.xu) {  // the staged up-projection rows (same layout as xs)
        smem = (smem + 15) & ~(size_t)15;
        b.xu_off = (int)smem;
        smem += (size_t)a.n * b.xs_ld * 2;
      }
      b.xraw_off = 0;
      if (!a.fast && a.ic % 8 == 0 && a.ldx % 8 == 0 && (((uintptr_t)a.x) & 15) == 0 &&
          smem + 16 + (size_t)a.n * ((a.ic + 7) & ~7) * 2 <= (size_t)kSmemMax) {
        smem = (smem + 15) & ~(size_t)15;
        b.xraw_off = (int)smem;
        smem += (size_t)a.n * ((a.ic + 7) & ~7) * 2;
      }
      if (smem > (size_t)kSmemMax) break;
      if (S == 1) break;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nclu * S);
      cfg.blockDim = dim3(NW * 32);
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
    }
    if (b.J > kMaxJ || smem == 0 || smem > (size_t)kSmemMax) continue;
    const int ncl = (a.n_rb + b.J - 1) / b.J;
    // + the cluster epilogue (~1.6 us measured, i.e. ~70 KB of one SM's HBM share)
    const double cost = b.J * smax + (S > 1 ? 70.0 * 1024 : 0.0);
    if (cost < best * 0.98) {
      best = cost;
      bestA = b;
      best_grid = ncl * S;
      best_smem = smem;
    }
  }
  if (best_grid == 0) return -1;  // partials do not fit shared memory: the generic kernel serves it
  static const int log = env_int("QEFT_GEMV2_LOG", 0);
  if (log)
    fprintf(stderr, "gemv2 n=%d rb=%d m_pad=%d: NT=%d NW=%d CPS=%d contig=%d S=%d J=%d grid=%d smem=%zu\n", a.n,
            a.n_rb, a.m_pad, NT, NW, CPS, a.contig, bestA.S, bestA.J, best_grid, best_smem);
  if (bestA.S > 1) {
    QEFT_CUDA(launch_pdl_cluster(kern, dim3(best_grid), dim3(NW * 32), best_smem, st, bestA.S, bestA));
  } else {
    QEFT_CUDA(launch_pdl(kern, dim3(best_grid), dim3(NW * 32), best_smem, st, bestA));
  }
  return 0;
}

template <int BITS, typename T>
int dispatch2(const G2Args& a, int gt, cudaStream_t st) {
  const bool nt2 = a.n > 8;
  // launch2 returns -1 when the plan does not fit shared memory: try the next shape
#define QEFT_G2(CONTIG, NT, NWV, CPSV)                                                   \
  {                                                                                      \
    int r_ = -1;                                                                         \
    switch (gt) {                                                                        \
      case 1: r_ = launch2<BITS, NT, 1, T, 2, NWV, CPSV, CONTIG>(a, st); break;          \
      case 2: r_ = launch2<BITS, NT, 2, T, 2, NWV, CPSV, CONTIG>(a, st); break;          \
      case 4: r_ = launch2<BITS, NT, 4, T, 2, NWV, CPSV, CONTIG>(a, st); break;          \
      default: if constexpr (CPSV >= 4) r_ = launch2<BITS, NT, 8, T, 2, NWV, (CPSV >= 4 ? CPSV : 4), CONTIG>(a, st); break; \
    }                                                                                    \
    if (r_ != -1) return r_;                                                             \
  }
  // 16 warps whenever the partials and the staged x fit (the decode + MMA issue rate is the
  // limit). Round-robin stage dealing streams neighbouring stages from all warps at once
  // (measured 3.5 % faster at n = 1) but needs J x NW partial slots; contiguous runs need
  // J + NW, so up to 8 columns fit beside 16 rings (n = 4: +31 %, n = 8: +26 %,
  // profiles/r02/batch_ab.json). 16 columns stage 16 rows of x and may need 2 KB stages or 8 warps.
  const int cmode = a.contig;  // QEFT_GEMV2_CONTIG: 0 never, 1 when it enables more warps
  if (nt2) {
    if (cmode) QEFT_G2(true, 2, 16, 4)
    if (cmode) QEFT_G2(true, 2, 16, 2)
    if (cmode) QEFT_G2(true, 2, 8, 4)
    if (cmode && gt <= 4) QEFT_G2(true, 2, 8, 2)
    QEFT_G2(false, 2, 8, 4)
  } else if (a.n > 2) {
    QEFT_G2(false, 1, 16, 4)
    if (cmode) QEFT_G2(true, 1, 16, 4)
    QEFT_G2(false, 1, 8, 4)
  } else {
    QEFT_G2(false, 1, 16, 4)
  }
  return -1;
#undef QEFT_G2
}

}  // namespace
#endif
