// Prefill / fine-tune GEMMs of the QEFT layer on 5th-generation tensor cores.
//
// Replaces the reference's dense fp32 products over the re-materialized weight
// (pkg/src/qeft/tuning.py:52-103):
//   fwd    Y[t][o]  = sum_j W_hat[o][j] X[t][j]            (qlinear_forward_train)
//   dgrad  dX[t][i] = sum_o W_hat[o][i] dY[t][o]           (qlinear_backward, dX)
//   wgrad  dW[o][w] = sum_t dY[t][o] X[t][weak_w]          (qlinear_backward, dW_weak)
// W_hat is never materialized in HBM: warp-specialized persistent kernels
//   * dequantize the 3/4-bit tile layout straight into SWIZZLE_128B shared memory
//     (K-major for fwd, MN-major for dgrad) with 8 producer warps (their instruction
//     rate, not load latency, bounds the tensor pipe: measured),
//   * stream activations with TMA (cp.async.bulk.tensor, OOB zero fill covers the
//     quantized/weak split of the B200 K order),
//   * issue tcgen05.mma (M=128, N=BN, K=16, fp32 accumulators in TMEM, double
//     buffered) from one thread,
//   * drain TMEM with tcgen05.ld in 4 epilogue warps, transposing through shared
//     memory into the row-major [tokens][channels] outputs.
// wgrad is a smaller TMA-only kernel (both operands MN-major) whose N is the
// weak block width.
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "qeft_common.cuh"
#include "qeft_internal.h"
#include "qeft_tc.cuh"

using namespace qeft;

#ifndef QEFT_GEMM_PROFILE
#define QEFT_GEMM_PROFILE 0  // 1: per-CTA globaltimer stamps + QEFT_GEMM_DIAG modes (scripts/trace_gemm.py)
#endif

namespace {

enum { MODE_FWD = 0, MODE_DGRAD = 1 };

constexpr int BM = 128;                 // MMA M (rows of W_hat or of W_hat^T)
constexpr int BK = 64;                  // K per stage (one SWIZZLE_128B row of fp16)
constexpr int kProdWarps = 8;           // dequant producers (two per SM sub-partition)
constexpr int kUPW = 8 / kProdWarps;    // 16x64 A units per producer warp per k-block
constexpr int kEpiWarps = 4;
constexpr int kThreads = (2 + kProdWarps + kEpiWarps) * 32;  // TMA, MMA, producers, epilogue
constexpr int kStageA = BM * BK * 2;    // 16 KB
constexpr int kEpiStride = 40;          // halves per staging row (32 + 8 pad)
constexpr int kRing = 8;                // stream-K fix-up: 4 KB bulk-copy slots per epilogue warp

struct GemmArgs {
  const uint8_t* qw;
  const float2* sz;
  const void* weak16;
  const int* colmap;
  int oc, m, m_pad, k, k_pad, g, ng;
  int T;
  int n_mblk, n_nblk, n_kblk, kq;  // kq: quantized k-blocks (fwd) / quantized m-tiles (dgrad)
  int n_items, n_full;             // work items: [0, n_full) whole tiles, then half tiles (NSUB == 2)
  void* out;
  int64_t ldo;
  int accumulate;
  int gathered;   // fwd: B from one map over a gathered B200-order buffer
  int fast_out;   // dgrad: output columns contiguous in 32-blocks (structured, m % 32 == 0)
  int out_cols;   // fwd: oc; dgrad: ic
  int g_shift;    // log2(g) when g is a power of two, else -1 (group index without a divide)
  // stream-K schedule (sk != 0): the n_items x n_kblk k-block units are cut into gridDim.x
  // contiguous ranges; a tile split across CTAs is finished by the CTA holding its last k-block,
  // which adds the fp32 partials the other CTAs left in part[cta] (flags[cta] = 1 when ready)
  int sk;
  float* part;
  int* flags;
  unsigned long long* trace;  // profiling only (qeft_gemv_trace slots): per-CTA globaltimer stamps
  int b200_out;    // dgrad: write dX in B200 K order (all m_pad + k_pad columns; a scatter follows)
  int tma_out;     // epilogue writes 32 x 32 output blocks with TMA stores (reduce-add to accumulate)
  int diag;  // profiling only (QEFT_GEMM_DIAG): 1 producers skip global loads, 2 skip dequant,
             // 3 no MMAs, 4 no activation TMA after the first ring, 5 = 2 + 4 -- results are garbage;
             // isolates the bounding pipeline
};

// The work of one CTA as a list of segments (tile, k-blocks [kb0, kb1)). Round-robin whole
// tiles, or (stream-K) the tiles of the CTA's unit range ordered so that the one segment that
// does NOT end its tile (a partial for a later CTA) runs first and the segment that finishes a
// tile started by earlier CTAs runs last: producers publish early, finishers consume late, and a
// CTA only ever waits on lower-numbered CTAs (no deadlock with in-order CTA dispatch).
struct Seg {
  int tile, kb0, kb1, fin;
};
template <bool SK>
struct SegPlan {
  int nseg, b, G, nk, sk;
  int t_first, head, tail, nfull;
  int64_t u0, u1, U;
  QEFT_DEV static int64_t ustart(int64_t p, int64_t U, int G) { return p * U / G; }
  QEFT_DEV void init(int ntiles, int nk_, int cg = 1) {
    b = blockIdx.x / cg; G = gridDim.x / cg; nk = nk_; sk = SK;  // a CTA pair shares one schedule
    if constexpr (!SK) {
      nseg = ntiles > b ? (ntiles - 1 - b) / G + 1 : 0;
      return;
    }
    U = (int64_t)ntiles * nk;
    u0 = ustart(b, U, G);
    u1 = ustart(b + 1, U, G);
    if (u1 <= u0) {
      nseg = 0;
      return;
    }
    t_first = (int)(u0 / nk);
    const int t_last = (int)((u1 - 1) / nk);
    head = (u1 % nk) != 0;                                 // t_last's segment stops short of its end
    tail = (u0 % nk) != 0 && !(t_first == t_last && head);  // t_first's segment finishes a split tile
    nseg = t_last - t_first + 1;
    nfull = nseg - head - tail;
  }
  QEFT_DEV Seg get(int i) const {
    Seg s;
    if constexpr (!SK) {
      s.tile = b + i * G; s.kb0 = 0; s.kb1 = nk; s.fin = 1;
      return s;
    }
    if (head && i == 0) {
      const int t = (int)((u1 - 1) / nk);
      s.tile = t;
      s.kb0 = (int)(max(u0, (int64_t)t * nk) - (int64_t)t * nk);
      s.kb1 = (int)(u1 - (int64_t)t * nk);
      s.fin = 0;
      return s;
    }
    const int j = i - head;
    if (j < nfull) {
      s.tile = t_first + tail + j; s.kb0 = 0; s.kb1 = nk; s.fin = 1;
      return s;
    }
    s.tile = t_first;
    s.kb0 = (int)(u0 - (int64_t)t_first * nk);
    s.kb1 = nk;
    s.fin = 1;
    return s;
  }
  QEFT_DEV int64_t start_of(int p) const { return ustart(p, U, G); }
};

template <typename T>
QEFT_DEV uint32_t pack2(float a, float b) {
  typename DTraits<T>::T2 v;
  v.x = from_f32<T>(a);
  v.y = from_f32<T>(b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Dequantize one lane's share of a 16-row x 64-column k-tile (rows g, g+8 of the
// row-block; columns 16t..16t+15) into fp32-exact (code*s + z) rounded to T.
// q4 holds the lane's 4-bit word (16 B) or, for 3-bit, w2 (8 B) + hb (4 B).
// out[0..7] = row g, cols 16t..16t+15 (T2 pairs); out[8..15] = row g+8.
template <int BITS, typename T>
QEFT_DEV void dequant_lane(const uint32_t* words, uint32_t hb, float2 p0, float2 p1, uint32_t out[16]) {
  // magic + code halves via the fp16 trick for 4-bit (rows g+8 scaled by 16), exact in fp32
  const float s0 = p0.x, z0 = p0.y - 1024.f * p0.x;
  const float s1 = (BITS == 4) ? p1.x * (1.f / 16.f) : p1.x;
  const float z1 = p1.y - 1024.f * s1;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t f[4];
    if constexpr (BITS == 4) {
      decode4<__half>(words[j], f);
    } else {
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) f[pp] = decode3_pair<__half>(words[j >> 1], hb, 4 * (j & 1) + pp, j >> 1);
    }
    const float2 a0 = __half22float2(*reinterpret_cast<__half2*>(&f[0]));  // row g, cols c, c+1
    const float2 a1 = __half22float2(*reinterpret_cast<__half2*>(&f[1]));  // row g+8, cols c, c+1
    const float2 a2 = __half22float2(*reinterpret_cast<__half2*>(&f[2]));  // row g, cols c+2, c+3
    const float2 a3 = __half22float2(*reinterpret_cast<__half2*>(&f[3]));  // row g+8, cols c+2, c+3
    out[2 * j] = pack2<T>(fmaf(a0.x, s0, z0), fmaf(a0.y, s0, z0));
    out[2 * j + 1] = pack2<T>(fmaf(a2.x, s0, z0), fmaf(a2.y, s0, z0));
    out[8 + 2 * j] = pack2<T>(fmaf(a1.x, s1, z1), fmaf(a1.y, s1, z1));
    out[8 + 2 * j + 1] = pack2<T>(fmaf(a3.x, s1, z1), fmaf(a3.y, s1, z1));
  }
}

// Packed path: the same fragments in the activation dtype's paired arithmetic.
// (magic + c) - magic = c exactly (HSUB2); c * s rounds once (HFMA2 into the high part of
// the zero point), then the low part of the zero point is added (HADD2). Splitting
// z = z_hi + z_lo keeps the per-group offset exact to ~2^-17, so no systematic per-group
// error appears; the scale carries one rounding to T (<= 2^-9 relative).
template <int BITS, typename T>
QEFT_DEV void dequant_lane_packed(const uint32_t* words, uint32_t hb, float2 p0, float2 p1, uint32_t out[16]) {
  using T2 = typename DTraits<T>::T2;
  constexpr bool hi = (BITS == 4) && DTraits<T>::kHiTrick;  // fp16 rows g+8 hold magic + 16 c
  uint32_t mw = DTraits<T>::kMagic;
  const T2 M2 = *reinterpret_cast<T2*>(&mw);
  auto split = [](float z, T2& zh, T2& zl) {
    const T h = from_f32<T>(z);
    const T l = from_f32<T>(z - to_f32<T>(h));
    zh.x = zh.y = h;
    zl.x = zl.y = l;
  };
  T2 S0, S1, Z0h, Z0l, Z1h, Z1l;
  S0.x = S0.y = from_f32<T>(p0.x);
  S1.x = S1.y = from_f32<T>(hi ? p1.x * (1.f / 16.f) : p1.x);
  split(p0.y, Z0h, Z0l);
  split(p1.y, Z1h, Z1l);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t f[4];
    if constexpr (BITS == 4) {
      decode4<T>(words[j], f);
    } else {
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) f[pp] = decode3_pair<T>(words[j >> 1], hb, 4 * (j & 1) + pp, j >> 1);
    }
    T2 v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const T2 c = __hsub2(*reinterpret_cast<const T2*>(&f[e]), M2);
      v[e] = (e & 1) ? __hadd2(__hfma2(c, S1, Z1h), Z1l) : __hadd2(__hfma2(c, S0, Z0h), Z0l);
    }
    out[2 * j] = *reinterpret_cast<uint32_t*>(&v[0]);          // row g,   cols c, c+1
    out[2 * j + 1] = *reinterpret_cast<uint32_t*>(&v[2]);      // row g,   cols c+2, c+3
    out[8 + 2 * j] = *reinterpret_cast<uint32_t*>(&v[1]);      // row g+8, cols c, c+1
    out[8 + 2 * j + 1] = *reinterpret_cast<uint32_t*>(&v[3]);  // row g+8, cols c+2, c+3
  }
}

// general group sizes: per-element (scale, zero)
template <int BITS, typename T>
QEFT_DEV void dequant_lane_general(const uint32_t* words, uint32_t hb, const float2* szrow0,
                                   const float2* szrow1, int col0, int g, int ng, uint32_t out[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t f[4];
    if constexpr (BITS == 4) {
      decode4<__half>(words[j], f);
    } else {
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) f[pp] = decode3_pair<__half>(words[j >> 1], hb, 4 * (j & 1) + pp, j >> 1);
    }
    float v[2][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int fi0 = (e < 2) ? 0 : 2, fi1 = (e < 2) ? 1 : 3;
      const float2 h0 = __half22float2(*reinterpret_cast<__half2*>(&f[fi0]));
      const float2 h1 = __half22float2(*reinterpret_cast<__half2*>(&f[fi1]));
      const float c0 = ((e & 1) ? h0.y : h0.x) - 1024.f;
      const float c1 = (BITS == 4) ? (((e & 1) ? h1.y : h1.x) - 1024.f) * (1.f / 16.f)
                                   : ((e & 1) ? h1.y : h1.x) - 1024.f;
      const int gi = min((col0 + 4 * j + e) / g, ng - 1);
      const float2 pa = szrow0[gi * 16], pb = szrow1[gi * 16];
      v[0][e] = c0 * pa.x + pa.y;
      v[1][e] = c1 * pb.x + pb.y;
    }
    out[2 * j] = pack2<T>(v[0][0], v[0][1]);
    out[2 * j + 1] = pack2<T>(v[0][2], v[0][3]);
    out[8 + 2 * j] = pack2<T>(v[1][0], v[1][1]);
    out[8 + 2 * j + 1] = pack2<T>(v[1][2], v[1][3]);
  }
}

// Ring depths: A stages (16 KB, dequantized / weak TMA) and B stages (BN x 64 activations).
// A tile of NSUB sub-tiles reuses each A stage for NSUB MMA groups (N = BN each), so the
// producers dequantize once per NSUB * BN tokens.
// CG = 2: a CTA pair (cluster of 2) runs one M = 256 MMA over both SMs' shared memory: each CTA
// dequantizes its own 128 rows of A and loads HALF of every B sub-tile (BN / 2 tokens), so the
// per-SM shared-memory operand traffic per MMA drops from 12 KB to 8 KB (measured: the 1-SM
// MMA of this kernel runs at ~58 % of the tcgen05 floor, shared-memory bound, with its producers
// and activation TMA removed -- QEFT_GEMM_DIAG=5).
template <int BN, int NSUB, int CG = 1>
struct GemmShape {
  static constexpr int kStageB = (BN / CG) * BK * 2;
  static constexpr int kStagesA = CG == 2 ? 4 : (NSUB == 2 ? 3 : (BN == 256 ? 4 : 6));
  static constexpr int kStagesB = CG == 2 ? (NSUB == 2 ? 8 : 6) : (NSUB == 2 ? 5 : kStagesA);
  // epilogue staging: 2 x [32 tokens][32 channels] per warp for TMA stores (>= the padded
  // [32][kEpiStride] transpose buffer of the scalar path)
  static constexpr size_t kEpiBytes = (size_t)kEpiWarps * 2 * 32 * 32 * 2;
  static_assert(kEpiBytes >= (size_t)kEpiWarps * 32 * kEpiStride * 2, "staging");
  static constexpr size_t kSmem = 1024 + (size_t)kStagesA * kStageA + (size_t)kStagesB * kStageB + kEpiBytes;
};

template <int MODE, int BITS, typename T, int BN, int NSUB, int CG, bool SKT>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_b0, const __grid_constant__ CUtensorMap map_b1,
            const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_y,
            const GemmArgs a) {
  using Sh = GemmShape<BN, NSUB, CG>;
  constexpr int kStageB = Sh::kStageB;
  constexpr int kStagesA = Sh::kStagesA, kStagesB = Sh::kStagesB;
  // two accumulator slots of BN columns: sub-tile q (running count) uses slot q & 1
  constexpr int kTmemCols = 2 * BN;
  constexpr int kTileN = BN * NSUB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base for SWIZZLE_128B atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStagesA * kStageA;
  T* sE = reinterpret_cast<T*>(sB + kStagesB * kStageB);  // epilogue staging [4 warps][32][kEpiStride]
  __shared__ __align__(8) uint64_t fullA[kStagesA], emptyA[kStagesA], fullB[kStagesB], emptyB[kStagesB];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t ring_full[kEpiWarps][kRing];  // stream-K fix-up ring
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if QEFT_GEMM_PROFILE
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * 8 : nullptr;
#else
  constexpr unsigned long long* tr = nullptr;  // profiling build only (make EXTRA=-DQEFT_GEMM_PROFILE=1)
#endif
  auto stamp = [&](int i) {
    if constexpr (QEFT_GEMM_PROFILE) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[(size_t)blockIdx.x * 8 + i] = t;
    }
  };
  if (tr && threadIdx.x == 0) stamp(0);
  const int ntiles = a.n_items;
#if QEFT_GEMM_PROFILE
  const int DIAG_ = a.diag;
#else
  constexpr int DIAG_ = 0;
#endif
  // CTA pair: rank 0 (leader) issues the MMAs; both CTAs produce their own A rows and B half
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  // whole tiles (SKT = false: the schedule and the producers' cursor are the plain tile-stride
  // loop) or stream-K segments -- separate instantiations, so the whole-tile kernel carries none
  // of the stream-K bookkeeping in registers
  SegPlan<SKT> plan;
  plan.init(ntiles, a.n_kblk, CG);
  // leader's copy of a barrier (shared::cluster address); the pair's producers arrive there
  auto lead = [&](uint64_t* bar) -> uint32_t { return CG == 2 ? tc::mapa_u32(bar, 0) : smem_u32(bar); };
  // work item -> (m-block, first token, sub-tiles). Items past n_full are the halves of the
  // last partial wave's tiles, so that wave spreads over twice as many SMs.
  struct Item {
    int m_blk, tok0, nsub;
  };
  auto item = [&](int i) {
    Item it;
    int t = i, half = 0;
    it.nsub = NSUB;
    if (NSUB == 2 && i >= a.n_full) {
      t = a.n_full + ((i - a.n_full) >> 1);
      half = (i - a.n_full) & 1;
      it.nsub = 1;
    }
    const int nm = CG == 2 ? a.n_mblk / 2 : a.n_mblk;  // pair tiles span two m-blocks
    const int n_blk = t / nm;
    it.m_blk = (t - n_blk * nm) * CG + (int)rank;
    it.tok0 = n_blk * kTileN + half * BN;
    return it;
  };

  // [32 tokens][32 channels] block of the accumulator (thread = channel row, r = its 32 token
  // columns) -> fp16/bf16 staging `buf` -> one TMA store (clipped at the tensor's edges;
  // reduce-add when accumulating). row_base: the block's first row (channel / B200 column).
  auto tma_block = [&](const uint32_t (&r)[32], int row_base, int tc0, T* buf) {
    int col0 = row_base;
    bool ok = true;
    if (MODE == MODE_FWD) {
      ok = row_base < a.oc;
    } else if (a.b200_out) {
      ok = true;  // B200 order: the scatter drops the padding columns
    } else if (row_base < a.m_pad) {
      ok = row_base < a.m;  // [m, m_pad) is padding: its columns belong to the weak block
    } else {
      col0 = a.m + (row_base - a.m_pad);
      ok = row_base - a.m_pad < a.k;
    }
    ok = ok && tc0 < a.T;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");  // buffer free
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 32; ++c) buf[c * 32 + lane] = from_f32<T>(__uint_as_float(r[c]));
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && ok) {
      if (a.accumulate)
        asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];\n"
                     ::"l"(&map_y), "r"(col0), "r"(tc0), "r"(smem_u32(buf)) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];\n"
                     ::"l"(&map_y), "r"(col0), "r"(tc0), "r"(smem_u32(buf)) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  };
  // whole-tile kernels: the producer warps, idle once their last k-block is dequantized, drain
  // two thirds of the CTA's LAST tile (its column blocks u = j * BN / 32 + cb with u % 3 != 0)
  // beside the epilogue warps -- that tile's epilogue is nobody else's overlap
  const bool join = !SKT && a.tma_out;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesA; ++s) {
      mbar_init(&fullA[s], 1 + CG * kProdWarps);  // leader's TMA warp (weak bytes, maybe 0) + producers
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < kStagesB; ++s) {
      mbar_init(&fullB[s], 1);  // the leader's TMA thread posts the pair's bytes
      mbar_init(&emptyB[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], CG * kEpiWarps);
    }
    for (int i = 0; i < kEpiWarps * kRing; ++i) mbar_init(&ring_full[i / kRing][i % kRing], 1);
    fence_mbar_init();
    tc::prefetch_tmap(&map_b0);
    tc::prefetch_tmap(&map_b1);
    if (a.k) tc::prefetch_tmap(&map_w);
  }
  if (warp == 1) {
    if constexpr (CG == 2) tc::tmem_alloc_pair(&tmem_base, kTmemCols);
    else tc::tmem_alloc(&tmem_base, kTmemCols);
  }
  tc::fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // the peer's barriers are initialised before any remote arrive
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  pdl_launch_dependents();
  // The grid dependency is waited for by the roles that read what earlier kernels write: the TMA
  // warp (activations, weak tiles), the epilogue (outputs) and the dequant producers after
  // their first two k-blocks of codes -- the frozen codes and scales never change, so those
  // loads overlap the previous kernel's tail.
  if (tr && threadIdx.x == 0) stamp(1);

  if (warp == 0) {
    // ================= TMA producer: activation tiles =================
    pdl_wait();
    if (lane == 0) {
      int it = 0, ib = 0;
      for (int si = 0; si < plan.nseg; ++si) {
        const Seg sg = plan.get(si);
        const Item ti = item(sg.tile);
        const int m_blk = ti.m_blk, tok0 = ti.tok0;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
          const int s = it % kStagesA;
          mbar_wait(&emptyA[s], ((it / kStagesA) & 1) ^ 1);
          // the weak block is already fp16/bf16 in 16 x 64 row-block tiles: TMA places it in
          // the A stage (SWIZZLE_128B, the layout the dequant producers write)
          auto weak_bytes = [&](int mb) -> uint32_t {
            if (MODE == MODE_FWD) return kb >= a.kq ? kStageA : 0;
            if (mb < a.kq) return 0;
            return (((mb - a.kq) * 2 + 1) * 64 < a.k_pad) ? kStageA : kStageA / 2;
          };
          const uint32_t wbytes = weak_bytes(m_blk);
          auto load4 = [&](uint8_t* dst, int c2, int c3) {
            if constexpr (CG == 2) tc::tma_load_4d_pair(dst, &map_w, 0, 0, c2, c3, lead(&fullA[s]));
            else tc::tma_load_4d(dst, &map_w, 0, 0, c2, c3, &fullA[s]);
          };
          // a pair's leader posts both CTAs' weak bytes (the peer's m-block is m_blk + 1); the
          // peer's copies may complete on the leader's barrier before this, which is allowed
          if (leader) mbar_expect_tx(&fullA[s], CG == 2 ? wbytes + weak_bytes(m_blk + 1) : wbytes);
          if (MODE == MODE_FWD && kb >= a.kq) {
            load4(sA + s * kStageA, kb - a.kq, 8 * m_blk);
          } else if (MODE == MODE_DGRAD && m_blk >= a.kq) {
            // MN-major A: two 64-row halves, one per weak K-tile (the second may be past k_pad)
            const int kw0 = (m_blk - a.kq) * 2;
            load4(sA + s * kStageA, kw0, 4 * kb);
            if (wbytes == kStageA) load4(sA + s * kStageA + 8192, kw0 + 1, 4 * kb);
          }
#pragma unroll
          for (int j = 0; j < NSUB; ++j, ++ib) {
            if (j >= ti.nsub) break;
            const int sb = ib % kStagesB;
            mbar_wait(&emptyB[sb], ((ib / kStagesB) & 1) ^ 1);
            if ((DIAG_ == 4 || DIAG_ == 5) && ib >= kStagesB) {  // profiling: no activation traffic after the first ring
              if (leader) mbar_arrive(&fullB[sb]);
              continue;
            }
            uint8_t* dst = sB + sb * kStageB;
            const CUtensorMap* mb = (MODE == MODE_FWD && !a.gathered && kb >= a.kq) ? &map_b1 : &map_b0;
            const int kc = (MODE == MODE_FWD && !a.gathered && kb >= a.kq) ? (kb - a.kq) * BK : kb * BK;
            if constexpr (CG == 2) {  // this CTA's half of the sub-tile's tokens
              if (leader) mbar_expect_tx(&fullB[sb], 2 * kStageB);
              tc::tma_load_2d_pair(dst, mb, kc, tok0 + j * BN + (int)rank * (BN / 2), lead(&fullB[sb]));
            } else {
              mbar_expect_tx(&fullB[sb], kStageB);
              tc::tma_load_2d(dst, mb, kc, tok0 + j * BN, &fullB[sb]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread; the leader CTA's for a pair) =================
    if (!leader) goto mma_done;
    {
    const uint32_t idesc = tc::idesc_f16(std::is_same<T, __nv_bfloat16>::value, BM * CG, BN,
                                         MODE == MODE_DGRAD, false);
    int it = 0, ib = 0, q0 = 0;
    auto wait = [&](uint64_t* bar, uint32_t par) { mbar_wait(bar, par); };
    auto commit = [&](uint64_t* bar) {
      if constexpr (CG == 2) tc::commit_pair(bar);
      else tc::commit(bar);
    };
    for (int si = 0; si < plan.nseg; ++si) {
      const Seg sg = plan.get(si);
      const int nsub = item(sg.tile).nsub;
      for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
        const int s = it % kStagesA;
        wait(&fullA[s], (it / kStagesA) & 1);
        tc::fence_after();
        const uint32_t a0 = smem_u32(sA + s * kStageA);
        // the CTA's last k-block: nobody waits for these stages again, and a pair's peer may
        // already have left -- only the accumulator-full arrival is signalled
        const bool last_kb = si == plan.nseg - 1 && kb == sg.kb1 - 1;
#pragma unroll
        for (int j = 0; j < NSUB; ++j, ++ib) {
          if (j >= nsub) break;
          const int q = q0 + j, slot = q & 1;
          if (kb == sg.kb0) {  // the epilogue has drained this slot's previous sub-tile
            wait(&tempty_bar[slot], ((q >> 1) & 1) ^ 1);
            tc::fence_after();
          }
          const int sb = ib % kStagesB;
          wait(&fullB[sb], (ib / kStagesB) & 1);
          tc::fence_after();
          if (lane == 0) {
            const uint32_t b0 = smem_u32(sB + sb * kStageB);
            if (tr && it == 0 && j == 0) stamp(2);
            if (tr && si == plan.nseg - 1 && kb == sg.kb1 - 1 && j == nsub - 1) stamp(3);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = (MODE == MODE_FWD) ? tc::smem_desc_sw128(a0 + 32 * k, 16, 1024)
                                                     : tc::smem_desc_sw128(a0 + 2048 * k, 8192, 1024);
              const uint64_t bd = tc::smem_desc_sw128(b0 + 32 * k, 16, 1024);
              const uint32_t acc = (kb != sg.kb0 || k) ? 1u : 0u;
              if (DIAG_ != 3) {
                if constexpr (CG == 2) tc::mma_f16_pair(tmem + slot * BN, ad, bd, idesc, acc);
                else tc::mma_f16(tmem + slot * BN, ad, bd, idesc, acc);
              }
            }
            if (CG == 1 || !last_kb) commit(&emptyB[sb]);
            if (kb == sg.kb1 - 1) commit(&tfull_bar[slot]);
          }
          __syncwarp();
        }
        if (lane == 0 && (CG == 1 || !last_kb)) commit(&emptyA[s]);
        __syncwarp();
      }
      q0 += nsub;
    }
    }
  mma_done:;
  } else if (warp < 2 + kProdWarps) {
    // ================= dequant producers: the A operand =================
    // Each warp fills two 16-row x 64-column units of the A tile per k-block:
    // Unit u = pw * kUPW + h (0..7) of the 128 x 64 A tile:
    //   fwd:   row-block 8*m_blk + u, B200 columns 64*kb.. (K-major rows)
    //   dgrad: row-block 4*kb + u/2, B200 columns 64*(2*m_blk + u%2).. (MN-major)
    // Global loads for k-block kb+2 are issued before k-block kb is processed.
    const int pw = warp - 2;
    const int g8 = lane >> 2, t4 = lane & 3;
    const bool fold16 = (a.g % 16) == 0;
    // weak tiles arrive by TMA (already fp16/bf16), so a unit in flight is 16 B of codes + params
    struct Pre {
      uint4 v[kUPW];  // lane codes of unit h (3-bit: .x,.y = 2-bit words, .z = hi word)
      float2 p0[kUPW], p1[kUPW];
    };
    // unit geometry: row-block, 64-column tile index in the B200 order, weak tile (or -1)
    auto unit = [&](int m_blk, int kb, int h, int& rb, int& jt, int& kw) {
      const int u = pw * kUPW + h;  // A unit 0..7 of the k-block
      if (MODE == MODE_FWD) {
        rb = m_blk * 8 + u;
        jt = kb;
        kw = kb >= a.kq ? kb - a.kq : -1;
      } else {
        rb = kb * 4 + (u >> 1);
        jt = 2 * m_blk + (u & 1);
        kw = m_blk >= a.kq ? (m_blk - a.kq) * 2 + (u & 1) : -1;
      }
    };
    auto load = [&](int m_blk, int kb, Pre& P) {
      if (DIAG_ == 1) {
#pragma unroll
        for (int h = 0; h < kUPW; ++h) {
          P.v[h] = make_uint4(lane * 0x01010101u, kb, m_blk, 7u);
          P.p0[h] = P.p1[h] = make_float2(0.01f, 0.f);
        }
        return;
      }
#pragma unroll
      for (int h = 0; h < kUPW; ++h) {
        int rb, jt, kw;
        unit(m_blk, kb, h, rb, jt, kw);
        if (kw >= 0 || rb * 16 >= a.oc) continue;  // weak tiles arrive by TMA
        if constexpr (BITS == 4) {
          P.v[h] = ldg_stream(a.qw + ((int64_t)rb * (a.m_pad >> 6) + jt) * 512 + lane * 16);
        } else {
          const uint8_t* tb = a.qw + ((int64_t)rb * (a.m_pad >> 7) + (jt >> 1)) * 768;
          const uint2 w2 = *reinterpret_cast<const uint2*>(tb + lane * 16 + 8 * (jt & 1));
          P.v[h] = make_uint4(w2.x, w2.y, *reinterpret_cast<const uint32_t*>(tb + 512 + lane * 8 + 4 * (jt & 1)), 0u);
        }
        if (fold16) {
          const float2* szr = a.sz + (int64_t)rb * a.ng * 16;
          const int col = jt * BK + 16 * t4;
          const int gi = min(a.g_shift >= 0 ? (col >> a.g_shift) : col / a.g, a.ng - 1);
          P.p0[h] = szr[gi * 16 + g8];
          P.p1[h] = szr[gi * 16 + g8 + 8];
        }
      }
    };
    auto process = [&](int m_blk, int kb, const Pre& P, uint8_t* st) {
#pragma unroll
      for (int h = 0; h < kUPW; ++h) {
        int rb, jt, kw;
        unit(m_blk, kb, h, rb, jt, kw);
        if (kw >= 0 && kw * 64 < a.k_pad) continue;  // written by the TMA warp
        uint32_t out[16];
        if (rb * 16 >= a.oc || kw >= 0) {
#pragma unroll
          for (int e = 0; e < 16; ++e) out[e] = 0u;
        } else {
          const uint32_t words[4] = {P.v[h].x, P.v[h].y, P.v[h].z, P.v[h].w};
          const uint32_t hb = (BITS == 3) ? P.v[h].z : 0u;
          if (fold16) {
            dequant_lane_packed<BITS, T>(words, hb, P.p0[h], P.p1[h], out);
          } else {
            const float2* szr = a.sz + (int64_t)rb * a.ng * 16;
            dequant_lane_general<BITS, T>(words, hb, szr + g8, szr + g8 + 8, jt * BK + 16 * t4, a.g, a.ng, out);
          }
        }
        uint32_t o0, o1, o2, o3;  // byte offsets of (row g, chunk 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)
        if (MODE == MODE_FWD) {
          const int r0 = 16 * (pw * kUPW + h) + g8, r1 = r0 + 8;
          o0 = tc::sw128(r0, 2 * t4); o1 = tc::sw128(r0, 2 * t4 + 1);
          o2 = tc::sw128(r1, 2 * t4); o3 = tc::sw128(r1, 2 * t4 + 1);
        } else {
          // MN-major: (m, k) at (m/64)*8192 + (k/8)*1024 + sw128(k%8, (m%64)/8)
          const int u = pw * kUPW + h;
          const int kr0 = 16 * (u >> 1) + g8, kr1 = kr0 + 8;
          const uint32_t base = (u & 1) * 8192;
          o0 = base + (kr0 >> 3) * 1024 + tc::sw128(kr0 & 7, 2 * t4);
          o1 = base + (kr0 >> 3) * 1024 + tc::sw128(kr0 & 7, 2 * t4 + 1);
          o2 = base + (kr1 >> 3) * 1024 + tc::sw128(kr1 & 7, 2 * t4);
          o3 = base + (kr1 >> 3) * 1024 + tc::sw128(kr1 & 7, 2 * t4 + 1);
        }
        *reinterpret_cast<uint4*>(st + o0) = make_uint4(out[0], out[1], out[2], out[3]);
        *reinterpret_cast<uint4*>(st + o1) = make_uint4(out[4], out[5], out[6], out[7]);
        *reinterpret_cast<uint4*>(st + o2) = make_uint4(out[8], out[9], out[10], out[11]);
        *reinterpret_cast<uint4*>(st + o3) = make_uint4(out[12], out[13], out[14], out[15]);
      }
    };
    // flatten (tile, kb) into one stream so the prefetch crosses tile boundaries; the
    // stream is walked with incremental cursors (no integer divides per k-block)
    int total = 0;
    for (int si = 0; si < plan.nseg; ++si) {
      const Seg sg = plan.get(si);
      total += sg.kb1 - sg.kb0;
    }
    const int per = a.n_kblk, wb = (int)blockIdx.x / CG, wg = (int)gridDim.x / CG;
    struct Cursor {
      int si, m_blk, kb, kb1;  // segment (stream-K) or tile (whole tiles), m-block, k-block, end
    };
    auto set_seg = [&](Cursor& c) {
      if (c.si < plan.nseg) {
        const Seg sg = plan.get(c.si);
        c.m_blk = item(sg.tile).m_blk;  // once per segment
        c.kb = sg.kb0;
        c.kb1 = sg.kb1;
      }
    };
    auto advance = [&](Cursor& c) {
      if constexpr (!SKT) {
        if (++c.kb == per) {
          c.kb = 0;
          c.si += wg;
          if (c.si < ntiles) c.m_blk = item(c.si).m_blk;  // once per tile
        }
      } else {
        if (++c.kb == c.kb1) {
          ++c.si;
          set_seg(c);
        }
      }
    };
    Cursor cl{0, 0, 0, 0};  // load cursor (2 ahead)
    if constexpr (!SKT) {
      cl.si = wb;
      cl.m_blk = wb < ntiles ? item(wb).m_blk : 0;
    } else {
      set_seg(cl);
    }
    Cursor cp = cl;                                              // process cursor
    auto coords = [&](int, int& m_blk, int& kb) {  // next position of the load cursor
      m_blk = cl.m_blk;
      kb = cl.kb;
      advance(cl);
    };
    Pre P0, P1, P2;  // register ring, rotated by value (no dynamic indexing -> no local memory)
    if (total > 0) {
      int mb, kb;
      coords(0, mb, kb);
      load(mb, kb, P0);
    }
    if (total > 1) {
      int mb, kb;
      coords(1, mb, kb);
      load(mb, kb, P1);
    }
    pdl_wait();
    for (int it = 0; it < total; ++it) {
      if (it + 2 < total) {
        int mb, kb;
        coords(it + 2, mb, kb);
        load(mb, kb, P2);
      }
      const int mb = cp.m_blk, kb = cp.kb;
      advance(cp);
      const int s = it % kStagesA;
      mbar_wait(&emptyA[s], ((it / kStagesA) & 1) ^ 1);
      if (DIAG_ != 2 && DIAG_ != 5) process(mb, kb, P0, sA + s * kStageA);
      if (tr && pw == 0 && lane == 0 && it == 0) stamp(6);
      P0 = P1;
      P1 = P2;
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) tc::mbar_arrive_cluster(lead(&fullA[s]));
        else mbar_arrive(&fullA[s]);
      }
    }
    if (join && plan.nseg > 0) {
      int q_last = 0;  // the epilogue's sub-tile counter at the CTA's last tile
      for (int si = 0; si + 1 < plan.nseg; ++si) q_last += item(plan.get(si).tile).nsub;
      const Item ti = item(plan.get(plan.nseg - 1).tile);
      // every MMA of the tile is done (so the A stages are free staging) once its last
      // sub-tile's accumulator is full
      const int ql = q_last + ti.nsub - 1;
      mbar_wait(&tfull_bar[ql & 1], (ql >> 1) & 1);
      tc::fence_after();
      const int quad = warp & 3, role = 1 + (pw >> 2);  // epilogue warp of this quadrant: role 0
      T* pbuf = reinterpret_cast<T*>(sA) + (size_t)pw * 2048;
      int nb = 0;
      for (int j = 0; j < ti.nsub; ++j) {
        const int qq = q_last + j;
        mbar_wait(&tfull_bar[qq & 1], (qq >> 1) & 1);
        tc::fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (qq & 1) * BN;
#pragma unroll 1
        for (int cb = 0; cb < BN / 32; ++cb) {
          if ((j * (BN / 32) + cb) % 3 != role) continue;
          uint32_t r[32];
          tc::tmem_ld32(tbase + cb * 32, r);
          tma_block(r, ti.m_blk * BM + quad * 32, ti.tok0 + j * BN + cb * 32, pbuf + (nb++ & 1) * 1024);
        }
      }
      tc::fence_before();
    }
  } else {
    // ================= epilogue: TMEM -> registers -> smem transpose -> global =================
    pdl_wait();
    const int ew = warp - (2 + kProdWarps);
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    T* stg = sE + ew * 32 * kEpiStride;
    int q = 0;
    const int erow = quad * 32 + lane;  // accumulator row of this thread
    for (int si = 0; si < plan.nseg; ++si) {
    const Seg sg = plan.get(si);
    const Item ti = item(sg.tile);
    // stream-K: a finisher of a tile begun by earlier CTAs waits for their partials, then streams
    // them (4 KB per warp, cb and producer) through a per-warp ring of bulk copies in the stage
    // memory -- free once the last sub-tile's MMAs are done, as the fix-up is the CTA's last
    // segment. Partial layout per CTA: [sub-tile][cb][quad][c / 4][lane][4] fp32.
    // schedule positions are per CTA pair (CG = 2); partials and flags per CTA: vid = p * CG + rank
    const int pb = plan.b;
    auto vid = [&](int pp) { return pp * CG + (int)rank; };
    int p_lo = pb;
    const bool fixup = SKT && sg.fin && sg.kb0 > 0;
    constexpr int kCbChunk = 32 * 32 * 4;  // bytes of one warp's 32 rows x 32 columns
    uint8_t* ring = sA + ew * kRing * kCbChunk;
    int n_chunk = 0, c_use = 0;
    auto chunk_src = [&](int c) {  // chunk c = (j, cb, producer) in consumption order
      const int np = pb - p_lo;
      const int p = p_lo + c % np, jc = c / np;
      return (const uint8_t*)a.part +
             ((size_t)vid(p) * (NSUB * BN * BM) + ((size_t)jc * 4 + quad) * 1024) * sizeof(float);
    };
    auto issue = [&](int c) {
      const int slot = c % kRing;
      mbar_expect_tx(&ring_full[ew][slot], kCbChunk);
      bulk_g2s(ring + slot * kCbChunk, chunk_src(c), kCbChunk, &ring_full[ew][slot]);
    };
    if (fixup) {
      const int64_t t0u = (int64_t)sg.tile * a.n_kblk;
      p_lo = pb - 1;
      while (plan.start_of(p_lo) > t0u) --p_lo;
      if (ew == 0 && lane == 0) {
        for (int p = p_lo; p < pb; ++p) {
          int f;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(f) : "l"(a.flags + vid(p)) : "memory");
          } while (f == 0);
        }
      }
      named_bar_sync(1, kEpiWarps * 32);
      // the stage memory is free when the tile's last sub-tile is accumulated
      const int ql = q + ti.nsub - 1;
      mbar_wait(&tfull_bar[ql & 1], (ql >> 1) & 1);
      n_chunk = ti.nsub * (BN / 32) * (pb - p_lo);
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        for (int c = 0; c < min(n_chunk, kRing); ++c) issue(c);
      }
      __syncwarp();
    }
    for (int j = 0; j < ti.nsub; ++j, ++q) {
      const int m_blk = ti.m_blk;
      const int acc = q & 1;
      mbar_wait(&tfull_bar[acc], (q >> 1) & 1);
      tc::fence_after();
      if (tr && ew == 0 && lane == 0 && q == 0) stamp(4);
      const int row_base = m_blk * BM + quad * 32;  // channel (fwd) / B200 column (dgrad) of lane 0
      auto body = [&](int cb, uint32_t (&r)[32]) {
        if (SKT && !sg.fin) {
          float4* dst = reinterpret_cast<float4*>(a.part + (size_t)vid(pb) * (NSUB * BN * BM) +
                                                  (((size_t)(j * (BN / 32) + cb) * 4 + quad) * 1024)) + lane;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            __stcg(dst + c4 * 32, make_float4(__uint_as_float(r[4 * c4]), __uint_as_float(r[4 * c4 + 1]),
                                              __uint_as_float(r[4 * c4 + 2]), __uint_as_float(r[4 * c4 + 3])));
          return;
        }
        if (fixup) {
          for (int p = p_lo; p < pb; ++p, ++c_use) {
            const int slot = c_use % kRing;
            mbar_wait(&ring_full[ew][slot], (c_use / kRing) & 1);
            const float4* src = reinterpret_cast<const float4*>(ring + slot * kCbChunk) + lane;
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const float4 v = src[c4 * 32];
              r[4 * c4] = __float_as_uint(__uint_as_float(r[4 * c4]) + v.x);
              r[4 * c4 + 1] = __float_as_uint(__uint_as_float(r[4 * c4 + 1]) + v.y);
              r[4 * c4 + 2] = __float_as_uint(__uint_as_float(r[4 * c4 + 2]) + v.z);
              r[4 * c4 + 3] = __float_as_uint(__uint_as_float(r[4 * c4 + 3]) + v.w);
            }
            __syncwarp();
            if (lane == 0 && c_use + kRing < n_chunk) {
              fence_proxy_async_smem();  // generic reads of the slot before the async overwrite
              issue(c_use + kRing);
            }
          }
        }
        if (DIAG_ == 6) return;  // profiling: TMEM loads only
        if (a.tma_out) {
          tma_block(r, row_base, ti.tok0 + j * BN + cb * 32, sE + (size_t)ew * 2048 + (cb & 1) * 1024);
          return;
        }
        // thread = one row (channel), 32 token columns -> staging [token][row]
#pragma unroll
        for (int c = 0; c < 32; ++c) stg[c * kEpiStride + lane] = from_f32<T>(__uint_as_float(r[c]));
        __syncwarp();
        // thread = one token, 32 consecutive rows
        const int tok = ti.tok0 + j * BN + cb * 32 + lane;
        if (tok < a.T && DIAG_ != 7) {  // 7: profiling, no global stores
          const T* src = stg + lane * kEpiStride;
          if (MODE == MODE_FWD || a.fast_out) {
            int col0 = row_base;
            if (MODE == MODE_DGRAD) col0 = row_base < a.m_pad ? row_base : a.m + (row_base - a.m_pad);
            const int lim = (MODE == MODE_FWD) ? a.oc : ((row_base < a.m_pad) ? a.m : a.m + a.k);
            T* dst = (T*)a.out + (int64_t)tok * a.ldo + col0;
            const bool vec = (col0 + 32 <= lim) && ((((uintptr_t)dst) & 15) == 0);
            if (vec && !a.accumulate) {
#pragma unroll
              for (int v = 0; v < 4; ++v)
                reinterpret_cast<uint4*>(dst)[v] = reinterpret_cast<const uint4*>(src)[v];
            } else {
              for (int e = 0; e < 32 && col0 + e < lim; ++e)
                dst[e] = a.accumulate ? from_f32<T>(to_f32<T>(dst[e]) + to_f32<T>(src[e])) : src[e];
            }
          } else {
            for (int e = 0; e < 32; ++e) {
              const int j = row_base + e;
              if (j >= a.m_pad + a.k_pad) break;
              const int col = a.colmap[j];
              if (col < 0) continue;
              T* dst = (T*)a.out + (int64_t)tok * a.ldo + col;
              *dst = a.accumulate ? from_f32<T>(to_f32<T>(*dst) + to_f32<T>(src[e])) : src[e];
            }
          }
        }
        __syncwarp();
      };
      // (loading the next column block ahead of the stores measured no gain and pushed the
      // kernel past 128 registers)
      const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + acc * BN;
      const bool shared_drain = join && si == plan.nseg - 1;  // producers take u % 3 != 0
#pragma unroll 1
      for (int cb = 0; cb < BN / 32; ++cb) {
        if (shared_drain && (j * (BN / 32) + cb) % 3 != 0) continue;
        uint32_t r[32];
        tc::tmem_ld32(tbase + cb * 32, r);
        body(cb, r);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) tc::mbar_arrive_cluster(lead(&tempty_bar[acc]));
        else mbar_arrive(&tempty_bar[acc]);
      }
    }
    if (SKT && !sg.fin) {
      // publish this CTA's partial: every writer fences, then one release store
      __threadfence();
      named_bar_sync(1, kEpiWarps * 32);
      if (ew == 0 && lane == 0)
        asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(a.flags + vid(pb)), "r"(1) : "memory");
    } else if (SKT && sg.fin && sg.kb0 > 0) {
      // every epilogue warp is done reading the partials: re-arm the producers' flags
      named_bar_sync(1, kEpiWarps * 32);
      if (ew == 0 && lane == 0)
        for (int p = p_lo; p < pb; ++p) a.flags[vid(p)] = 0;
    }
    }
  }

  if (warp >= 2 && lane == 0 && a.tma_out)
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // output stores done before exit
  if (tr && warp == 2 + kProdWarps && lane == 0) stamp(5);
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // both CTAs done: no arrivals in flight to the peer
  if (warp == 1) {
    tc::fence_after();
    if constexpr (CG == 2) tc::tmem_dealloc_pair(tmem, kTmemCols);
    else tc::tmem_dealloc(tmem, kTmemCols);
  }
  if (tr && threadIdx.x == 0) stamp(7);
}

// ---------------------------------------------------------------------------
// wgrad: dW[o][w] (+)= sum_t dY[t][o] * Xw[t][w]; M = 128 channels, N = k_pad, K = tokens.
// Both operands MN-major via TMA boxes of {64 (M or N), 64 (t)}.
// Split-K over tokens runs inside a thread-block cluster: the S CTAs of a cluster (gridDim.x
// = S, blockIdx.y = channel block) each accumulate their token range in TMEM, stage the fp32
// partial in their own (now idle) stage memory, and CTA r then sums rows [r*128/S, ...) of
// all S partials over DSMEM in rank order (deterministic) and writes them to dW. The 128
// rows of one channel block are one contiguous (128 x k) fp32 chunk of dW, so the
// read-modify-write is fully coalesced float4 traffic.
template <int NW>
struct WgradShape {
  static constexpr int N = NW * 64;
  static constexpr int kSA = BM * 64 * 2;  // 16 KB: 2 boxes of 64 channels x 64 tokens
  static constexpr int kSB = N * 64 * 2;   // NW boxes of 64 weak columns x 64 tokens
  static constexpr int kStages = (192 * 1024) / (kSA + kSB) > 8 ? 8 : (192 * 1024) / (kSA + kSB);
  static constexpr int kStride = N + 4;  // staging row pitch (floats): 16-B aligned, conflict-free
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kSA + kSB);
  static_assert((size_t)BM * kStride * 4 <= (size_t)kStages * (kSA + kSB), "staging fits the stages");
};

// Up to 3 layers that share the weak input columns (a block's q/k/v, or gate/up) in one
// launch: blockIdx.y runs over all of their 128-channel blocks.
constexpr int kMaxWgLayers = 3;
struct WgradGroup {
  CUtensorMap dy[kMaxWgLayers];
  float* dw[kMaxWgLayers];
  int oc[kMaxWgLayers];
  int blk_end[kMaxWgLayers];  // cumulative channel blocks
  int nl;
};

template <typename T, int NW>
__global__ void __launch_bounds__(192, 1)
wgrad_kernel(const __grid_constant__ WgradGroup grp, const __grid_constant__ CUtensorMap map_xw, int k, int T_,
             int accumulate, int kb_split, int vec_out) {
  using Sh = WgradShape<NW>;
  constexpr int N = Sh::N, kSA = Sh::kSA, kSB = Sh::kSB, kStages = Sh::kStages, kStride = Sh::kStride;
  constexpr int kCols = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kSA;
  float* stg = reinterpret_cast<float*>(smem);  // [128][kStride] fp32 partial, after the mainloop
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], done_bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.x, rank = blockIdx.x;  // cluster = the S token splits of one channel block
  int l = 0;
  while (l + 1 < grp.nl && (int)blockIdx.y >= grp.blk_end[l]) ++l;
  const CUtensorMap& map_dy = grp.dy[l];
  float* __restrict__ dw = grp.dw[l];
  const int oc = grp.oc[l];
  const int o0 = ((int)blockIdx.y - (l ? grp.blk_end[l - 1] : 0)) * BM;
  const int kb0 = rank * kb_split;
  const int nkb = max(0, min((T_ + 63) / 64 - kb0, kb_split));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, kCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  pdl_launch_dependents();
  pdl_wait();
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&empty_bar[s], ((kb / kStages) & 1) ^ 1);
        mbar_expect_tx(&full_bar[s], kSA + kSB);
        const int t0 = (kb0 + kb) * 64;
        tc::tma_load_2d(sA + s * kSA, &map_dy, o0, t0, &full_bar[s]);
        tc::tma_load_2d(sA + s * kSA + 8192, &map_dy, o0 + 64, t0, &full_bar[s]);
#pragma unroll
        for (int b = 0; b < NW; ++b) tc::tma_load_2d(sB + s * kSB + b * 8192, &map_xw, b * 64, t0, &full_bar[s]);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = tc::idesc_f16(std::is_same<T, __nv_bfloat16>::value, BM, N, true, true);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kStages;
      mbar_wait(&full_bar[s], (kb / kStages) & 1);
      tc::fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + s * kSA), b0 = smem_u32(sB + s * kSB);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc::mma_f16(tmem, tc::smem_desc_sw128(a0 + 2048 * kk, 8192, 1024),
                      tc::smem_desc_sw128(b0 + 2048 * kk, 8192, 1024), idesc, (kb | kk) ? 1u : 0u);
        tc::commit(&empty_bar[s]);
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (nkb > 0) tc::commit(&done_bar);
      else mbar_arrive(&done_bar);  // empty split: its partial is zero
    }
    __syncwarp();
  } else {
    // TMEM -> staging (thread = channel row, 32 columns per load)
    const int quad = warp & 3;
    mbar_wait(&done_bar, 0);
    tc::fence_after();
    float* row = stg + (quad * 32 + lane) * kStride;
#pragma unroll 1
    for (int cb = 0; cb < N / 32; ++cb) {
      uint32_t r[32];
      if (nkb > 0) {
        tc::tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + cb * 32, r);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = 0u;
      }
#pragma unroll
      for (int c = 0; c < 32; c += 4)
        *reinterpret_cast<float4*>(row + cb * 32 + c) =
            make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]), __uint_as_float(r[c + 2]),
                        __uint_as_float(r[c + 3]));
    }
    tc::fence_before();
  }
  __syncthreads();
  if (S > 1) cluster_sync();  // every split's partial is staged
  // rows [rank * R, (rank + 1) * R) of the channel block: dW (+)= sum over splits, rank order
  const int R = BM / S;
  const uint32_t stg_base = smem_u32(stg);
  if (vec_out) {
    // batches of 8 float4 per thread: the dW loads of a batch are in flight together
    constexpr int C4 = N / 4, kB = 8;
    const int n4 = R * C4;
    for (int i0 = 0; i0 < n4; i0 += kB * (int)blockDim.x) {
      float4 v[kB];
      float4* dst[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int i = i0 + b * blockDim.x + threadIdx.x;
        const int rr = rank * R + i / C4, c = (i % C4) * 4;
        const bool ok = i < n4 && o0 + rr < oc && c < k;
        dst[b] = ok ? reinterpret_cast<float4*>(dw + (int64_t)(o0 + rr) * k + c) : nullptr;
        v[b] = (ok && accumulate) ? *dst[b] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        if (!dst[b]) continue;
        const int i = i0 + b * blockDim.x + threadIdx.x;
        const int rr = rank * R + i / C4, c = (i % C4) * 4;
        const uint32_t off = stg_base + (uint32_t)(rr * kStride + c) * 4;
        for (int sp = 0; sp < S; ++sp) {
          float4 p;
          if (S == 1) {
            p = *reinterpret_cast<const float4*>(stg + rr * kStride + c);
          } else {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(off), "r"(sp));
            asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(p.x), "=f"(p.y), "=f"(p.z), "=f"(p.w)
                         : "r"(remote)
                         : "memory");
          }
          v[b].x += p.x; v[b].y += p.y; v[b].z += p.z; v[b].w += p.w;
        }
        *dst[b] = v[b];
      }
    }
  } else {
    for (int i = threadIdx.x; i < R * N; i += blockDim.x) {
      const int rr = rank * R + i / N, c = i % N;
      const int o = o0 + rr;
      if (o >= oc || c >= k) continue;
      const uint32_t off = stg_base + (uint32_t)(rr * kStride + c) * 4;
      float* dst = dw + (int64_t)o * k + c;
      float v = accumulate ? *dst : 0.f;
      for (int sp = 0; sp < S; ++sp) v += (S == 1) ? stg[rr * kStride + c] : ld_dsmem_f32(off, sp);
      *dst = v;
    }
  }
  if (S > 1) cluster_sync();  // keep this CTA's partial alive until every rank has read it
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, kCols);
  }
}

// ---------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 2-D row-major [rows][ld] tensor, box {64 inner, box_rows}, SWIZZLE_128B, OOB -> 0
int make_map(CUtensorMap* m, const void* base, int dtype, int64_t inner, int64_t rows, int64_t ld_elems,
             int box_rows) {
  auto fn = encode_fn();
  QEFT_CHECK(fn != nullptr, QEFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  QEFT_CHECK(((uintptr_t)base & 15) == 0 && (ld_elems * 2) % 16 == 0, QEFT_ERR_LAYOUT,
             "TMA needs 16-byte aligned base and row stride");
  // driver-API call: threads that have only used the runtime implicitly (e.g. the
  // autograd engine's worker) may have no current context yet
  static auto get_ctx = []() -> CUresult (*)(CUcontext*) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (CUresult(*)(CUcontext*))p;
    return nullptr;
  }();
  CUcontext ctx = nullptr;
  if (get_ctx == nullptr || get_ctx(&ctx) != CUDA_SUCCESS || ctx == nullptr) {
    int dev = 0;
    QEFT_CUDA(cudaGetDevice(&dev));
    QEFT_CUDA(cudaSetDevice(dev));
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, dtype == QEFT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  QEFT_CHECK(r == CUDA_SUCCESS, QEFT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

// output [rows][ld] tensor, box {32 columns, 32 rows}, no swizzle (epilogue TMA stores)
int make_out_map(CUtensorMap* m, void* base, int dtype, int64_t inner, int64_t rows, int64_t ld_elems) {
  auto fn = encode_fn();
  if (fn == nullptr) return QEFT_ERR_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 2)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, dtype == QEFT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base,
                  dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : QEFT_ERR_CUDA;
}

// weak16 [oc_pad/16][k_pad/64][16][64] as a 4-D tensor, box {64, 16, 1, box_rb}, SWIZZLE_128B
int make_weak_map(CUtensorMap* m, const void* weak16, int dtype, int k_pad, int n_rb, int box_rb) {
  auto fn = encode_fn();
  QEFT_CHECK(fn != nullptr, QEFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  QEFT_CHECK(((uintptr_t)weak16 & 15) == 0, QEFT_ERR_LAYOUT, "weak16 must be 16-byte aligned");
  cuuint64_t dims[4] = {64, 16, (cuuint64_t)(k_pad / 64), (cuuint64_t)n_rb};
  cuuint64_t strides[3] = {128, 2048, (cuuint64_t)(k_pad / 64) * 2048};
  cuuint32_t box[4] = {64, 16, 1, (cuuint32_t)box_rb};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, dtype == QEFT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                  const_cast<void*>(weak16), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  QEFT_CHECK(r == CUDA_SUCCESS, QEFT_ERR_CUDA, "cuTensorMapEncodeTiled (weak) failed (%d)", (int)r);
  return 0;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// stream-K scratch, one per (device, stream): flags[sms] (zero between launches: each finisher
// re-arms the flags it consumed) + one fp32 partial tile (2 x 256 x 128) per CTA. Allocated on
// first use outside graph capture; a capturing stream without one falls back to whole tiles.
int g_sk_mode = getenv("QEFT_GEMM_SK") ? atoi(getenv("QEFT_GEMM_SK")) : -1;
// CTA pairs: implemented and parity-tested, not the default -- measured equal or 1-2 % slower
// (profiles/r02/gemm_ab.json): this kernel's 1-SM MMA already runs at the cuBLAS per-SM rate
// with its producers removed (QEFT_GEMM_DIAG=5), so halving B's per-SM traffic buys nothing
int g_cg_mode = getenv("QEFT_GEMM_CG") ? (atoi(getenv("QEFT_GEMM_CG")) == 2 ? 2 : 1) : 1;

struct SkBuf {
  float* part = nullptr;
  int* flags = nullptr;
};
SkBuf sk_buffers(cudaStream_t st) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SkBuf> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = bufs.find({dev, st});
  if (it != bufs.end()) return it->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return SkBuf{};
  }
  const size_t bytes = 1024 + (size_t)num_sms() * 2 * 256 * BM * sizeof(float);
  void* p = nullptr;
  if (num_sms() > 256 || cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return SkBuf{};
  }
  if (cudaMemsetAsync(p, 0, 1024, st) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p);
    return SkBuf{};
  }
  SkBuf b;
  b.flags = (int*)p;
  b.part = (float*)((char*)p + 1024);
  bufs[{dev, st}] = b;
  return b;
}

template <int MODE, int BITS, typename T, int BN, int NSUB, int CG>
int launch_gemm(const CUtensorMap& m0, const CUtensorMap& m1, const CUtensorMap& mw, const CUtensorMap& my,
                const GemmArgs& a, cudaStream_t st) {
  using Sh = GemmShape<BN, NSUB, CG>;
  const size_t smem = Sh::kSmem;
  static_assert(Sh::kSmem <= 227 * 1024, "GEMM smem");
  static_assert(kEpiWarps * kRing * 4096 <= Sh::kStagesA * kStageA + Sh::kStagesB * Sh::kStageB,
                "stream-K fix-up ring fits the stage memory");
  auto kern_dp = gemm_kernel<MODE, BITS, T, BN, NSUB, CG, false>;
  auto kern_sk = gemm_kernel<MODE, BITS, T, BN, NSUB, CG, true>;
  static bool attr = false;
  if (!attr) {
    QEFT_CUDA(cudaFuncSetAttribute(kern_dp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    QEFT_CUDA(cudaFuncSetAttribute(kern_sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  GemmArgs b = a;
  static const int diag = getenv("QEFT_GEMM_DIAG") ? atoi(getenv("QEFT_GEMM_DIAG")) : 0;
  b.diag = diag;
  b.trace = trace_next_slot();
  // workers: CTAs, or CTA pairs (CG = 2: a tile is 256 rows = two m-blocks)
  const int sms = num_sms(), workers = sms / CG;
  const int tiles = (a.n_mblk / CG) * a.n_nblk;
  b.n_items = b.n_full = tiles;
  double dp_span = (tiles + workers - 1) / workers;  // makespan of the round-robin schedule, in tile times
  if (NSUB == 2 && tiles > workers) {
    // split the last partial wave's tiles into halves when they then fit in one wave
    const int waves = (tiles + workers - 1) / workers, r = tiles - (waves - 1) * workers;
    if (r < workers && 2 * r <= workers) {
      b.n_full = (waves - 1) * workers;
      b.n_items = b.n_full + 2 * r;
      dp_span = waves - 0.5;
    }
  }
  // stream-K when whole tiles leave SMs idle: every worker gets tiles * n_kblk / workers
  // k-blocks. Measured (profiles/r02/streamk_ab.json, 1-SM tiles): it loses 4-12 % at 128 tiles
  // on 148 SMs (two epilogues per CTA, the 256 KB partial store exposed while both TMEM slots
  // are held), gains 2-3 % at 344 tiles, 27-50 % at 160 tiles and 30-70 % at 80 tiles (13B,
  // T = 2048 / 512): worth it when it saves more than a tenth of a tile time
  const int sk_mode = g_sk_mode;
  const double sk_span = (double)tiles / workers + 0.06;
  const int64_t units = (int64_t)tiles * a.n_kblk;
  const bool sk_ok = sk_mode == 1 ? units >= workers : units >= 8LL * workers;
  if (sk_mode != 0 && sk_ok && (sk_mode == 1 || sk_span + 0.1 < dp_span)) {
    SkBuf sb = sk_buffers(st);
    if (sb.part) {
      b.sk = 1;
      b.part = sb.part;
      b.flags = sb.flags;
      b.n_items = b.n_full = tiles;
    }
  }
  const int grid = CG * (b.sk ? workers : std::min(b.n_items, workers));
  auto kern = b.sk ? kern_sk : kern_dp;
  if (CG == 2) {
    QEFT_CUDA(launch_pdl_cluster(kern, dim3(grid), dim3(kThreads), smem, st, 2, m0, m1, mw, my, b));
  } else {
    QEFT_CUDA(launch_pdl(kern, dim3(grid), dim3(kThreads), smem, st, m0, m1, mw, my, b));
  }
  return 0;
}

// Tile plan of one GEMM: N per sub-tile (BN), sub-tiles sharing each dequantized A stage (NSUB),
// CTAs per MMA (CG). The activation maps' box is BN / CG tokens.
struct GemmPlan {
  int bn, nsub, cg;
};
GemmPlan gemm_plan(int n_mblk, int T_, int n_kblk) {
  // tile N: 128 tokens (T <= 128), 256, or 2 x 256 sharing each dequantized A stage (T > 256;
  // QEFT_GEMM_NSUB=1 forces single sub-tiles)
  static const int nsub_env = getenv("QEFT_GEMM_NSUB") ? atoi(getenv("QEFT_GEMM_NSUB")) : 0;
  GemmPlan p;
  const bool big = T_ > 128;
  // paired sub-tiles halve dequant work per FLOP, but when even twice the items of single
  // sub-tiles fit one wave (few m-blocks, short T: 13B T=512), parallelism wins
  const int pair_items = n_mblk * ((T_ + 511) / 512);
  // ... unless the K loop is long enough that stream-K still gives every SM >= 40 k-blocks of
  // paired tiles (13B T = 512: 5120 x 13824 fwd 675 -> 744 TFLOP/s, 5120 x 5120 stays single)
  const bool long_k = (int64_t)pair_items * n_kblk >= 40LL * num_sms();
  p.nsub = (T_ > 256 && nsub_env != 1 && (nsub_env == 2 || 2 * pair_items > num_sms() || long_k)) ? 2 : 1;
  p.bn = big ? 256 : 128;
  // CTA pairs (M = 256) for 256-token sub-tiles over an even number of m-blocks
  p.cg = (big && n_mblk % 2 == 0 && g_cg_mode == 2) ? 2 : 1;
  return p;
}

template <int MODE, typename T>
int dispatch_gemm(const qeft_linear_t* L, int T_, const GemmPlan& p, const CUtensorMap& m0, const CUtensorMap& m1,
                  GemmArgs& a, cudaStream_t st) {
  const bool pair = p.nsub == 2, big = p.bn == 256;
  a.n_nblk = (T_ + p.bn * p.nsub - 1) / (p.bn * p.nsub);
  // weak block as a 4-D tensor {64 columns, 16 rows, k_pad/64 tiles, row-blocks} of the
  // row-block tile layout (weak_off, qeft_common.cuh); box = 8 row-blocks (fwd: the 128 rows of
  // the K-major A tile) or 4 row-blocks (dgrad: one 64-row half of the MN-major A tile)
  CUtensorMap mw = m0;
  if (L->k) {
    if (int r = make_weak_map(&mw, L->weak16, L->act_dtype, L->k_pad, L->oc_pad / 16, MODE == MODE_FWD ? 8 : 4))
      return r;
  }
  // output blocks by TMA store: contiguous output columns (fwd, or dgrad's structured layout),
  // 16-byte aligned rows (QEFT_GEMM_TMA_OUT=0: per-thread stores through a padded transpose)
  static const int tma_env = getenv("QEFT_GEMM_TMA_OUT") ? atoi(getenv("QEFT_GEMM_TMA_OUT")) : 1;
  CUtensorMap my = m0;
  a.tma_out = 0;
  if (tma_env && (MODE == MODE_FWD || a.fast_out || a.b200_out) && (a.ldo * 2) % 16 == 0 &&
      ((uintptr_t)a.out & 15) == 0) {
    if (make_out_map(&my, a.out, L->act_dtype, a.out_cols, T_, a.ldo) == 0) a.tma_out = 1;
  }
#define QEFT_GL(B)                                                                                    \
  if (p.cg == 2) {                                                                                    \
    if (pair) return launch_gemm<MODE, B, T, 256, 2, 2>(m0, m1, mw, my, a, st);                            \
    return launch_gemm<MODE, B, T, 256, 1, 2>(m0, m1, mw, my, a, st);                                      \
  }                                                                                                   \
  if (pair) return launch_gemm<MODE, B, T, 256, 2, 1>(m0, m1, mw, my, a, st);                              \
  return big ? launch_gemm<MODE, B, T, 256, 1, 1>(m0, m1, mw, my, a, st) : launch_gemm<MODE, B, T, 128, 1, 1>(m0, m1, mw, my, a, st);
  if (L->bits == 4) {
    QEFT_GL(4)
  }
  QEFT_GL(3)
#undef QEFT_GL
}

GemmArgs base_args(const qeft_linear_t* L, int T_) {
  GemmArgs a{};
  a.qw = (const uint8_t*)L->qweight;
  a.sz = (const float2*)L->sz;
  a.weak16 = L->weak16;
  a.colmap = L->colmap;
  a.oc = L->oc; a.m = L->m; a.m_pad = L->m_pad; a.k = L->k; a.k_pad = L->k_pad;
  a.g = L->g; a.ng = L->ng;
  a.g_shift = (L->g & (L->g - 1)) == 0 ? __builtin_ctz((unsigned)L->g) : -1;
  a.T = T_;
  return a;
}

}  // namespace

namespace qeft {

// cluster size (token splits) of the wgrad reduction: a power of two <= 8 so that the clusters
// of all channel blocks fit one wave, with >= 4 k-blocks per split
int wgrad_splits(int oc, int T_) {
  const int mb = (oc + BM - 1) / BM, nkb = (T_ + 63) / 64;
  static const int forced = getenv("QEFT_WGRAD_SPLITS") ? atoi(getenv("QEFT_WGRAD_SPLITS")) : 0;  // tuning
  int lim = forced > 0 ? forced : std::min(num_sms() / mb, nkb / 4);
  lim = std::max(1, std::min(lim, 8));
  int s = 1;
  while (s * 2 <= lim) s *= 2;
  return s;
}

int gemm_set_schedule(int what, int value) {
  if (what == QEFT_SCHED_STREAMK) {
    const int prev = g_sk_mode;
    g_sk_mode = value < 0 ? -1 : (value > 0 ? 1 : 0);
    return prev;
  }
  if (what == QEFT_SCHED_CTA_PAIRS) {
    const int prev = g_cg_mode;
    g_cg_mode = value == 2 ? 2 : 1;
    return prev;
  }
  set_error("gemm_set_schedule: unknown setting %d", what);
  return QEFT_ERR_SHAPE;
}

size_t gemm_workspace_bytes(const qeft_linear_t* L, int T_) {
  // gathered activations in B200 K order (fwd, non-structured layouts), weak columns
  // (wgrad), or a 16-byte-pitched copy of dY (dgrad/wgrad when oc % 8 != 0)
  // fwd: gathered x [T][m_pad + k_pad]; dgrad: pitched dY [T][pad(oc, 8)] then B200-order dX
  // [T][m_pad + k_pad] (non-structured layouts); wgrad: x weak columns then pitched dY
  const size_t kk = (size_t)(L->m_pad + L->k_pad);
  return (size_t)T_ * (kk + pad_to(L->oc, 8) + L->k_pad) * 2 + 2048;
}

// dY with a row pitch TMA cannot address -> copy into ws with pitch roundup(oc, 8)
static int pitch_dy(const qeft_linear_t* L, const void*& dy, int64_t& lddy, int T_, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
  if (lddy % 8 == 0 && ((uintptr_t)dy & 15) == 0) return 0;
  const int ld = pad_to(L->oc, 8);
  QEFT_CHECK(ws_bytes >= (size_t)T_ * ld * 2, QEFT_ERR_SHAPE, "workspace too small for dY copy");
  QEFT_CUDA(cudaMemset2DAsync(ws, (size_t)ld * 2, 0, (size_t)ld * 2, T_, st));
  QEFT_CUDA(cudaMemcpy2DAsync(ws, (size_t)ld * 2, dy, (size_t)lddy * 2, (size_t)L->oc * 2, T_,
                              cudaMemcpyDeviceToDevice, st));
  dy = ws;
  lddy = ld;
  return 0;
}

int gemm_fwd(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int T_, void* ws,
             size_t ws_bytes, cudaStream_t st) {
  QEFT_CHECK(T_ >= 1, QEFT_ERR_SHAPE, "gemm_fwd: T=%d", T_);
  QEFT_CHECK(ldx >= L->ic && ldy >= L->oc, QEFT_ERR_SHAPE, "gemm_fwd: ld too small");
  GemmArgs a = base_args(L, T_);
  a.n_mblk = (L->oc_pad + BM - 1) / BM;
  a.kq = L->m_pad / BK;
  a.n_kblk = a.kq + L->k_pad / BK;
  a.out = y;
  a.ldo = ldy;
  a.out_cols = L->oc;
  CUtensorMap m0, m1;
  const bool fast = (L->flags & QEFT_FLAG_STRUCTURED_FAST) && ldx % 8 == 0 && ((uintptr_t)x & 15) == 0;
  const GemmPlan plan = gemm_plan(a.n_mblk, T_, a.n_kblk);
  const int box = plan.bn / plan.cg;
  if (fast) {
    if (int r = make_map(&m0, x, L->act_dtype, L->m, T_, ldx, box)) return r;
    const void* xw = (const char*)x + (size_t)L->m * 2;
    if (int r = make_map(&m1, xw, L->act_dtype, std::max(L->k, 1), T_, ldx, box)) return r;
  } else {
    const int kk = L->m_pad + L->k_pad;
    QEFT_CHECK(ws_bytes >= (size_t)T_ * kk * 2, QEFT_ERR_SHAPE, "gemm_fwd: workspace too small");
    if (int r = gather_rows(x, ldx, L->ic, L->colmap, kk, T_, L->act_dtype, ws, st)) return r;
    if (int r = make_map(&m0, ws, L->act_dtype, kk, T_, kk, box)) return r;
    m1 = m0;
    a.gathered = 1;
  }
  if (L->act_dtype == QEFT_F16) return dispatch_gemm<MODE_FWD, __half>(L, T_, plan, m0, m1, a, st);
  return dispatch_gemm<MODE_FWD, __nv_bfloat16>(L, T_, plan, m0, m1, a, st);
}

int gemm_dgrad(const qeft_linear_t* L, const void* dy, int64_t lddy, void* dx, int64_t lddx, int T_,
               int accumulate, void* ws, size_t ws_bytes, cudaStream_t st) {
  QEFT_CHECK(T_ >= 1, QEFT_ERR_SHAPE, "gemm_dgrad: T=%d", T_);
  QEFT_CHECK(lddy >= L->oc && lddx >= L->ic, QEFT_ERR_SHAPE, "gemm_dgrad: ld too small");
  if (int r = pitch_dy(L, dy, lddy, T_, ws, ws_bytes, st)) return r;
  GemmArgs a = base_args(L, T_);
  a.n_mblk = (L->m_pad + L->k_pad + BM - 1) / BM;
  a.kq = L->m_pad / BM;
  a.n_kblk = (L->oc_pad + BK - 1) / BK;
  a.out = dx;
  a.ldo = lddx;
  a.accumulate = accumulate;
  a.out_cols = L->ic;
  a.fast_out = (L->flags & QEFT_FLAG_STRUCTURED_FAST) && (L->m % 32 == 0);
  // non-structured layouts (irregular W_O, online reorder): dX in B200 order into the workspace
  // by TMA-store blocks, then one row-staged scatter through the column map (+ accumulate)
  const int kk = L->m_pad + L->k_pad;
  const size_t dy_bytes = (dy == ws) ? (((size_t)T_ * pad_to(L->oc, 8) * 2 + 255) & ~(size_t)255) : 0;
  void* dxb = (char*)ws + dy_bytes;
  const bool b200 = !a.fast_out && ws != nullptr && ws_bytes >= dy_bytes + (size_t)T_ * kk * 2 &&
                    (((uintptr_t)dxb) & 15) == 0 && getenv("QEFT_GEMM_SCATTER_EPI") == nullptr;
  if (b200) {
    a.b200_out = 1;
    a.out = dxb;
    a.ldo = kk;
    a.out_cols = kk;
    a.accumulate = 0;
  }
  CUtensorMap m0;
  const GemmPlan plan = gemm_plan(a.n_mblk, T_, a.n_kblk);
  if (int r = make_map(&m0, dy, L->act_dtype, L->oc, T_, lddy, plan.bn / plan.cg)) return r;
  int r = L->act_dtype == QEFT_F16 ? dispatch_gemm<MODE_DGRAD, __half>(L, T_, plan, m0, m0, a, st)
                                   : dispatch_gemm<MODE_DGRAD, __nv_bfloat16>(L, T_, plan, m0, m0, a, st);
  if (r || !b200) return r;
  return scatter_rows(dxb, kk, L->colmap, L->ic, T_, L->act_dtype, dx, lddx, accumulate, st);
}

template <typename T, int NW>
int launch_wgrad(const WgradGroup& g, const CUtensorMap& mx, int k, int T_, int acc, int vec, cudaStream_t st);

int dispatch_wgrad(const qeft_linear_t* L, const WgradGroup& g, const CUtensorMap& mx, int T_, int acc, int vec,
                   cudaStream_t st) {
  const int nw = L->k_pad / 64;
  const bool bf = L->act_dtype == QEFT_BF16;
#define QEFT_WG(NW)                                                                        \
  if (nw == NW)                                                                            \
    return bf ? launch_wgrad<__nv_bfloat16, NW>(g, mx, L->k, T_, acc, vec, st)              \
              : launch_wgrad<__half, NW>(g, mx, L->k, T_, acc, vec, st);
  QEFT_WG(1) QEFT_WG(2) QEFT_WG(3) QEFT_WG(4)
#undef QEFT_WG
  set_error("gemm_wgrad: unsupported k_pad");
  return QEFT_ERR_LAYOUT;
}

template <typename T, int NW>
int launch_wgrad(const WgradGroup& g, const CUtensorMap& mx, int k, int T_, int acc, int vec,
                 cudaStream_t st) {
  const size_t smem = WgradShape<NW>::kSmem;
  auto kern = wgrad_kernel<T, NW>;
  static bool attr = false;
  if (!attr) {
    QEFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int nkb = (T_ + 63) / 64;
  const int blocks = g.blk_end[g.nl - 1];
  const int S = wgrad_splits(blocks * BM, T_);
  const int kbs = (nkb + S - 1) / S;
  QEFT_CUDA(launch_pdl_cluster(kern, dim3(S, blocks), dim3(192), smem, st, S, g, mx, k, T_, acc, kbs, vec));
  return 0;
}

int gemm_wgrad_weak_multi(const qeft_linear_t* const* Ls, int nl, const void* const* dys, const int64_t* lddys,
                          const void* x_weak, int64_t ldxw, float* const* dws, int T_, int accumulate,
                          cudaStream_t st) {
  QEFT_CHECK(nl >= 1 && nl <= kMaxWgLayers && T_ >= 1, QEFT_ERR_SHAPE, "wgrad_multi: %d layers", nl);
  const qeft_linear_t* L = Ls[0];
  if (L->k == 0) return 0;
  QEFT_CHECK(L->k_pad <= 256, QEFT_ERR_LAYOUT, "gemm_wgrad: k_pad=%d > 256", L->k_pad);
  QEFT_CHECK(ldxw >= L->k && ldxw % 8 == 0 && ((uintptr_t)x_weak & 15) == 0, QEFT_ERR_SHAPE,
             "wgrad_multi: x_weak needs a 16-byte aligned row pitch >= k");
  WgradGroup g{};
  g.nl = nl;
  int vec = L->k % 4 == 0;
  int blocks = 0;
  for (int l = 0; l < nl; ++l) {
    const qeft_linear_t* Li = Ls[l];
    QEFT_CHECK(Li->k == L->k && Li->k_pad == L->k_pad && Li->act_dtype == L->act_dtype, QEFT_ERR_SHAPE,
               "wgrad_multi: layer %d does not share the weak geometry", l);
    QEFT_CHECK(lddys[l] >= Li->oc && lddys[l] % 8 == 0 && ((uintptr_t)dys[l] & 15) == 0, QEFT_ERR_SHAPE,
               "wgrad_multi: dY of layer %d needs a 16-byte aligned row pitch", l);
    if (int r = make_map(&g.dy[l], dys[l], Li->act_dtype, Li->oc, T_, lddys[l], 64)) return r;
    g.dw[l] = dws[l];
    g.oc[l] = Li->oc;
    blocks += (Li->oc + BM - 1) / BM;
    g.blk_end[l] = blocks;
    vec = vec && (((uintptr_t)dws[l] & 15) == 0);
  }
  CUtensorMap mx;
  if (int r = make_map(&mx, x_weak, L->act_dtype, L->k, T_, ldxw, 64)) return r;
  return dispatch_wgrad(L, g, mx, T_, accumulate, vec, st);
}

int gemm_wgrad(const qeft_linear_t* L, const void* dy, int64_t lddy, const void* x, int64_t ldx, float* dw,
               int T_, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st, bool x_is_weak) {
  QEFT_CHECK(T_ >= 1, QEFT_ERR_SHAPE, "gemm_wgrad: T=%d", T_);
  if (L->k == 0) return 0;
  QEFT_CHECK(L->k_pad <= 256, QEFT_ERR_LAYOUT, "gemm_wgrad: k_pad=%d > 256", L->k_pad);
  CUtensorMap md, mx;
  // workspace: [weak columns of x (T x k_pad)] [pitched dY copy]
  const size_t xw_bytes = (size_t)T_ * L->k_pad * 2;
  const size_t dy_off = (xw_bytes + 255) & ~(size_t)255;
  void* ws_dy = (char*)ws + dy_off;
  const size_t ws_dy_bytes = ws_bytes > dy_off ? ws_bytes - dy_off : 0;
  if (int r = pitch_dy(L, dy, lddy, T_, ws_dy, ws_dy_bytes, st)) return r;
  if (int r = make_map(&md, dy, L->act_dtype, L->oc, T_, lddy, 64)) return r;
  const bool fast = (L->flags & QEFT_FLAG_STRUCTURED_FAST) && ldx % 8 == 0 && ((uintptr_t)x & 15) == 0;
  if (x_is_weak) {
    // the caller saved only x[:, weak] (T x k, row pitch ldx) in the forward pass
    QEFT_CHECK(ldx >= L->k && ldx % 8 == 0 && ((uintptr_t)x & 15) == 0, QEFT_ERR_SHAPE,
               "gemm_wgrad_weak: x_weak needs a 16-byte aligned row pitch >= k (ld=%lld)", (long long)ldx);
    if (int r = make_map(&mx, x, L->act_dtype, L->k, T_, ldx, 64)) return r;
  } else if (fast) {
    if (int r = make_map(&mx, (const char*)x + (size_t)L->m * 2, L->act_dtype, L->k, T_, ldx, 64)) return r;
  } else {
    QEFT_CHECK(ws_bytes >= xw_bytes, QEFT_ERR_SHAPE, "gemm_wgrad: workspace too small");
    if (int r = gather_rows(x, ldx, L->ic, L->colmap + L->m_pad, L->k_pad, T_, L->act_dtype, ws, st)) return r;
    if (int r = make_map(&mx, ws, L->act_dtype, L->k_pad, T_, L->k_pad, 64)) return r;
  }
  WgradGroup g{};
  g.dy[0] = md;
  g.dw[0] = dw;
  g.oc[0] = L->oc;
  g.blk_end[0] = (L->oc + BM - 1) / BM;
  g.nl = 1;
  const int vec = (L->k % 4 == 0) && (((uintptr_t)dw & 15) == 0);
  return dispatch_wgrad(L, g, mx, T_, accumulate, vec, st);
}

}  // namespace qeft
