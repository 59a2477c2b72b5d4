// Fused elementwise kernels of the fine-tuning step's host model (the non-linear
// parts around the QEFT linears, pkg/src/qeft/model.py:262-266 RMS-norm,
// 249-259 rotary, SwiGLU at 389-391), forward and backward, bf16/fp16 activations
// with fp32 math. Gains are frozen in weak-column tuning (tuning.py:187-248,
// backward_batch with param_grads=False), so the RMS-norm backward returns dX only.
// HBM-bound: each kernel reads and writes every element once.
#include <type_traits>

#include "qeft_common.cuh"
#include "qeft_internal.h"

using namespace qeft;

namespace {

constexpr float kRmsEps = 1e-5f;  // model.py:22

template <typename T>
QEFT_DEV float ld(const T* p) { return to_f32<T>(*p); }

// one CTA per row; 8 consecutive elements per thread per iteration (16-byte accesses)
template <typename T>
__global__ void rmsnorm_fwd_kernel(const T* __restrict__ x, const float* __restrict__ gain, T* __restrict__ y,
                                   float* __restrict__ rstd, int C) {
  __shared__ float red[32];
  const int row = blockIdx.x;
  const T* xr = x + (int64_t)row * C;
  T* yr = y + (int64_t)row * C;
  float ss = 0.f;
  for (int c = threadIdx.x * 8; c < C; c += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + c);
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float f = to_f32<T>(e[i]);
      ss += f * f;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = rsqrtf(v / (float)C + kRmsEps);
  }
  __syncthreads();
  const float r = red[0];
  if (threadIdx.x == 0) rstd[row] = r;
  for (int c = threadIdx.x * 8; c < C; c += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + c);
    const T* e = reinterpret_cast<const T*>(&v);
    uint4 o;
    T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int i = 0; i < 8; ++i) oe[i] = from_f32<T>(gain[c + i] * to_f32<T>(e[i]) * r);
    *reinterpret_cast<uint4*>(yr + c) = o;
  }
}

// dx = g*dy*r - x * r^3 * sum(g*dy*x) / C   (model.py:269-275, dgain not formed)
// optional accumulation: dx += residual gradient (fuses the residual add of the block)
template <typename T>
__global__ void rmsnorm_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ gain,
                                   const float* __restrict__ rstd, const T* __restrict__ dres, T* __restrict__ dx,
                                   int C) {
  __shared__ float red[32];
  const int row = blockIdx.x;
  const T* xr = x + (int64_t)row * C;
  const T* dyr = dy + (int64_t)row * C;
  const float r = rstd[row];
  float dot = 0.f;
  for (int c = threadIdx.x * 8; c < C; c += blockDim.x * 8) {
    const uint4 xv = *reinterpret_cast<const uint4*>(xr + c);
    const uint4 gv = *reinterpret_cast<const uint4*>(dyr + c);
    const T* xe = reinterpret_cast<const T*>(&xv);
    const T* ge = reinterpret_cast<const T*>(&gv);
#pragma unroll
    for (int i = 0; i < 8; ++i) dot += gain[c + i] * to_f32<T>(ge[i]) * to_f32<T>(xe[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float k = red[0] * r * r * r / (float)C;
  for (int c = threadIdx.x * 8; c < C; c += blockDim.x * 8) {
    const uint4 xv = *reinterpret_cast<const uint4*>(xr + c);
    const uint4 gv = *reinterpret_cast<const uint4*>(dyr + c);
    const T* xe = reinterpret_cast<const T*>(&xv);
    const T* ge = reinterpret_cast<const T*>(&gv);
    uint4 rv = make_uint4(0, 0, 0, 0);
    if (dres) rv = *reinterpret_cast<const uint4*>(dres + (int64_t)row * C + c);
    const T* re = reinterpret_cast<const T*>(&rv);
    uint4 o;
    T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float v = gain[c + i] * to_f32<T>(ge[i]) * r - to_f32<T>(xe[i]) * k;
      if (dres) v += to_f32<T>(re[i]);
      oe[i] = from_f32<T>(v);
    }
    *reinterpret_cast<uint4*>(dx + (int64_t)row * C + c) = o;
  }
}

// rotary on (rows = B*T tokens) x (H heads x hd): pairs (j, j + hd/2) of every head rotate by
// angle t * inv_freq[j] (model.py:256-259); dir = -1 applies the inverse (backward).
// One CTA per token row: the row's cos/sin are read once, 8 pairs per thread-iteration with
// 16-byte accesses (hd/2 % 8 == 0).
// P pairs per thread: 8 (16-byte vectors, head_dim % 16 == 0) or 1 (any even head_dim)
template <typename T, int P>
__global__ void rope_kernel(const T* __restrict__ in, T* __restrict__ out, const float* __restrict__ cosv,
                            const float* __restrict__ sinv, int T_, int H, int hd, float dir) {
  const int half = hd >> 1;
  const int64_t row = blockIdx.x;
  const int t = (int)(row % T_);
  const float* cr = cosv + (int64_t)t * half;
  const float* sr = sinv + (int64_t)t * half;
  const int chunks = half / P;  // P-pair chunks per head
  for (int e = threadIdx.x; e < H * chunks; e += blockDim.x) {
    const int h = e / chunks, j = (e - h * chunks) * P;
    const int64_t base = (row * H + h) * hd;
    T ae[P], be[P], oae[P], obe[P];
    if constexpr (P == 8) {
      *reinterpret_cast<uint4*>(ae) = *reinterpret_cast<const uint4*>(in + base + j);
      *reinterpret_cast<uint4*>(be) = *reinterpret_cast<const uint4*>(in + base + j + half);
    } else {
      ae[0] = in[base + j];
      be[0] = in[base + j + half];
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const float c = cr[j + i], s = dir * sr[j + i];
      const float a = to_f32<T>(ae[i]), b = to_f32<T>(be[i]);
      oae[i] = from_f32<T>(a * c - b * s);
      obe[i] = from_f32<T>(a * s + b * c);
    }
    if constexpr (P == 8) {
      *reinterpret_cast<uint4*>(out + base + j) = *reinterpret_cast<const uint4*>(oae);
      *reinterpret_cast<uint4*>(out + base + j + half) = *reinterpret_cast<const uint4*>(obe);
    } else {
      out[base + j] = oae[0];
      out[base + j + half] = obe[0];
    }
  }
}

// One decode step's rotary + KV-cache append (model.py:249-259, 372-380 at one position):
// q_out = rot(q), k_cache[b][h][pos] = rot(k), v_cache[b][h][pos] = v. q, k, v are (B, H*hd)
// GEMV outputs; caches (B, H, T_cache, hd). pos is read on device (one CUDA graph per step).
template <typename T>
__global__ void rope_kv_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                               T* __restrict__ q_out, T* __restrict__ kc, T* __restrict__ vc,
                               const float* __restrict__ cosv, const float* __restrict__ sinv,
                               const int64_t* __restrict__ pos_dev, int H, int hd, int T_cache) {
  const int b = blockIdx.x, half = hd >> 1;
  const int64_t pos = *pos_dev;
  const float* cr = cosv + pos * half;
  const float* sr = sinv + pos * half;
  for (int e = threadIdx.x; e < H * half; e += blockDim.x) {
    const int h = e / half, j = e - h * half;
    const int64_t src = ((int64_t)b * H + h) * hd;
    const int64_t dst = (((int64_t)b * H + h) * T_cache + pos) * hd;
    const float c = cr[j], s = sr[j];
    float a = to_f32<T>(q[src + j]), bb = to_f32<T>(q[src + j + half]);
    q_out[src + j] = from_f32<T>(a * c - bb * s);
    q_out[src + j + half] = from_f32<T>(a * s + bb * c);
    a = to_f32<T>(k[src + j]);
    bb = to_f32<T>(k[src + j + half]);
    kc[dst + j] = from_f32<T>(a * c - bb * s);
    kc[dst + j + half] = from_f32<T>(a * s + bb * c);
    vc[dst + j] = v[src + j];
    vc[dst + j + half] = v[src + j + half];
  }
}

// One decode step's attention, with the rotary + KV-cache append fused in (model.py:249-275
// rotary, the engine's causal softmax attention): grid (head, batch, split). Every CTA rotates q
// at the device position; the split holding position pos also rotates the new k and appends
// k/v to the caches. Each split attends to its contiguous chunk of positions 0..pos with an
// fp32 online softmax: half-warps own positions (16 lanes x 8 dims, 16-byte loads), K and V of
// UNR positions are loaded together, the 32 half-warp states are merged in shared memory, and
// the split's (max, sum, o) goes to the scratch; the last split to finish (a per-head counter)
// merges the splits in split order (deterministic), writes o and re-arms the counter.
constexpr int kAttnSplits = 4;

template <typename T, int HD>
__global__ void __launch_bounds__(512) decode_attn_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                          const T* __restrict__ v, T* __restrict__ kc,
                                                          T* __restrict__ vc, const float* __restrict__ cosv,
                                                          const float* __restrict__ sinv,
                                                          const int64_t* __restrict__ pos_dev, T* __restrict__ o,
                                                          float* __restrict__ scratch, int* __restrict__ counters,
                                                          int H, int T_cache, float scale) {
  constexpr int DPL = HD / 16;  // dims per lane of a half-warp
  constexpr int HALF = HD / 2;
  constexpr int UNR = 8;
  constexpr int NHW = 512 / 16;  // half-warps
  constexpr int PART = HD + 2;   // scratch floats per split: o[HD], max, sum
  static_assert(DPL == 8, "16-byte lanes: HD = 128");
  __shared__ __align__(16) T qs[HD];
  __shared__ float s_m[NHW], s_l[NHW];
  __shared__ __align__(16) float s_o[NHW][HD];
  __shared__ int s_last;
  const int h = blockIdx.x, b = blockIdx.y, split = blockIdx.z, S = gridDim.z;
  const int pos = (int)*pos_dev;
  const int n = pos + 1;
  const int c0 = (int)((int64_t)split * n / S), c1 = (int)((int64_t)(split + 1) * n / S);
  const int64_t src = ((int64_t)b * H + h) * HD;
  const int64_t crow = ((int64_t)b * H + h) * T_cache;
  const int hw = threadIdx.x >> 4, l16 = threadIdx.x & 15;
  const T* kbase = kc + crow * HD + l16 * DPL;
  const T* vbase = vc + crow * HD + l16 * DPL;
  // before the grid dependency: the rotary constants and the first UNR cached rows of this
  // half-warp (rows < pos were written by earlier steps; row pos is appended below)
  float cs = 0.f, sn = 0.f;
  if (threadIdx.x < HALF) {
    cs = cosv[(int64_t)pos * HALF + threadIdx.x];
    sn = sinv[(int64_t)pos * HALF + threadIdx.x];
  }
  uint4 kv[UNR], vv[UNR];
  const int t00 = c0 + (hw & ~1);
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const int t = t00 + (hw & 1) + u * NHW;
    kv[u] = make_uint4(0u, 0u, 0u, 0u);
    vv[u] = kv[u];
    if (t < c1 && t < pos) {
      kv[u] = __ldcg(reinterpret_cast<const uint4*>(kbase + (int64_t)t * HD));
      vv[u] = __ldcg(reinterpret_cast<const uint4*>(vbase + (int64_t)t * HD));
    }
  }
  pdl_launch_dependents();
  pdl_wait();  // q / k / v come from the preceding projection
  if (threadIdx.x < HALF) {
    const int j = threadIdx.x;
    const float c = cs, s = sn;
    float a = to_f32<T>(q[src + j]), bb = to_f32<T>(q[src + j + HALF]);
    qs[j] = from_f32<T>(a * c - bb * s);
    qs[j + HALF] = from_f32<T>(a * s + bb * c);
    if (c1 == n) {  // this split's chunk ends at pos: append the new row
      a = to_f32<T>(k[src + j]);
      bb = to_f32<T>(k[src + j + HALF]);
      kc[(crow + pos) * HD + j] = from_f32<T>(a * c - bb * s);
      kc[(crow + pos) * HD + j + HALF] = from_f32<T>(a * s + bb * c);
      vc[(crow + pos) * HD + j] = v[src + j];
      vc[(crow + pos) * HD + j + HALF] = v[src + j + HALF];
    }
  }
  __syncthreads();  // rotated q in shared memory, the new cache row written (same CTA)
  float qf[DPL];
  {
    const uint4 qv = *reinterpret_cast<const uint4*>(qs + l16 * DPL);
    const T* e = reinterpret_cast<const T*>(&qv);
#pragma unroll
    for (int i = 0; i < DPL; ++i) qf[i] = to_f32<T>(e[i]);
  }
  float m = -INFINITY, lsum = 0.f, acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
  // warp-uniform trip count (the even half-warp's positions); the odd half masks its tail
  for (int t0 = t00; t0 < c1; t0 += NHW * UNR) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = t0 + (hw & 1) + u * NHW;
      // the first iteration's rows were prefetched, except the one appended above
      if (t < c1 && (t0 != t00 || t >= pos)) {
        kv[u] = __ldcg(reinterpret_cast<const uint4*>(kbase + (int64_t)t * HD));
        vv[u] = __ldcg(reinterpret_cast<const uint4*>(vbase + (int64_t)t * HD));
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = t0 + (hw & 1) + u * NHW;
      const T* ke = reinterpret_cast<const T*>(&kv[u]);
      float d = 0.f;
#pragma unroll
      for (int i = 0; i < DPL; ++i) d = fmaf(qf[i], to_f32<T>(ke[i]), d);
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
      if (t < c1) {
        const float sc = d * scale;
        const float mn = fmaxf(m, sc);
        const float corr = __expf(m - mn), p = __expf(sc - mn);
        lsum = lsum * corr + p;
        const T* ve = reinterpret_cast<const T*>(&vv[u]);
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[i] = fmaf(p, to_f32<T>(ve[i]), acc[i] * corr);
        m = mn;
      }
    }
  }
  if (l16 == 0) {
    s_m[hw] = m;
    s_l[hw] = lsum;
  }
#pragma unroll
  for (int i = 0; i < DPL; ++i) s_o[hw][l16 * DPL + i] = acc[i];
  __syncthreads();
  // this split's state: merge the half-warps in order
  float* part = scratch + (((int64_t)b * H + h) * S + split) * PART;
  if (threadIdx.x < HD) {
    float M = -INFINITY;
    for (int w = 0; w < NHW; ++w) M = fmaxf(M, s_m[w]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < NHW; ++w) {
      if (s_m[w] == -INFINITY) continue;  // a half-warp with no position
      const float f = __expf(s_m[w] - M);
      L += s_l[w] * f;
      O += s_o[w][threadIdx.x] * f;
    }
    part[threadIdx.x] = O;
    if (threadIdx.x == 0) {
      part[HD] = M;
      part[HD + 1] = L;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counters + (int64_t)b * H + h, 1) == S - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < HD) {
    const float* p0 = scratch + ((int64_t)b * H + h) * S * PART;
    float M = -INFINITY;
    for (int sp = 0; sp < S; ++sp) M = fmaxf(M, __ldcg(p0 + sp * PART + HD));
    float L = 0.f, O = 0.f;
    for (int sp = 0; sp < S; ++sp) {
      const float ms = __ldcg(p0 + sp * PART + HD);
      if (ms == -INFINITY) continue;  // an empty split
      const float f = __expf(ms - M);
      L += __ldcg(p0 + sp * PART + HD + 1) * f;
      O += __ldcg(p0 + sp * PART + threadIdx.x) * f;
    }
    o[src + threadIdx.x] = from_f32<T>(O / L);
  }
  if (threadIdx.x == 0) counters[(int64_t)b * H + h] = 0;
}

// f = silu(g) * u (SwiGLU, model.py:389-391) and its backward
template <typename T>
__global__ void silu_mul_fwd_kernel(const T* __restrict__ g, const T* __restrict__ u, T* __restrict__ f, int64_t n) {
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += (int64_t)gridDim.x * blockDim.x * 8) {
    const uint4 gv = *reinterpret_cast<const uint4*>(g + i);
    const uint4 uv = *reinterpret_cast<const uint4*>(u + i);
    const T* ge = reinterpret_cast<const T*>(&gv);
    const T* ue = reinterpret_cast<const T*>(&uv);
    uint4 o;
    T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float x = to_f32<T>(ge[k]);
      oe[k] = from_f32<T>(x / (1.f + __expf(-x)) * to_f32<T>(ue[k]));
    }
    *reinterpret_cast<uint4*>(f + i) = o;
  }
}

template <typename T>
__global__ void silu_mul_bwd_kernel(const T* __restrict__ df, const T* __restrict__ g, const T* __restrict__ u,
                                    T* __restrict__ dg, T* __restrict__ du, int64_t n) {
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += (int64_t)gridDim.x * blockDim.x * 8) {
    const uint4 fv = *reinterpret_cast<const uint4*>(df + i);
    const uint4 gv = *reinterpret_cast<const uint4*>(g + i);
    const uint4 uv = *reinterpret_cast<const uint4*>(u + i);
    const T* fe = reinterpret_cast<const T*>(&fv);
    const T* ge = reinterpret_cast<const T*>(&gv);
    const T* ue = reinterpret_cast<const T*>(&uv);
    uint4 og, ou;
    T* oge = reinterpret_cast<T*>(&og);
    T* oue = reinterpret_cast<T*>(&ou);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float x = to_f32<T>(ge[k]), d = to_f32<T>(fe[k]), uu = to_f32<T>(ue[k]);
      const float sg = 1.f / (1.f + __expf(-x));
      oue[k] = from_f32<T>(d * x * sg);                                // du = df * silu(g)
      oge[k] = from_f32<T>(d * uu * (sg * (1.f + x * (1.f - sg))));     // dg (model.py:438)
    }
    *reinterpret_cast<uint4*>(dg + i) = og;
    *reinterpret_cast<uint4*>(du + i) = ou;
  }
}

// Next-token cross-entropy over fp16/bf16 logits (the reference's fp32 log-softmax NLL,
// model.py:531-547): one CTA per row, the row read once into registers (16-byte vectors), fp32
// max / sum of exp by block reduction in a fixed order (deterministic), loss[row] = lse - z_t.
// The backward recomputes exp(z - lse) from the logits and the saved lse:
// dz = (softmax - onehot(t)) * g, written in the logits' dtype, g = dL/dloss / rows (device).
constexpr int kCeThreads = 512, kCeVec = 8;

template <int NT>
__device__ __forceinline__ float block_reduce(float v, float* sh, bool is_max) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, w) : v + w;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // sh reuse across calls
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  v = lane < NT / 32 ? sh[lane] : (is_max ? -INFINITY : 0.f);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, w) : v + w;
  }
  return v;
}

template <typename T, int PER>
__global__ void __launch_bounds__(kCeThreads) ce_fwd_kernel(const T* __restrict__ z, int64_t ldz, int V,
                                                            const int64_t* __restrict__ tgt, float* __restrict__ loss,
                                                            float* __restrict__ lse_out) {
  __shared__ float sh[32];
  const T* row = z + (int64_t)blockIdx.x * ldz;
  const int nv = V / kCeVec;
  uint4 v[PER];
  float m = -INFINITY;
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int i = threadIdx.x + p * kCeThreads;
    if (i < nv) {
      v[p] = *reinterpret_cast<const uint4*>(row + (int64_t)i * kCeVec);
      const T* e = reinterpret_cast<const T*>(&v[p]);
#pragma unroll
      for (int k = 0; k < kCeVec; ++k) m = fmaxf(m, to_f32<T>(e[k]));
    }
  }
  m = block_reduce<kCeThreads>(m, sh, true);
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int i = threadIdx.x + p * kCeThreads;
    if (i < nv) {
      const T* e = reinterpret_cast<const T*>(&v[p]);
#pragma unroll
      for (int k = 0; k < kCeVec; ++k) s += __expf(to_f32<T>(e[k]) - m);
    }
  }
  s = block_reduce<kCeThreads>(s, sh, false);
  if (threadIdx.x == 0) {
    const float lse = m + __logf(s);
    lse_out[blockIdx.x] = lse;
    loss[blockIdx.x] = lse - to_f32<T>(row[tgt[blockIdx.x]]);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) ce_bwd_kernel(const T* __restrict__ z, int64_t ldz, int V,
                                                     const int64_t* __restrict__ tgt, const float* __restrict__ lse,
                                                     const float* __restrict__ gscale, T* __restrict__ dz,
                                                     int64_t lddz) {
  const T* row = z + (int64_t)blockIdx.y * ldz;
  T* drow = dz + (int64_t)blockIdx.y * lddz;
  const float l = lse[blockIdx.y], g = *gscale;
  const int t = (int)tgt[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V / kCeVec; i += gridDim.x * blockDim.x) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + (int64_t)i * kCeVec);
    const T* e = reinterpret_cast<const T*>(&v);
    uint4 o;
    T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int k = 0; k < kCeVec; ++k) {
      const float p = __expf(to_f32<T>(e[k]) - l) - (i * kCeVec + k == t ? 1.f : 0.f);
      oe[k] = from_f32<T>(p * g);
    }
    *reinterpret_cast<uint4*>(drow + (int64_t)i * kCeVec) = o;
  }
}

int grid_for(int64_t n, int per_thread) {
  const int64_t blocks = (n / per_thread + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 16));
}

}  // namespace

namespace qeft {

int rmsnorm_fwd(const void* x, const float* gain, void* y, float* rstd, int rows, int C, int dt, cudaStream_t st) {
  QEFT_CHECK(C % 8 == 0 && rows >= 0, QEFT_ERR_SHAPE, "rmsnorm: C=%d must be a multiple of 8", C);
  if (!rows) return 0;
  const int thr = std::min(1024, std::max(32, C / 8 / 32 * 32));
  if (dt == QEFT_BF16)
    rmsnorm_fwd_kernel<__nv_bfloat16><<<rows, thr, 0, st>>>((const __nv_bfloat16*)x, gain, (__nv_bfloat16*)y, rstd, C);
  else
    rmsnorm_fwd_kernel<__half><<<rows, thr, 0, st>>>((const __half*)x, gain, (__half*)y, rstd, C);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int rmsnorm_bwd(const void* dy, const void* x, const float* gain, const float* rstd, const void* dres, void* dx,
                int rows, int C, int dt, cudaStream_t st) {
  QEFT_CHECK(C % 8 == 0 && rows >= 0, QEFT_ERR_SHAPE, "rmsnorm: C=%d must be a multiple of 8", C);
  if (!rows) return 0;
  const int thr = std::min(1024, std::max(32, C / 8 / 32 * 32));
  if (dt == QEFT_BF16)
    rmsnorm_bwd_kernel<__nv_bfloat16><<<rows, thr, 0, st>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, gain,
                                                           rstd, (const __nv_bfloat16*)dres, (__nv_bfloat16*)dx, C);
  else
    rmsnorm_bwd_kernel<__half><<<rows, thr, 0, st>>>((const __half*)dy, (const __half*)x, gain, rstd,
                                                    (const __half*)dres, (__half*)dx, C);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int rope_kv(const void* q, const void* k, const void* v, void* q_out, void* kc, void* vc, const float* cosv,
            const float* sinv, const int64_t* pos_dev, int B, int H, int hd, int T_cache, int dt, cudaStream_t st) {
  QEFT_CHECK(hd % 2 == 0 && hd > 0 && B >= 1 && H >= 1 && T_cache >= 1, QEFT_ERR_SHAPE,
             "rope_kv: B=%d H=%d hd=%d T=%d", B, H, hd, T_cache);
  const int thr = std::min(512, std::max(32, H * hd / 2));
  if (dt == QEFT_BF16)
    rope_kv_kernel<__nv_bfloat16><<<B, thr, 0, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                     (const __nv_bfloat16*)v, (__nv_bfloat16*)q_out,
                                                     (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, cosv, sinv, pos_dev,
                                                     H, hd, T_cache);
  else
    rope_kv_kernel<__half><<<B, thr, 0, st>>>((const __half*)q, (const __half*)k, (const __half*)v, (__half*)q_out,
                                              (__half*)kc, (__half*)vc, cosv, sinv, pos_dev, H, hd, T_cache);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

size_t decode_attention_workspace_bytes(int B, int H, int hd) {
  // counters [B*H] (zero between calls; the kernel re-arms them), then the split partials
  return 256 + (((size_t)B * H * 4 + 63) & ~(size_t)63) + (size_t)B * H * kAttnSplits * (hd + 2) * 4;
}

int decode_attention(const void* q, const void* k, const void* v, void* kc, void* vc, const float* cosv,
                     const float* sinv, const int64_t* pos_dev, void* o, int B, int H, int hd, int T_cache, int dt,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  QEFT_CHECK(hd == 128 && B >= 1 && H >= 1 && T_cache >= 1, QEFT_ERR_SHAPE,
             "decode_attention: hd=%d (128 supported), B=%d H=%d T=%d", hd, B, H, T_cache);
  QEFT_CHECK(ws != nullptr && ws_bytes >= decode_attention_workspace_bytes(B, H, hd) && ((uintptr_t)ws & 15) == 0,
             QEFT_ERR_SHAPE, "decode_attention: workspace too small");
  int* counters = (int*)ws;
  float* scratch = (float*)((char*)ws + 256 + (((size_t)B * H * 4 + 63) & ~(size_t)63));
  const float scale = 1.f / sqrtf((float)hd);
  const dim3 grid(H, B, kAttnSplits);
  if (dt == QEFT_BF16)
    QEFT_CUDA(launch_pdl(decode_attn_kernel<__nv_bfloat16, 128>, grid, dim3(512), 0, st, (const __nv_bfloat16*)q,
                         (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, cosv,
                         sinv, pos_dev, (__nv_bfloat16*)o, scratch, counters, H, T_cache, scale));
  else
    QEFT_CUDA(launch_pdl(decode_attn_kernel<__half, 128>, grid, dim3(512), 0, st, (const __half*)q, (const __half*)k,
                         (const __half*)v, (__half*)kc, (__half*)vc, cosv, sinv, pos_dev, (__half*)o, scratch,
                         counters, H, T_cache, scale));
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int rope(const void* in, void* out, const float* cosv, const float* sinv, int64_t rows, int T_, int H, int hd,
         int inverse, int dt, cudaStream_t st) {
  QEFT_CHECK(hd % 2 == 0 && hd > 0 && T_ > 0, QEFT_ERR_SHAPE, "rope: head_dim %d must be even", hd);
  if (!rows) return 0;
  const float dir = inverse ? -1.f : 1.f;
  const bool vec = hd % 16 == 0 && ((uintptr_t)in & 15) == 0 && ((uintptr_t)out & 15) == 0;
  const int thr = std::min(256, std::max(32, H * (vec ? hd / 16 : hd / 2)));
  auto go = [&](auto tag, auto p) {
    using T = decltype(tag);
    rope_kernel<T, decltype(p)::value><<<(unsigned)rows, thr, 0, st>>>((const T*)in, (T*)out, cosv, sinv, T_, H, hd,
                                                                       dir);
  };
  if (dt == QEFT_BF16) {
    if (vec) go(__nv_bfloat16{}, std::integral_constant<int, 8>{});
    else go(__nv_bfloat16{}, std::integral_constant<int, 1>{});
  } else {
    if (vec) go(__half{}, std::integral_constant<int, 8>{});
    else go(__half{}, std::integral_constant<int, 1>{});
  }
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int cross_entropy_fwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, float* loss, float* lse,
                      int dt, cudaStream_t st) {
  QEFT_CHECK(V % kCeVec == 0 && ldz % kCeVec == 0 && V > 0 && rows >= 0, QEFT_ERR_SHAPE,
             "cross_entropy: V=%d and ld=%lld must be multiples of 8", V, (long long)ldz);
  QEFT_CHECK(V <= 16 * kCeThreads * kCeVec, QEFT_ERR_SHAPE, "cross_entropy: V=%d > %d", V, 16 * kCeThreads * kCeVec);
  if (!rows) return 0;
  const int per = (V / kCeVec + kCeThreads - 1) / kCeThreads;
  auto go = [&](auto tag, auto perc) {
    using T = decltype(tag);
    ce_fwd_kernel<T, decltype(perc)::value><<<rows, kCeThreads, 0, st>>>((const T*)z, ldz, V, tgt, loss, lse);
  };
#define QEFT_CE(P)                                                                              \
  if (per <= P) {                                                                               \
    if (dt == QEFT_BF16) go(__nv_bfloat16{}, std::integral_constant<int, P>{});                 \
    else go(__half{}, std::integral_constant<int, P>{});                                        \
  } else
  QEFT_CE(2) QEFT_CE(4) QEFT_CE(8) QEFT_CE(16) {}
#undef QEFT_CE
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int cross_entropy_bwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, const float* lse,
                      const float* gscale, void* dz, int64_t lddz, int dt, cudaStream_t st) {
  QEFT_CHECK(V % kCeVec == 0 && ldz % kCeVec == 0 && lddz % kCeVec == 0 && V > 0, QEFT_ERR_SHAPE,
             "cross_entropy_bwd: V=%d and lds must be multiples of 8", V);
  if (!rows) return 0;
  const dim3 grid((V / kCeVec + 255) / 256, rows);
  if (dt == QEFT_BF16)
    ce_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)z, ldz, V, tgt, lse, gscale,
                                                       (__nv_bfloat16*)dz, lddz);
  else
    ce_bwd_kernel<__half><<<grid, 256, 0, st>>>((const __half*)z, ldz, V, tgt, lse, gscale, (__half*)dz, lddz);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int silu_mul_fwd(const void* g, const void* u, void* f, int64_t n, int dt, cudaStream_t st) {
  QEFT_CHECK(n % 8 == 0, QEFT_ERR_SHAPE, "silu_mul: n=%lld must be a multiple of 8", (long long)n);
  if (!n) return 0;
  if (dt == QEFT_BF16)
    silu_mul_fwd_kernel<__nv_bfloat16><<<grid_for(n, 8), 256, 0, st>>>((const __nv_bfloat16*)g, (const __nv_bfloat16*)u,
                                                                       (__nv_bfloat16*)f, n);
  else
    silu_mul_fwd_kernel<__half><<<grid_for(n, 8), 256, 0, st>>>((const __half*)g, (const __half*)u, (__half*)f, n);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

int silu_mul_bwd(const void* df, const void* g, const void* u, void* dg, void* du, int64_t n, int dt,
                 cudaStream_t st) {
  QEFT_CHECK(n % 8 == 0, QEFT_ERR_SHAPE, "silu_mul: n=%lld must be a multiple of 8", (long long)n);
  if (!n) return 0;
  if (dt == QEFT_BF16)
    silu_mul_bwd_kernel<__nv_bfloat16><<<grid_for(n, 8), 256, 0, st>>>(
        (const __nv_bfloat16*)df, (const __nv_bfloat16*)g, (const __nv_bfloat16*)u, (__nv_bfloat16*)dg,
        (__nv_bfloat16*)du, n);
  else
    silu_mul_bwd_kernel<__half><<<grid_for(n, 8), 256, 0, st>>>((const __half*)df, (const __half*)g, (const __half*)u,
                                                                (__half*)dg, (__half*)du, n);
  QEFT_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace qeft
