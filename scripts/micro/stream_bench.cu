// Streaming microbenchmark: which load pattern reaches HBM peak on B200?
// A: LDG.128 unrolled; B: cp.async.bulk ring (consumers only wait/arrive);
// C: B with bigger/smaller stages. Prints GB/s per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_08661_b200/csrc/qeft_common.cuh"
using namespace qeft;

template <int U>
__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  unsigned acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_stream(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

// per CTA: contiguous chunk of `per_cta` bytes streamed through S slots of B bytes
__global__ void bulk_kernel(const uint8_t* p, size_t per_cta, int B, int S, int nwarps, unsigned* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = (int)(per_cta / B);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], nwarps); }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* base = p + (size_t)blockIdx.x * per_cta;
  if (warp == nwarps) {
    if (lane == 0) {
      for (int s = 0; s < nst; ++s) {
        int slot = s % S;
        if (s >= S) mbar_wait(&empty[slot], ((s / S) - 1) & 1);
        mbar_expect_tx(&full[slot], B);
        bulk_g2s(smem + (size_t)slot * B, base + (size_t)s * B, B, &full[slot]);
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int s = 0; s < nst; ++s) {
    int slot = s % S;
    mbar_wait(&full[slot], (s / S) & 1);
    const uint4* q = reinterpret_cast<const uint4*>(smem + (size_t)slot * B);
    for (int i = warp * 32 + lane; i < B / 16; i += nwarps * 32) { uint4 v = q[i]; acc ^= v.x ^ v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 0x12345678) out[0] = acc;
}

// producer lanes: lane l issues stages s with s % P == l (each lane its own slots)
__global__ void bulk_multi_kernel(const uint8_t* p, size_t per_cta, int B, int S, int P, unsigned* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const int nwarps = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = (int)(per_cta / B);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], nwarps); }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* base = p + (size_t)blockIdx.x * per_cta;
  if (warp == nwarps) {
    if (lane < P) {
      for (int s = lane; s < nst; s += P) {
        int slot = s % S;
        if (s >= S) mbar_wait(&empty[slot], ((s / S) - 1) & 1);
        mbar_expect_tx(&full[slot], B);
        bulk_g2s(smem + (size_t)slot * B, base + (size_t)s * B, B, &full[slot]);
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int s = 0; s < nst; ++s) {
    int slot = s % S;
    mbar_wait(&full[slot], (s / S) & 1);
    const uint4* q = reinterpret_cast<const uint4*>(smem + (size_t)slot * B);
    for (int i = warp * 32 + lane; i < B / 16; i += nwarps * 32) { uint4 v = q[i]; acc ^= v.x ^ v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 0x12345678) out[0] = acc;
}

// warp-per-stream LDG: each warp streams its own contiguous region, U loads in flight per lane
template <int U>
__global__ void ldg_warp_kernel(const uint4* __restrict__ p, size_t per_warp16, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const size_t w = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint4* b = p + w * per_warp16;
  unsigned acc = 0;
  for (size_t i = lane; i + 32 * (U - 1) < per_warp16; i += 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_stream(b + i + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  size_t bytes = 1ull << 30;  // 1 GiB >> L2
  uint8_t* d; unsigned* o;
  cudaMalloc(&d, bytes); cudaMalloc(&o, 4);
  cudaMemset(d, 1, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto fn) { fn(); cudaDeviceSynchronize(); cudaEventRecord(e0); for (int r = 0; r < 5; ++r) fn(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return bytes * 5 / (ms * 1e-3) / 1e9; };
  for (int blocks : {148, 296, 592, 1184}) for (int thr : {256, 512}) {
    double g = timeit([&] { ldg_kernel<4><<<blocks, thr>>>((const uint4*)d, bytes / 16, o); });
    printf("LDG U4 blocks=%d thr=%d : %.0f GB/s\n", blocks, thr, g);
  }
  double g8 = timeit([&] { ldg_kernel<8><<<592, 512>>>((const uint4*)d, bytes / 16, o); });
  printf("LDG U8 592x512 : %.0f GB/s\n", g8);
  for (int wps : {4, 8, 16}) for (int thr : {128, 256}) {
    int blocks = 148 * wps * 32 / thr; size_t nw = (size_t)blocks * thr / 32; size_t per = bytes / 16 / nw / 256 * 256;
    double g = timeit([&] { ldg_warp_kernel<8><<<blocks, thr>>>((const uint4*)d, per, o); });
    printf("LDGWARP U8 warps/SM=%d thr=%d : %.0f GB/s\n", wps, thr, g * (double)per * 16 * nw / bytes);
    double g2 = timeit([&] { ldg_warp_kernel<4><<<blocks, thr>>>((const uint4*)d, per, o); });
    printf("LDGWARP U4 warps/SM=%d thr=%d : %.0f GB/s\n", wps, thr, g2 * (double)per * 16 * nw / bytes);
  }
  cudaFuncSetAttribute(bulk_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int P : {1, 2, 4, 8}) for (int B : {2048, 4096}) {
    int S = 16; int grid = 148; size_t smem = (size_t)B * S;
    size_t per = bytes / grid / B * B;
    double g = timeit([&] { bulk_multi_kernel<<<grid, 5 * 32, smem>>>(d, per, B, S, P, o); });
    printf("BULKMULTI P=%d B=%d S=%d : %.0f GB/s\n", P, B, S, g * (double)per * grid / bytes);
  }
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int ctas_per_sm : {1, 2, 4}) for (int B : {2048, 4096, 8192, 16384, 32768}) for (int S : {2, 4, 8}) {
    size_t smem = (size_t)B * S;
    if (smem * ctas_per_sm > 220 * 1024) continue;
    int grid = 148 * ctas_per_sm;
    size_t per = bytes / grid / B * B;
    double g = timeit([&] { bulk_kernel<<<grid, 5 * 32, smem>>>(d, per, B, S, 4, o); });
    printf("BULK cps=%d B=%d S=%d inflight/SM=%zuKB : %.0f GB/s\n", ctas_per_sm, B, S, smem * ctas_per_sm / 1024, g * (double)per * grid / bytes);
  }
  cudaError_t e = cudaGetLastError(); printf("err %s\n", cudaGetErrorString(e));
}
