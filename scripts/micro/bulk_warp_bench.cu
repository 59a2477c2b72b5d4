// Streaming microbenchmark for the GEMV v2 design: every warp owns a private ring of R
// stages of B bytes fed by its own lane 0 with cp.async.bulk (1-D TMA) on an mbarrier;
// all 32 lanes read the whole stage back with LDS.128 (what the decode+MMA consumer
// does), then lane 0 refills the slot. Prints GB/s per (warps/CTA, CTAs/SM, B, R).
// Also: one producer warp feeding a CTA-wide ring (the classic TMA pipeline) for contrast.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 bulk_warp_bench.cu -o bulk_warp_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_08661_b200/csrc/qeft_common.cuh"
using namespace qeft;

// each warp streams `per_warp` contiguous bytes (a multiple of B)
__global__ void warp_ring_kernel(const uint8_t* p, size_t per_warp, int B, int R, unsigned* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint8_t* ring = smem + (size_t)warp * R * B;
  const size_t w = (size_t)blockIdx.x * nw + warp;
  const uint8_t* base = p + w * per_warp;
  const int nst = (int)(per_warp / B);
  if (lane == 0) {
    for (int i = 0; i < R; ++i) mbar_init(&full[warp][i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0)
    for (int s = 0; s < R && s < nst; ++s) {
      mbar_expect_tx(&full[warp][s], B);
      bulk_g2s(ring + (size_t)s * B, base + (size_t)s * B, B, &full[warp][s]);
    }
  unsigned acc = 0;
  for (int s = 0; s < nst; ++s) {
    const int slot = s % R;
    mbar_wait(&full[warp][slot], (s / R) & 1);
    const uint4* q = reinterpret_cast<const uint4*>(ring + (size_t)slot * B);
#pragma unroll 4
    for (int i = lane; i < B / 16; i += 32) { uint4 v = q[i]; acc ^= v.x ^ v.w; }
    __syncwarp();
    if (lane == 0 && s + R < nst) {
      mbar_expect_tx(&full[warp][slot], B);
      bulk_g2s(ring + (size_t)slot * B, base + (size_t)(s + R) * B, B, &full[warp][slot]);
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  size_t bytes = 1ull << 30;  // 1 GiB >> L2
  uint8_t* d; unsigned* o;
  cudaMalloc(&d, bytes); cudaMalloc(&o, 4);
  cudaMemset(d, 1, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto fn) {
    fn(); cudaDeviceSynchronize(); cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5;
  };
  cudaFuncSetAttribute(warp_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int nw : {4, 8, 12, 16}) for (int cps : {1, 2}) for (int B : {2048, 4096, 8192, 16384}) for (int R : {2, 3, 4, 6, 8}) {
    size_t smem = (size_t)nw * R * B;
    if (smem * cps > 220 * 1024) continue;
    int grid = 148 * cps;
    size_t nwt = (size_t)grid * nw;
    size_t per = bytes / nwt / B * B;
    float ms = timeit([&] { warp_ring_kernel<<<grid, nw * 32, smem>>>(d, per, B, R, o); });
    double gbs = (double)per * nwt / (ms * 1e-3) / 1e9;
    printf("WARPRING warps=%d cps=%d B=%d R=%d inflight/SM=%zuKB : %.0f GB/s\n", nw, cps, B, R,
           smem * cps / 1024, gbs);
  }
  cudaError_t e = cudaGetLastError(); printf("err %s\n", cudaGetErrorString(e));
}
