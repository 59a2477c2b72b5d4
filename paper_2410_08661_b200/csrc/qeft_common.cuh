// Shared device helpers for the QEFT B200 library (sm_100a only).
//
// B200 packed layout ("tile layout"), shared by every kernel:
//   * the quantized part of a layer is cut into row-blocks of 16 output rows;
//     each row-block is a run of K-tiles (4-bit: 64 codes wide, 512 B;
//     3-bit: 128 codes wide, 768 B). Lane l = 4*g + t of a warp owns rows
//     g and g+8 of the row-block and the 16 consecutive columns [16t, 16t+16)
//     of every 64-wide K half, so one warp moves one tile with fully
//     coalesced 128-bit loads and each lane's codes are exactly the operands
//     it needs (mma m16n8k16 A fragments, with K permuted inside each k16
//     subtile identically for both operands, or 2 x 16 B swizzled smem rows
//     for the tcgen05 producer).
//   * 4-bit: u32 j of a lane's 16 B is k16-subtile j (columns 16t+4j..+3):
//       nibble 0:(g,c) 1:(g+8,c) 2:(g,c+2) 3:(g+8,c+2)
//              4:(g,c+1) 5:(g+8,c+1) 6:(g,c+3) 7:(g+8,c+3)      c = 16t+4j
//     so (q & 0x000F000F) | magic yields the half2 fragment (g, c..c+1).
//   * 3-bit: 2-bit plane (lane 16 B at l*16) + 1-bit plane (lane 8 B at
//     512 + l*8). Half h (K cols 64h..64h+63) uses 2-bit words 2h, 2h+1 and
//     hi-bit word h. Word ww of a half holds subtiles 2ww, 2ww+1; pair p (0..7)
//     = subtile 2ww + p/4, fragment p%4 (same element pairs as 4-bit); the
//     pair's two low fields sit at bits 2p and 16+2p, its high bits at
//     (2+p+8ww) mod 32 and (18+p+8ww) mod 32 of the hi word, so
//     rotr(hi, p+8ww) & 0x00040004 drops them into place.
//   * sz: (scale, zero) pairs in the activation dtype, [oc_pad/16][ng][16].
//   * weak16: weak columns in the activation dtype, row-major [oc_pad][k_pad].
//   * colmap: int32 [m_pad + k_pad]; B200 K position -> original input column
//     (quant positions, then weak indices; -1 for padding).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <type_traits>

#define QEFT_DEV __device__ __forceinline__

namespace qeft {

constexpr int kRowBlock = 16;

QEFT_DEV uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  // (a & b) | c
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

QEFT_DEV uint32_t rotr32(uint32_t x, uint32_t s) {
  uint32_t d;
  asm("shf.r.wrap.b32 %0, %1, %1, %2;\n" : "=r"(d) : "r"(x), "r"(s));
  return d;
}

template <typename T> struct DTraits;
template <> struct DTraits<__half> {
  using T2 = __half2;
  static constexpr uint32_t kMagic = 0x64006400u;   // fp16 1024.0 in both halves
  static constexpr float kMagicF = 1024.f;
  static constexpr bool kHiTrick = true;            // 1024 + 16c is exact in fp16
  static constexpr uint32_t kOne2 = 0x3C003C00u;
};
template <> struct DTraits<__nv_bfloat16> {
  using T2 = __nv_bfloat162;
  static constexpr uint32_t kMagic = 0x43004300u;   // bf16 128.0
  static constexpr float kMagicF = 128.f;
  static constexpr bool kHiTrick = false;
  static constexpr uint32_t kOne2 = 0x3F803F80u;
};

// 4-bit u32 -> four (magic + code) fragments (a0a1, a2a3, a4a5, a6a7).
// fp16: rows g+8 (frags 1 and 3) come out as 1024 + 16*c (callers scale by 1/16).
template <typename T>
QEFT_DEV void decode4(uint32_t q, uint32_t f[4]) {
  constexpr uint32_t M = DTraits<T>::kMagic;
  if constexpr (DTraits<T>::kHiTrick) {
    f[0] = lop3_and_or(q, 0x000F000Fu, M);
    f[1] = lop3_and_or(q, 0x00F000F0u, M);
    q >>= 8;
    f[2] = lop3_and_or(q, 0x000F000Fu, M);
    f[3] = lop3_and_or(q, 0x00F000F0u, M);
  } else {
    f[0] = lop3_and_or(q, 0x000F000Fu, M);
    f[1] = lop3_and_or(q >> 4, 0x000F000Fu, M);
    f[2] = lop3_and_or(q >> 8, 0x000F000Fu, M);
    f[3] = lop3_and_or(q >> 12, 0x000F000Fu, M);
  }
}

// 3-bit: fragment p (0..7) of 2-bit word w (word index ww within its half),
// hi-bit word hb.  Result is magic + code in both halves.
template <typename T>
QEFT_DEV uint32_t decode3_pair(uint32_t w, uint32_t hb, int p, int ww) {
  constexpr uint32_t M = DTraits<T>::kMagic;
  uint32_t lo = lop3_and_or(w >> (2 * p), 0x00030003u, M);
  return lop3_and_or(rotr32(hb, (uint32_t)(p + 8 * ww)), 0x00040004u, lo);
}

// magic+code (or magic + 16*code for the fp16 hi trick) -> exact code as T2
template <typename T>
QEFT_DEV typename DTraits<T>::T2 magic_to_code(uint32_t v, bool hi16) {
  using T2 = typename DTraits<T>::T2;
  T2 h = *reinterpret_cast<T2*>(&v);
  if constexpr (DTraits<T>::kHiTrick) {
    if (hi16) {
      const T2 k = __floats2half2_rn(1.f / 16.f, 1.f / 16.f);
      const T2 b = __floats2half2_rn(-64.f, -64.f);
      return __hfma2(h, k, b);
    }
    const T2 b = __floats2half2_rn(-1024.f, -1024.f);
    return __hadd2(h, b);
  } else {
    const T2 b = __floats2bfloat162_rn(-128.f, -128.f);
    return __hadd2(h, b);
  }
}

template <typename T> QEFT_DEV float to_f32(T v);
template <> QEFT_DEV float to_f32<__half>(__half v) { return __half2float(v); }
template <> QEFT_DEV float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> QEFT_DEV T from_f32(float v);
template <> QEFT_DEV __half from_f32<__half>(float v) { return __float2half_rn(v); }
template <> QEFT_DEV __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> QEFT_DEV float from_f32<float>(float v) { return v; }

template <typename T2> QEFT_DEV float2 t2_to_f2(T2 v);
template <> QEFT_DEV float2 t2_to_f2<__half2>(__half2 v) { return __half22float2(v); }
template <> QEFT_DEV float2 t2_to_f2<__nv_bfloat162>(__nv_bfloat162 v) { return __bfloat1622float2(v); }

// mma.sync m16n8k16, fp32 accumulate (register-fed A fragments for the GEMV).
template <typename T>
QEFT_DEV void mma16816(float d[4], const uint32_t a[4], uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<T, __half>::value) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
}

QEFT_DEV uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
QEFT_DEV uint2 ldg_stream64(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];\n"
               : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// ---- programmatic dependent launch (griddepcontrol) ----
QEFT_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
QEFT_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Launch with cudaLaunchAttributeProgrammaticStreamSerialization so the kernel
// may begin while its stream predecessor drains (it calls pdl_wait() before
// touching the predecessor's outputs). Captured into CUDA graphs as
// programmatic edges.
template <typename Kern, typename... Args>
inline cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool no_pdl = getenv("QEFT_NO_PDL") != nullptr;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Kern, typename... Args>
inline cudaError_t launch_pdl_cluster(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  static const bool no_pdl = getenv("QEFT_NO_PDL") != nullptr;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 1 : 2;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---- mbarrier / bulk async copy (TMA 1-D) ----
QEFT_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

QEFT_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
QEFT_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
QEFT_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

QEFT_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
QEFT_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
QEFT_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n.reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0)
QEFT_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// named barrier over a subset of the CTA's warps (id 1..15; id 0 is __syncthreads)
QEFT_DEV void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- cp.async (LDGSTS): per-thread async global -> shared copies ----
QEFT_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
QEFT_DEV void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
QEFT_DEV void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
QEFT_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
QEFT_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---- clusters / distributed shared memory ----
QEFT_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
QEFT_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
// read a float from CTA `rank`'s shared memory at the same offset as local_addr
QEFT_DEV float ld_dsmem_f32(uint32_t local_addr, uint32_t rank) {
  uint32_t remote;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local_addr), "r"(rank));
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// weak16 element (r, j): row-block tiles of 16 rows x 64 columns (2 KB, contiguous),
// tile (r/16, j/64) at ((r/16) * (k_pad/64) + j/64) * 1024 elements, row-major inside.
__host__ __device__ inline int64_t weak_off(int r, int j, int k_pad) {
  return (((int64_t)(r >> 4) * (k_pad >> 6) + (j >> 6)) << 10) + ((r & 15) << 6) + (j & 63);
}

// ---- code addressing in the tile layout (used by repack/debug kernels) ----

// byte offset of the 16-row block rb inside qweight
__host__ __device__ inline int64_t rowblock_bytes(int bits, int m_pad) {
  return bits == 4 ? (int64_t)m_pad * 8 : (int64_t)m_pad * 6;
}

// Locate code (r, j) of the tile layout.  For 4-bit returns byte offset and
// nibble shift; for 3-bit the 2-bit field position and the hi-bit position.
struct CodeLoc {
  int64_t lo_word;   // u32 index of the 4-bit word / 2-bit word
  int lo_shift;      // bit shift inside that word
  int64_t hi_word;   // u32 index of the 3-bit hi word
  int hi_shift;
};

__host__ __device__ inline CodeLoc locate_code(int bits, int m_pad, int r, int j) {
  CodeLoc L{};
  const int rb = r >> 4, rr = r & 15;
  const int g = rr & 7, upper = rr >> 3;   // upper: row g+8
  if (bits == 4) {
    const int kt = j >> 6, jc = j & 63;
    const int t = jc >> 4, sub = (jc >> 2) & 3, e = jc & 3;  // column c + e
    const int lane = 4 * g + t;
    // element e in {0,1,2,3} -> nibble: e=0:0/1, e=1:4/5, e=2:2/3, e=3:6/7
    const int nib = ((e & 1) ? 4 : 0) + ((e & 2) ? 2 : 0) + upper;
    const int64_t tile_u32 = ((int64_t)rb * (m_pad >> 6) + kt) * 128;  // 512 B = 128 u32
    L.lo_word = tile_u32 + lane * 4 + sub;
    L.lo_shift = 4 * nib;
  } else {
    const int kt = j >> 7, jc = j & 127;
    const int h = jc >> 6, jh = jc & 63;
    const int t = jh >> 4, sub = (jh >> 2) & 3, e = jh & 3;
    const int lane = 4 * g + t;
    const int ww = sub >> 1;
    const int pp = (e >> 1) * 2 + upper;        // fragment index 0..3
    const int p = 4 * (sub & 1) + pp;           // pair index 0..7
    const int hiside = e & 1;                   // low or high element of the pair
    const int64_t tile_u32 = ((int64_t)rb * (m_pad >> 7) + kt) * 192;  // 768 B
    L.lo_word = tile_u32 + lane * 4 + 2 * h + ww;
    L.lo_shift = 2 * p + 16 * hiside;
    L.hi_word = tile_u32 + 128 + lane * 2 + h;
    L.hi_shift = ((hiside ? 18 : 2) + p + 8 * ww) & 31;
  }
  return L;
}

}  // namespace qeft
