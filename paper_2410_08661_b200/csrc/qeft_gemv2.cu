// Decode GEMV, bulk-copy warp rings: planner entry, tracing. The kernels and their host
// launch plans are in qeft_gemv2.cuh, instantiated per (bits, dtype) in qeft_gemv2_*.cu.
#include "qeft_gemv2.cuh"

using namespace qeft::g2;

namespace qeft {

bool gemv2_supported(const qeft_linear_t* L, int n) {
  if (L->sz16 == nullptr || env_int("QEFT_GEMV_V1", 0)) return false;
  if (L->g % 64 != 0) return false;
  const int gt = L->g / 64;
  return (gt == 1 || gt == 2 || gt == 4 || gt == 8) && n >= 1 && n <= 16 && L->m > 0;
}

size_t gemv2_workspace_bytes(const qeft_linear_t*, int) { return 0; }

// profiling: per-CTA timestamps of the next launches (8 per CTA, 512 CTAs per launch slot)
static unsigned long long* g_trace = nullptr;
static int g_trace_slots = 0, g_trace_next = 0;
constexpr int kTraceCtas = 512;

unsigned long long* trace_next_slot() {
  if (g_trace && g_trace_next < g_trace_slots) return g_trace + (size_t)(g_trace_next++) * kTraceCtas * 8;
  return nullptr;
}

int gemv_trace(int slots, unsigned long long* host_out) {
  if (slots > 0) {  // arm: allocate and clear
    if (g_trace) cudaFree(g_trace);
    QEFT_CUDA(cudaMalloc(&g_trace, (size_t)slots * kTraceCtas * 8 * sizeof(unsigned long long)));
    QEFT_CUDA(cudaMemset(g_trace, 0, (size_t)slots * kTraceCtas * 8 * sizeof(unsigned long long)));
    g_trace_slots = slots;
    g_trace_next = 0;
    return 0;
  }
  if (host_out && g_trace) {
    QEFT_CUDA(cudaDeviceSynchronize());
    QEFT_CUDA(cudaMemcpy(host_out, g_trace, (size_t)g_trace_slots * kTraceCtas * 8 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost));
  }
  if (g_trace) cudaFree(g_trace);
  g_trace = nullptr;
  g_trace_slots = 0;
  return 0;
}

int gemv2_multi(const qeft_linear_t* const* Ls, int nl, const void* x, int64_t ldx, void* const* ys, int64_t ldy,
                int y_f32, int n, void*, size_t, cudaStream_t st, const float* ngain, const void* xu) {
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
  a.ic = L->ic;
  // stages per warp L2-prefetched before the grid dependency (A/B on two boxes: stack +2 % /
  // -0.3 %, decode step -1.6 % on both; 2 or 3 stages lose 4-7 %)
  static const int l2pf = env_int("QEFT_GEMV2_L2PF", 1);
  a.l2pf = l2pf;
  if (xu) {
    // fused SwiGLU: structured layers (x moved by bulk copies), 16-byte aligned rows
    if (!a.fast || (((uintptr_t)xu) & 15) != 0) return -1;
    a.xu = xu;
  }
  if (ngain) {
    // fused RMS-norm: 16-byte rows (the stand-alone kernel's layout), its block size kept
    if (L->ic % 8 != 0 || ldx % 8 != 0 || (((uintptr_t)x) & 15) != 0) return -1;
    a.ngain = ngain;
    a.nthr = std::min(1024, std::max(32, L->ic / 8 / 32 * 32));
  }
  a.m_pad = L->m_pad;
  a.k = L->k;
  a.k_pad = L->k_pad;
  a.g = L->g;
  a.n = n;
  a.n_rb = rb_total;
  a.nch = L->m_pad / 128;
  a.ng16 = (L->m_pad + L->g - 1) / L->g;
  a.rbb = rowblock_bytes(L->bits, L->m_pad);
  static const int contig = env_int("QEFT_GEMV2_CONTIG", 1);
  a.contig = contig;
  a.trace = nullptr;
  a.trace = trace_next_slot();
  const int gt = L->g / 64;
  const bool bf = L->act_dtype == QEFT_BF16;
  if (L->bits == 4) return bf ? dispatch_4b(a, gt, st) : dispatch_4h(a, gt, st);
  return bf ? dispatch_3b(a, gt, st) : dispatch_3h(a, gt, st);
}

}  // namespace qeft
