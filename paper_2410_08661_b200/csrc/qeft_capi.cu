// extern "C" boundary of libqeft_b200.so (declared in include/qeft_b200.h).
// Thin argument validation + error mapping over the kernels in this directory.
#include <stdarg.h>
#include <string.h>

#include "qeft_common.cuh"
#include "qeft_internal.h"

namespace qeft {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int check_layer(const qeft_linear_t* L) {
  QEFT_CHECK(L != nullptr, QEFT_ERR_SHAPE, "null layer");
  QEFT_CHECK(L->bits == 3 || L->bits == 4, QEFT_ERR_SHAPE, "bits must be 3 or 4, got %d", L->bits);
  QEFT_CHECK(L->k >= 0 && L->k < L->ic, QEFT_ERR_SHAPE, "k=%d must be < IC=%d", L->k, L->ic);
  QEFT_CHECK(L->m == L->ic - L->k, QEFT_ERR_SHAPE, "m=%d != ic-k", L->m);
  QEFT_CHECK(L->g >= 1 && L->ng == (L->m + L->g - 1) / L->g, QEFT_ERR_SHAPE, "bad g/ng");
  QEFT_CHECK(L->m_pad == pad_to(L->m, 128) && L->k_pad == pad_to(L->k, 64) &&
                 L->oc_pad == pad_to(L->oc, 16),
             QEFT_ERR_SHAPE, "bad padding fields");
  QEFT_CHECK(L->act_dtype == QEFT_F16 || L->act_dtype == QEFT_BF16, QEFT_ERR_SHAPE, "bad dtype");
  return 0;
}

}  // namespace qeft

using namespace qeft;

#define ST(s) ((cudaStream_t)(s))

extern "C" {

const char* qeft_last_error(void) { return qeft::g_err; }

const char* qeft_version(void) { return "qeft_b200 0.1 sm_100a"; }

size_t qeft_qweight_bytes(int oc, int m, int bits) {
  return (size_t)(pad_to(oc, 16) / 16) * (size_t)rowblock_bytes(bits, pad_to(m, 128));
}

int qeft_repack_to_tiles(const uint8_t* ref, int oc, int m, int bits, void* qw, void* s) {
  QEFT_CHECK(bits == 3 || bits == 4, QEFT_ERR_SHAPE, "unsupported bit width %d", bits);
  QEFT_CHECK(oc >= 0 && m >= 0, QEFT_ERR_SHAPE, "negative shape");
  return repack_ref_to_tiles(ref, oc, m, bits, qw, ST(s));
}

int qeft_repack_to_ref(const void* qw, int oc, int m, int bits, uint8_t* ref, void* s) {
  QEFT_CHECK(bits == 3 || bits == 4, QEFT_ERR_SHAPE, "unsupported bit width %d", bits);
  return repack_tiles_to_ref(qw, oc, m, bits, ref, ST(s));
}

size_t qeft_sz16_bytes(int oc, int m, int g) { return sz16_bytes(oc, m, g); }

int qeft_pack_sz16(const float* sc, const float* zr, int oc, int m, int g, void* out, void* s) {
  return pack_sz16(sc, zr, oc, m, g, out, ST(s));
}

int qeft_pack_sz(const float* sc, const float* zr, int oc, int ng, void* out, void* s) {
  return pack_sz(sc, zr, oc, ng, out, ST(s));
}

int qeft_pack_weak(const float* w, int oc, int k, int dt, void* out, void* s) {
  return pack_weak(w, oc, k, dt, out, ST(s));
}

int qeft_dequant_full(const qeft_linear_t* L, float* out, void* s) {
  if (int r = check_layer(L)) return r;
  return dequant_full(L, out, ST(s));
}

int qeft_gather_cols(const void* x, int64_t ldx, const int32_t* colmap, int kk, int rows, int dt,
                     void* xb, void* s) {
  return gather_cols(x, ldx, colmap, kk, rows, dt, xb, ST(s));
}

int qeft_grid_params(const float* w, int oc, int m, int g, int bits, int steps, double alpha_min, float* sc,
                     float* zr, void* s) {
  return grid_params(w, oc, m, g, bits, steps, alpha_min, sc, zr, ST(s));
}

int qeft_nearest_codes(const float* w, int oc, int m, int g, int bits, const float* sc, const float* zr,
                       uint8_t* codes, void* s) {
  return nearest_codes(w, oc, m, g, bits, sc, zr, codes, ST(s));
}

int qeft_optq_codes(double* w64, const double* u64, const float* sc, const float* zr, int oc, int m, int g,
                    int bits, double* err_ws, uint8_t* codes, void* s) {
  return optq_codes(w64, u64, sc, zr, oc, m, g, bits, err_ws, codes, ST(s));
}

int qeft_quantize_rtn(const float* w, int oc, int m, int g, int bits, float* sc, float* zr,
                      uint8_t* codes, void* s) {
  return quantize_rtn(w, oc, m, g, bits, sc, zr, codes, ST(s));
}

int qeft_gemv_trace(int slots, unsigned long long* host_out) { return gemv_trace(slots, host_out); }

size_t qeft_gemv_workspace_bytes(const qeft_linear_t* L, int n) { return gemv_workspace_bytes(L, n); }

int qeft_gemv(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int y_f32,
              int n, void* ws, size_t wsb, void* s) {
  if (int r = check_layer(L)) return r;
  return gemv(L, x, ldx, y, ldy, y_f32, n, ws, wsb, ST(s));
}

int qeft_gemv_swiglu(const qeft_linear_t* L, const void* g, const void* u, int64_t ldx, void* y, int64_t ldy,
                     int y_flags, int n, void* ws, size_t wsb, void* s) {
  if (int r = check_layer(L)) return r;
  QEFT_CHECK(g != nullptr && u != nullptr, QEFT_ERR_SHAPE, "gemv_swiglu: null input");
  return gemv_multi(&L, 1, g, ldx, &y, ldy, y_flags, n, ws, wsb, ST(s), nullptr, u);
}

int qeft_gemv_multi_rmsnorm(const qeft_linear_t* const* Ls, int nl, const void* x, int64_t ldx, const float* gain,
                            void* const* ys, int64_t ldy, int y_f32, int n, void* ws, size_t wsb, void* s) {
  QEFT_CHECK(Ls != nullptr && ys != nullptr && nl >= 1 && gain != nullptr, QEFT_ERR_SHAPE, "gemv_multi_rmsnorm: args");
  for (int l = 0; l < nl; ++l)
    if (int r = check_layer(Ls[l])) return r;
  return gemv_multi(Ls, nl, x, ldx, ys, ldy, y_f32, n, ws, wsb, ST(s), gain);
}

int qeft_gemv_multi(const qeft_linear_t* const* Ls, int nl, const void* x, int64_t ldx, void* const* ys,
                    int64_t ldy, int y_f32, int n, void* ws, size_t wsb, void* s) {
  QEFT_CHECK(Ls != nullptr && ys != nullptr && nl >= 1, QEFT_ERR_SHAPE, "gemv_multi: no layers");
  for (int l = 0; l < nl; ++l)
    if (int r = check_layer(Ls[l])) return r;
  return gemv_multi(Ls, nl, x, ldx, ys, ldy, y_f32, n, ws, wsb, ST(s));
}

size_t qeft_gemm_workspace_bytes(const qeft_linear_t* L, int T) { return gemm_workspace_bytes(L, T); }

int qeft_gemm_set_schedule(int what, int value) { return gemm_set_schedule(what, value); }

int qeft_gemm_wgrad_weak_multi(const qeft_linear_t* const* Ls, int nl, const void* const* dys, const int64_t* lddys,
                               const void* x_weak, int64_t ldxw, float* const* dws, int T, int accumulate, void* s) {
  QEFT_CHECK(Ls != nullptr && dys != nullptr && dws != nullptr && lddys != nullptr, QEFT_ERR_SHAPE,
             "wgrad_multi: null argument");
  for (int l = 0; l < nl; ++l)
    if (int r = check_layer(Ls[l])) return r;
  return gemm_wgrad_weak_multi(Ls, nl, dys, lddys, x_weak, ldxw, dws, T, accumulate, ST(s));
}

int qeft_gemm_fwd(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int T,
                  void* ws, size_t wsb, void* s) {
  if (int r = check_layer(L)) return r;
  return gemm_fwd(L, x, ldx, y, ldy, T, ws, wsb, ST(s));
}

int qeft_gemm_dgrad(const qeft_linear_t* L, const void* dy, int64_t lddy, void* dx, int64_t lddx,
                    int T, int acc, void* ws, size_t wsb, void* s) {
  if (int r = check_layer(L)) return r;
  return gemm_dgrad(L, dy, lddy, dx, lddx, T, acc, ws, wsb, ST(s));
}

int qeft_gemm_wgrad(const qeft_linear_t* L, const void* dy, int64_t lddy, const void* x, int64_t ldx,
                    float* dw, int T, int acc, void* ws, size_t wsb, void* s) {
  if (int r = check_layer(L)) return r;
  return gemm_wgrad(L, dy, lddy, x, ldx, dw, T, acc, ws, wsb, ST(s));
}

int qeft_gemm_wgrad_weak(const qeft_linear_t* L, const void* dy, int64_t lddy, const void* xw,
                         int64_t ldxw, float* dw, int T, int acc, void* ws, size_t wsb, void* s) {
  if (int r = check_layer(L)) return r;
  return gemm_wgrad(L, dy, lddy, xw, ldxw, dw, T, acc, ws, wsb, ST(s), true);
}

int qeft_grad_sqnorm(const float* g, int64_t n, double* scratch, double* out, void* s) {
  return grad_sqnorm(g, n, scratch, out, ST(s));
}

int qeft_div_scalar(float* g, int64_t n, float d, void* s) { return div_scalar(g, n, d, ST(s)); }

int qeft_adam_clip(float* w, float* m, float* v, const float* g, int64_t n, const double* sq,
                   double max_norm, float lr, float c_b1, float c_1mb1, float c_b2, float c_1mb2,
                   float bc1, float bc2, float eps, int* flag, void* s) {
  return adam_clip(w, m, v, g, n, sq, max_norm, lr, c_b1, c_1mb1, c_b2, c_1mb2, bc1, bc2, eps, flag,
                   ST(s));
}

int qeft_grad_sqnorm_div(const float* g, int64_t n, float divisor, double* scratch, double* out, void* s) {
  QEFT_CHECK(divisor != 0.f, QEFT_ERR_SHAPE, "grad_sqnorm_div: zero divisor");
  return grad_sqnorm(g, n, scratch, out, ST(s), divisor);
}

int qeft_adam_step_flat(float* w32, float* m, float* v, const float* g, const qeft_shadow_desc_t* descs,
                        int n_layers, int max_rows, float divisor, const double* sq, double max_norm, float lr,
                        float c_b1, float c_1mb1, float c_b2, float c_1mb2, float bc1, float bc2, float eps,
                        int* flag, void* s) {
  return adam_step_flat(w32, m, v, g, descs, n_layers, max_rows, divisor, sq, max_norm, lr, c_b1, c_1mb1, c_b2,
                        c_1mb2, bc1, bc2, eps, flag, ST(s));
}

int qeft_weak_shadow(const float* w32, const qeft_shadow_desc_t* d, int n, int max_elems, void* s) {
  return weak_shadow(w32, d, n, max_elems, ST(s));
}

int qeft_rmsnorm_fwd(const void* x, const float* gain, void* y, float* rstd, int rows, int C, int dt, void* s) {
  return rmsnorm_fwd(x, gain, y, rstd, rows, C, dt, ST(s));
}

int qeft_rmsnorm_bwd(const void* dy, const void* x, const float* gain, const float* rstd, const void* dres,
                     void* dx, int rows, int C, int dt, void* s) {
  return rmsnorm_bwd(dy, x, gain, rstd, dres, dx, rows, C, dt, ST(s));
}

int qeft_rope_kv(const void* q, const void* k, const void* v, void* q_out, void* k_cache, void* v_cache,
                 const float* cos_t, const float* sin_t, const int64_t* pos, int B, int H, int hd, int T_cache, int dt,
                 void* s) {
  return rope_kv(q, k, v, q_out, k_cache, v_cache, cos_t, sin_t, pos, B, H, hd, T_cache, dt, ST(s));
}

int qeft_rope(const void* in, void* out, const float* cosv, const float* sinv, int64_t rows, int T, int H, int hd,
              int inverse, int dt, void* s) {
  return rope(in, out, cosv, sinv, rows, T, H, hd, inverse, dt, ST(s));
}

size_t qeft_decode_attention_workspace_bytes(int B, int H, int hd) { return decode_attention_workspace_bytes(B, H, hd); }

int qeft_decode_attention(const void* q, const void* k, const void* v, void* kc, void* vc, const float* cos_t,
                          const float* sin_t, const int64_t* pos, void* o, int B, int H, int hd, int T_cache, int dt,
                          void* ws, size_t ws_bytes, void* s) {
  return decode_attention(q, k, v, kc, vc, cos_t, sin_t, pos, o, B, H, hd, T_cache, dt, ws, ws_bytes, ST(s));
}

int qeft_cross_entropy_fwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, float* loss,
                           float* lse, int dt, void* s) {
  return cross_entropy_fwd(z, ldz, rows, V, tgt, loss, lse, dt, ST(s));
}

int qeft_cross_entropy_bwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, const float* lse,
                           const float* gscale, void* dz, int64_t lddz, int dt, void* s) {
  return cross_entropy_bwd(z, ldz, rows, V, tgt, lse, gscale, dz, lddz, dt, ST(s));
}

int qeft_silu_mul_fwd(const void* g, const void* u, void* f, int64_t n, int dt, void* s) {
  return silu_mul_fwd(g, u, f, n, dt, ST(s));
}

int qeft_silu_mul_bwd(const void* df, const void* g, const void* u, void* dg, void* du, int64_t n, int dt, void* s) {
  return silu_mul_bwd(df, g, u, dg, du, n, dt, ST(s));
}

}  // extern "C"
