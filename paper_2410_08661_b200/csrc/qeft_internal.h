// Internal host-side helpers shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/qeft_b200.h"

namespace qeft {

void set_error(const char* fmt, ...);

inline int pad_to(int x, int a) { return (x + a - 1) / a * a; }

#define QEFT_CUDA(expr)                                                              \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::qeft::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return QEFT_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define QEFT_CHECK(cond, code, ...)      \
  do {                                   \
    if (!(cond)) {                       \
      ::qeft::set_error(__VA_ARGS__);    \
      return code;                       \
    }                                    \
  } while (0)

int repack_ref_to_tiles(const uint8_t* ref, int oc, int m, int bits, void* qw, cudaStream_t st);
int repack_tiles_to_ref(const void* qw, int oc, int m, int bits, uint8_t* ref, cudaStream_t st);
int pack_sz(const float* s, const float* z, int oc, int ng, void* out, cudaStream_t st);
size_t sz16_bytes(int oc, int m, int g);
int pack_sz16(const float* s, const float* z, int oc, int m, int g, void* out, cudaStream_t st);
int pack_weak(const float* w, int oc, int k, int dtype, void* out, cudaStream_t st);
int dequant_full(const qeft_linear_t* L, float* out, cudaStream_t st);
int gather_rows(const void* x, int64_t ldx, int src_cols, const int* colmap, int kk, int rows, int dtype,
                void* xb, cudaStream_t st);
int scatter_rows(const void* xb, int kk, const int* colmap, int ic, int rows, int dtype, void* out, int64_t ldo,
                 int accumulate, cudaStream_t st);
int gather_cols(const void* x, int64_t ldx, const int* colmap, int kk, int rows, int dtype, void* xb,
                cudaStream_t st);
int grid_params(const float* w, int oc, int m, int g, int bits, int steps, double amin, float* s, float* z,
                cudaStream_t st);
int nearest_codes(const float* w, int oc, int m, int g, int bits, const float* s, const float* z, uint8_t* codes,
                  cudaStream_t st);
int optq_codes(double* w, const double* u, const float* s, const float* z, int oc, int m, int g, int bits,
               double* err, uint8_t* codes, cudaStream_t st);
int quantize_rtn(const float* w, int oc, int m, int g, int bits, float* s, float* z, uint8_t* codes,
                 cudaStream_t st);

size_t gemv_workspace_bytes(const qeft_linear_t* L, int n);
int gemv(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int y_f32, int n,
         void* ws, size_t ws_bytes, cudaStream_t st);
int gemv_multi(const qeft_linear_t* const* Ls, int nl, const void* x, int64_t ldx, void* const* ys, int64_t ldy,
               int y_f32, int n, void* ws, size_t ws_bytes, cudaStream_t st, const float* ngain = nullptr,
               const void* xu = nullptr);
// bulk-copy warp-ring GEMV (qeft_gemv2.cu); gemv2_multi returns -1 when the launch needs the
// generic path (its partials would not fit shared memory)
int gemv_trace(int slots, unsigned long long* host_out);
// next armed trace slot (512 CTAs x 8 u64) of qeft_gemv_trace, or null: GEMV and GEMM launches
unsigned long long* trace_next_slot();
bool gemv2_supported(const qeft_linear_t* L, int n);
size_t gemv2_workspace_bytes(const qeft_linear_t* L, int n);
int gemv2_multi(const qeft_linear_t* const* Ls, int nl, const void* x, int64_t ldx, void* const* ys,
                int64_t ldy, int y_f32, int n, void* ws, size_t ws_bytes, cudaStream_t st,
                const float* ngain = nullptr, const void* xu = nullptr);
int silu_mul_fwd(const void* g, const void* u, void* f, int64_t n, int dt, cudaStream_t st);
int rmsnorm_fwd(const void* x, const float* gain, void* y, float* rstd, int rows, int C, int dt, cudaStream_t st);

size_t gemm_workspace_bytes(const qeft_linear_t* L, int T);
int gemm_set_schedule(int what, int value);
size_t decode_attention_workspace_bytes(int B, int H, int hd);
int decode_attention(const void* q, const void* k, const void* v, void* kc, void* vc, const float* cosv,
                     const float* sinv, const int64_t* pos_dev, void* o, int B, int H, int hd, int T_cache, int dt,
                     void* ws, size_t ws_bytes, cudaStream_t st);
int gemm_wgrad_weak_multi(const qeft_linear_t* const* Ls, int nl, const void* const* dys, const int64_t* lddys,
                          const void* x_weak, int64_t ldxw, float* const* dws, int T, int accumulate,
                          cudaStream_t st);
int cross_entropy_fwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, float* loss, float* lse,
                      int dt, cudaStream_t st);
int cross_entropy_bwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, const float* lse,
                      const float* gscale, void* dz, int64_t lddz, int dt, cudaStream_t st);
int gemm_fwd(const qeft_linear_t* L, const void* x, int64_t ldx, void* y, int64_t ldy, int T,
             void* ws, size_t ws_bytes, cudaStream_t st);
int gemm_dgrad(const qeft_linear_t* L, const void* dy, int64_t lddy, void* dx, int64_t lddx, int T,
               int accumulate, void* ws, size_t ws_bytes, cudaStream_t st);
int gemm_wgrad(const qeft_linear_t* L, const void* dy, int64_t lddy, const void* x, int64_t ldx,
               float* dw, int T, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st,
               bool x_is_weak = false);

int grad_sqnorm(const float* g, int64_t n, double* scratch, double* out, cudaStream_t st, float div = 1.f);
int div_scalar(float* g, int64_t n, float d, cudaStream_t st);
int adam_step_flat(float* w, float* m, float* v, const float* g, const qeft_shadow_desc_t* descs, int n_layers,
                   int max_rows, float div, const double* sqnorm, double max_norm, float lr, float c_b1,
                   float c_1mb1, float c_b2, float c_1mb2, float bc1, float bc2, float eps, int* flag,
                   cudaStream_t st);
int adam_clip(float* w, float* m, float* v, const float* g, int64_t n, const double* sqnorm,
              double max_norm, float lr, float c_b1, float c_1mb1, float c_b2, float c_1mb2, float bc1,
              float bc2, float eps, int* flag, cudaStream_t st);
int weak_shadow(const float* w32, const qeft_shadow_desc_t* d, int n_layers, int max_elems,
                cudaStream_t st);

int rmsnorm_fwd(const void* x, const float* gain, void* y, float* rstd, int rows, int C, int dt, cudaStream_t st);
int rmsnorm_bwd(const void* dy, const void* x, const float* gain, const float* rstd, const void* dres, void* dx,
                int rows, int C, int dt, cudaStream_t st);
int rope_kv(const void* q, const void* k, const void* v, void* q_out, void* kc, void* vc, const float* cosv,
            const float* sinv, const int64_t* pos_dev, int B, int H, int hd, int T_cache, int dt, cudaStream_t st);
int rope(const void* in, void* out, const float* cosv, const float* sinv, int64_t rows, int T, int H, int hd,
         int inverse, int dt, cudaStream_t st);
int silu_mul_fwd(const void* g, const void* u, void* f, int64_t n, int dt, cudaStream_t st);
int silu_mul_bwd(const void* df, const void* g, const void* u, void* dg, void* du, int64_t n, int dt,
                 cudaStream_t st);

}  // namespace qeft
