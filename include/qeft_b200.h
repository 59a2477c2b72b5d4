/*
 * qeft_b200.h — C ABI of the B200-native QEFT structured mixed-precision
 * linear layer (arXiv 2410.08661). Built as libqeft_b200.so for sm_100a.
 *
 * This is the drop-in boundary for the reference package's hot path
 * (/root/reference/pkg/src/qeft). Each entry point names the reference
 * function it replaces. Conventions:
 *   - all pointers are DEVICE pointers unless stated; the caller owns all
 *     memory and the library never allocates (workspace is passed in);
 *   - calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy);
 *   - return 0 on success, QEFT_ERR_SHAPE (1) for shape/argument errors
 *     (the reference raises qeft.errors.ShapeError, errors.py:16-17),
 *     QEFT_ERR_LAYOUT (2) for unsupported layouts, QEFT_ERR_CUDA (3) for
 *     CUDA failures; qeft_last_error() returns a thread-local message.
 *   - activations are row-major [rows][ld] in fp16 or bf16 (act_dtype):
 *     the torch orientation. The reference's (channels, tokens) arrays are the
 *     transpose; the host adapter converts.
 */
#ifndef QEFT_B200_H
#define QEFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QEFT_OK 0
#define QEFT_ERR_SHAPE 1
#define QEFT_ERR_LAYOUT 2
#define QEFT_ERR_CUDA 3

#define QEFT_F16 0
#define QEFT_BF16 1

/* flags */
#define QEFT_FLAG_STRUCTURED_FAST 1 /* colmap == identity-with-gap, m%8==0, ic%8==0 */

/*
 * One quantized linear layer in the B200 tile layout (see csrc/qeft_common.cuh).
 * Field meaning follows QuantizedLinear (pkg/src/qeft/quantizer.py:42-65):
 * m = ic - k quantized columns in groups of g (last group ragged), ng groups.
 */
typedef struct qeft_linear {
  int32_t oc, ic, k, bits, g;
  int32_t m, ng;
  int32_t m_pad;   /* roundup(m, 128) */
  int32_t k_pad;   /* roundup(k, 64), 0 when k == 0 */
  int32_t oc_pad;  /* roundup(oc, 16) */
  int32_t act_dtype; /* QEFT_F16 / QEFT_BF16: dtype of weak16 and activations */
  int32_t flags;
  const void* qweight;   /* tile-layout codes, (oc_pad/16) * rowblock bytes */
  const void* sz;        /* fp32 (scale, zero) pairs [oc_pad/16][ng][16][2] */
  const void* weak16;    /* [oc_pad][k_pad] */
  const int32_t* colmap; /* [m_pad + k_pad]: B200 K position -> input column, -1 pad */
  const void* sz16;      /* decode-GEMV copy of (scale, zero): fp16 pairs [oc_pad/16][ng16][8][2],
                            ng16 = ceil(m_pad / g); see qeft_pack_sz16. NULL: generic GEMV path */
} qeft_linear_t;

/* ---- format conversion (packing.py:24-72, quantizer.py:42-100) ---- */

/* Bytes of the tile-layout qweight for (oc, m, bits). */
size_t qeft_qweight_bytes(int oc, int m, int bits);

/* Reference packed bytes (pack_codes output, packing.py:24-52) -> tiles. */
int qeft_repack_to_tiles(const uint8_t* ref_packed, int oc, int m, int bits, void* qweight,
                         void* stream);
/* Tiles -> reference packed bytes, bit-exact inverse (unpack/pack round trip). */
int qeft_repack_to_ref(const void* qweight, int oc, int m, int bits, uint8_t* ref_packed,
                       void* stream);
/* fp32 scales/zeros [oc][ng] (quantizer.py:50-51) -> fp32 (scale, zero) pairs in the
 * row-block-major sz layout (the reference's storage precision, 8 B per group). */
int qeft_pack_sz(const float* scales, const float* zeros, int oc, int ng, void* sz, void* stream);
/* fp32 scales/zeros [oc][ng] -> the decode GEMV's fp16 (scale, zero) copy: half2 pairs
 * [oc_pad/16][ng16][8][2] (rows r and r+8 adjacent, 64 B per row-block and group, zero
 * padded to ng16 = ceil(roundup(m,128)/g) groups). qeft_sz16_bytes() gives its size. */
size_t qeft_sz16_bytes(int oc, int m, int g);
int qeft_pack_sz16(const float* scales, const float* zeros, int oc, int m, int g, void* sz16, void* stream);
/* fp32 weak block [oc][k] (quantizer.py:52) -> weak16 [oc_pad][k_pad]. */
int qeft_pack_weak(const float* weak, int oc, int k, int act_dtype, void* weak16, void* stream);
/* QuantizedLinear.dequant_full (quantizer.py:95-100) of the device layer, fp32 [oc][ic]. */
int qeft_dequant_full(const qeft_linear_t* layer, float* out, void* stream);
/* xb[r][j] = x[r][colmap[j]] (0 for padding): input gather for irregular /
 * online-reorder layers (kernels.py:110, kernels.py:123-124). */
int qeft_gather_cols(const void* x, int64_t ldx, const int32_t* colmap, int kk, int rows,
                     int act_dtype, void* xb, void* stream);

/* ---- offline quantization (quantizer.py:115-218): RTN min-max params + nearest codes ---- */
/* w_dense [oc][m] fp32 (already split to quantized columns). Outputs fp32 scales/zeros
 * [oc][ng] and uint8 codes [oc][m]; bit-exact with _minmax_params/_nearest_codes. */
int qeft_quantize_rtn(const float* w_dense, int oc, int m, int g, int bits, float* scales,
                      float* zeros, uint8_t* codes, void* stream);

/* alpha-grid search (quantizer.py:144-179, grid_search_group_params): per (row, group) the
 * range shrink alpha in {alpha_min + i (1 - alpha_min)/(steps - 1)} with least fp64 squared
 * error (larger alpha on ties), params stored fp32. Bit-exact with the reference (same fp64
 * op order, numpy pairwise summation of the errors). */
int qeft_grid_params(const float* w_dense, int oc, int m, int g, int bits, int steps, double alpha_min,
                     float* scales, float* zeros, void* stream);
/* nearest codes on fixed fp32 params (quantizer.py:211-218 _nearest_codes), uint8 [oc][m]. */
int qeft_nearest_codes(const float* w_dense, int oc, int m, int g, int bits, const float* scales,
                       const float* zeros, uint8_t* codes, void* stream);

/* OPTQ greedy rounding (quantizer.py:221-259 optq_quantize) given the reference's factor
 * u64 = chol(inv(H_damped)).T [m][m] (host numpy, as the reference computes it). w64 [oc][m]
 * is the fp64 working copy (overwritten); err_ws is oc*m fp64 scratch. Codes uint8 [oc][m],
 * bit-exact: each weight gets its updates in the reference's order with separate roundings. */
int qeft_optq_codes(double* w64, const double* u64, const float* scales, const float* zeros, int oc, int m,
                    int g, int bits, double* err_ws, uint8_t* codes, void* stream);

#define QEFT_Y_F32 1
#define QEFT_Y_ACCUMULATE 2

/* ---- decode GEMV (kernels.py:87-157 matvec_structured/irregular/online) ----
 * y[n][o] = sum_i W_hat[o][i] * x[n][i] for n < n_cols (1..16), x/y row-major.
 * y_f32 is a flags word: QEFT_Y_F32 (bit 0) writes fp32 y instead of act_dtype;
 * QEFT_Y_ACCUMULATE (bit 1) adds to y (y += W x, rounded once: a fused residual add).
 * Needs qeft_gemv_workspace_bytes() of scratch: the split-K partials and per-row-block
 * counters of the bulk-copy path (whose first bytes must be ZERO on entry; every call leaves
 * them zero again -- do not share this scratch with other kernels), or the x gather buffer of
 * the generic path. */
size_t qeft_gemv_workspace_bytes(const qeft_linear_t* layer, int n_cols);
int qeft_gemv(const qeft_linear_t* layer, const void* x, int64_t ldx, void* y, int64_t ldy, int y_f32,
              int n_cols, void* workspace, size_t workspace_bytes, void* stream);

/* Profiling only: slots > 0 arms per-CTA globaltimer stamps for the next `slots` bulk-copy
 * GEMV launches (8 x u64 per CTA, 512 CTAs per slot: start, after the PDL wait, after x
 * staging, first stage landed (warp 0), loop done (warp 0), all warps done, end); slots == 0
 * copies them to host_out (slots x 512 x 8 u64, may be NULL) and disarms. */
int qeft_gemv_trace(int slots, unsigned long long* host_out);

/* Several layers that read the same x in ONE launch (a decoder's q/k/v or gate/up): their
 * rows are concatenated, each layer writes its own y (ys[l], common ldy). Up to 3 layers with
 * identical ic, k, bits, g, act_dtype, flags (and column map). */
int qeft_gemv_multi(const qeft_linear_t* const* layers, int n_layers, const void* x, int64_t ldx,
                    void* const* ys, int64_t ldy, int y_f32, int n_cols, void* workspace,
                    size_t workspace_bytes, void* stream);

/* The same launch with x first RMS-normalised (model.py:249-256: x * rsqrt(mean(x^2) + 1e-5)
 * * gain, fp32 gain [ic], the result rounded to the activation dtype) -- bit-identical to
 * qeft_rmsnorm_fwd followed by qeft_gemv_multi; the norm runs inside the GEMV's x staging
 * (or, when that plan cannot host it, as the stand-alone kernel into the workspace, which then
 * needs ldx == ic). Used by the decode step for q/k/v and gate/up. */
int qeft_gemv_multi_rmsnorm(const qeft_linear_t* const* layers, int n_layers, const void* x, int64_t ldx,
                            const float* gain, void* const* ys, int64_t ldy, int y_f32, int n_cols,
                            void* workspace, size_t workspace_bytes, void* stream);

/* y (+)= W_hat (silu(g) * u) for g, u of shape (n, ic), common row pitch ldx (the decode step's
 * down projection over the gate / up outputs, model.py:389-391) -- bit-identical to
 * qeft_silu_mul_fwd followed by qeft_gemv; structured layers combine g and u inside the x
 * staging, other layouts run the stand-alone kernel into the workspace (ldx == ic). */
int qeft_gemv_swiglu(const qeft_linear_t* layer, const void* g, const void* u, int64_t ldx, void* y, int64_t ldy,
                     int y_flags, int n_cols, void* workspace, size_t workspace_bytes, void* stream);

/* ---- prefill / fine-tune GEMMs on tcgen05 (tuning.py:52-103) ----
 * fwd:   y[t][o]  = sum_i W_hat[o][i] x[t][i]                       (qlinear_forward_train)
 * dgrad: dx[t][i] = sum_o W_hat[o][i] dy[t][o]  (+= if accumulate)  (qlinear_backward dX)
 * wgrad: dw[o][j] (+)= sum_t dy[t][o] x[t][weak_j]   fp32 out       (qlinear_backward dW_weak)
 * workspace: qeft_gemm_workspace_bytes() (gather buffer for non-fast layouts). */
size_t qeft_gemm_workspace_bytes(const qeft_linear_t* layer, int T);
/* Tile schedule of the fwd / dgrad GEMMs (process-wide; returns the previous setting of `what`).
 * what = QEFT_SCHED_STREAMK: -1 automatic (stream-K when whole tiles would leave SMs idle in
 *   the last wave), 0 whole tiles only, 1 stream-K whenever every SM gets >= 1 k-block.
 *   Stream-K keeps one ~39 MB fp32 partial buffer per (device, stream), allocated on first use
 *   outside CUDA-graph capture. Initial value: QEFT_GEMM_SK.
 * what = QEFT_SCHED_CTA_PAIRS: 1 one CTA per MMA tile (default), 2 CTA pairs (cta_group::2,
 *   M = 256 over two SMs; even m-block counts, T > 128). Initial value: QEFT_GEMM_CG. */
#define QEFT_SCHED_STREAMK 0
#define QEFT_SCHED_CTA_PAIRS 1
int qeft_gemm_set_schedule(int what, int value);
int qeft_gemm_fwd(const qeft_linear_t* layer, const void* x, int64_t ldx, void* y, int64_t ldy,
                  int T, void* workspace, size_t workspace_bytes, void* stream);
int qeft_gemm_dgrad(const qeft_linear_t* layer, const void* dy, int64_t lddy, void* dx,
                    int64_t lddx, int T, int accumulate, void* workspace, size_t workspace_bytes,
                    void* stream);
int qeft_gemm_wgrad(const qeft_linear_t* layer, const void* dy, int64_t lddy, const void* x,
                    int64_t ldx, float* dw, int T, int accumulate, void* workspace,
                    size_t workspace_bytes, void* stream);
/* wgrad from the saved weak slice only: x_weak[t][j] = x[t][weak_j] (T x k, row pitch
 * ldxw >= k, ldxw % 8 == 0, 16-byte aligned) -- the TrainableLayerState.x_weak of
 * qlinear_forward_train (tuning.py:30-34, 70-71), so the forward pass keeps k of IC columns. */
int qeft_gemm_wgrad_weak(const qeft_linear_t* layer, const void* dy, int64_t lddy, const void* x_weak,
                         int64_t ldxw, float* dw, int T, int accumulate, void* workspace,
                         size_t workspace_bytes, void* stream);

/* dW_weak of up to 3 layers that read the same input (a block's q/k/v, gate/up) in one
 * launch: dws[l] (+)= dys[l]^T x_weak, layers sharing k; dY row pitches 16-byte aligned. */
int qeft_gemm_wgrad_weak_multi(const qeft_linear_t* const* layers, int n_layers, const void* const* dys,
                               const int64_t* lddys, const void* x_weak, int64_t ldxw, float* const* dws, int T,
                               int accumulate, void* stream);

/* ---- optimizer (tuning.py:137-160 adam_step, tuning.py:226-236 clip) ---- */
/* out[0] = sum(g^2) in fp64 (deterministic two-pass). scratch >= 4096 doubles. */
int qeft_grad_sqnorm(const float* g, int64_t n, double* scratch, double* out, void* stream);
/* g /= divisor in fp32 (the reference's acc[name] /= grad_accum, tuning.py:228). */
int qeft_div_scalar(float* g, int64_t n, float divisor, void* stream);
/* Fused clip + Adam over a flat fp32 bucket, in place on w32/m/v.
 * sqnorm: device fp64 from qeft_grad_sqnorm. If it is non-finite nothing is
 * updated and *nonfinite_flag (device int) is set to 1 (DivergenceError).
 * Constants are fp32 images of the reference's Python scalars:
 * c_b1 = f32(b1), c_1mb1 = f32(1-b1), c_b2, c_1mb2, bc1 = f32(1-b1**t),
 * bc2 = f32(1-b2**t). max_norm <= 0 disables clipping. */
int qeft_adam_clip(float* w32, float* m, float* v, const float* g, int64_t n, const double* sqnorm,
                   double max_norm, float lr, float c_b1, float c_1mb1, float c_b2, float c_1mb2,
                   float bc1, float bc2, float eps, int* nonfinite_flag, void* stream);
/* Refresh the weak16 shadows from the fp32 masters after the update.
 * descs: device array of n_layers {int64 offset, int32 oc, k, k_pad, dtype, ptr}. */
typedef struct qeft_shadow_desc {
  int64_t offset; /* element offset of the layer's [oc][k] master in w32 */
  int32_t oc, k, k_pad, act_dtype;
  void* weak16;
} qeft_shadow_desc_t;
int qeft_weak_shadow(const float* w32, const qeft_shadow_desc_t* descs, int n_layers, int max_elems,
                     void* stream);
/* The fine-tune step's optimizer in two passes over the flat bucket (tuning.py:226-236):
 *   qeft_grad_sqnorm_div: out = sum((g / divisor)^2) in fp64, g / divisor rounded to fp32 first
 *                         (the reference's acc /= grad_accum, then the fp64 norm);
 *   qeft_adam_step_flat:  per element of every layer in descs: g / divisor -> global clip (from
 *                         *sqnorm, max_norm a double) -> fp32 Adam on w32/m/v -> weak16 shadow.
 *                         max_rows = the largest oc among the layers. g is not modified. */
int qeft_grad_sqnorm_div(const float* g, int64_t n, float divisor, double* scratch, double* out, void* stream);
int qeft_adam_step_flat(float* w32, float* m, float* v, const float* g, const qeft_shadow_desc_t* descs,
                        int n_layers, int max_rows, float divisor, const double* sqnorm, double max_norm,
                        float lr, float c_b1, float c_1mb1, float c_b2, float c_1mb2, float bc1, float bc2,
                        float eps, int* nonfinite_flag, void* stream);

/* ---- fused elementwise ops of the fine-tuning host model (model.py:249-275, 389-391) ----
 * Activations row-major fp16/bf16 (dt), fp32 math; gains frozen (tuning.py: param_grads=False).
 * rmsnorm: y = gain * x * rstd, rstd[row] = 1/sqrt(mean(x^2) + 1e-5); C % 8 == 0.
 * rmsnorm_bwd: dx = gain*dy*rstd - x*rstd^3*sum(gain*dy*x)/C (+ dres if non-NULL).
 * rope: rotate (j, j + hd/2) pairs of every head of rows = B*T tokens (token t = row % T) by
 *       angle t*inv_freq[j] using cos/sin tables [T][hd/2]; inverse != 0 rotates back (backward);
 *       hd even (16-byte vector path when hd % 16 == 0).
 * silu_mul: f = silu(g) * u and (dg, du) from df; n % 8 == 0. */
int qeft_rmsnorm_fwd(const void* x, const float* gain, void* y, float* rstd, int rows, int C, int dt, void* stream);
int qeft_rmsnorm_bwd(const void* dy, const void* x, const float* gain, const float* rstd, const void* dres,
                     void* dx, int rows, int C, int dt, void* stream);
/* Decode step: q_out = rope(q), k_cache[b][h][pos] = rope(k), v_cache[b][h][pos] = v for q/k/v
 * of shape (B, H*hd) at the position *pos (a device int64, so one CUDA graph serves every
 * step); caches (B, H, T_cache, hd); cos/sin tables [T_cache][hd/2]. */
int qeft_rope_kv(const void* q, const void* k, const void* v, void* q_out, void* k_cache, void* v_cache,
                 const float* cos_t, const float* sin_t, const int64_t* pos, int B, int H, int hd, int T_cache, int dt,
                 void* stream);
/* Decode step attention with the rotary + cache append fused in: q, k, v (B, H*hd) of the new
 * token; k rotated and k/v written to the caches (B, H, T_cache, hd) at *pos (device int64);
 * o (B, H*hd) = softmax(rot(q) . K[0..pos]^T / sqrt(hd)) V[0..pos], fp32 softmax; hd = 128. */
size_t qeft_decode_attention_workspace_bytes(int B, int H, int hd);
/* workspace: qeft_decode_attention_workspace_bytes(), zero-filled once (its counters are left at
 * zero by every call), one per stream. */
int qeft_decode_attention(const void* q, const void* k, const void* v, void* k_cache, void* v_cache,
                          const float* cos_t, const float* sin_t, const int64_t* pos, void* o, int B, int H, int hd,
                          int T_cache, int dt, void* workspace, size_t workspace_bytes, void* stream);
int qeft_rope(const void* in, void* out, const float* cos_t, const float* sin_t, int64_t rows, int T, int H,
              int hd, int inverse, int dt, void* stream);
int qeft_silu_mul_fwd(const void* g, const void* u, void* f, int64_t n, int dt, void* stream);
int qeft_silu_mul_bwd(const void* df, const void* g, const void* u, void* dg, void* du, int64_t n, int dt,
                      void* stream);

/* Next-token cross-entropy over fp16/bf16 logits z [rows][ldz] (V classes, V and the row
 * pitches multiples of 8, V <= 65536), fp32 math (model.py:531-547):
 * fwd: loss[r] = lse[r] - z[r][tgt[r]], lse[r] = log(sum_v exp(z[r][v])) (saved for bwd);
 * bwd: dz[r][v] = (exp(z[r][v] - lse[r]) - [v == tgt[r]]) * (*gscale), in z's dtype
 *      (gscale: device fp32, e.g. dL/dmean / rows). */
int qeft_cross_entropy_fwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, float* loss,
                           float* lse, int dt, void* stream);
int qeft_cross_entropy_bwd(const void* z, int64_t ldz, int rows, int V, const int64_t* tgt, const float* lse,
                           const float* gscale, void* dz, int64_t lddz, int dt, void* stream);

/* Thread-local message for the last non-zero return. */
const char* qeft_last_error(void);
/* Library build string (arch, version). */
const char* qeft_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QEFT_B200_H */
