/*
 * elis_ops.h -- per-kernel entry points of libelis, for parity tests and
 * microbenchmarks.  Same conventions as elis.h (DEVICE pointers, `void*`
 * stream, host-validated errors return before anything is enqueued).  bf16
 * arrays are passed as raw uint16_t bit patterns.  These calls allocate and
 * free their own small scratch (they synchronise `stream` when they do), so
 * they are NOT for the hot path -- the predictor runs the same kernels.
 */
#ifndef ELIS_OPS_H_
#define ELIS_OPS_H_

#include "elis.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ELIS_EPI_BIAS_BF16 = 0,      /* out bf16 [M,N] = A W^T + bias                       (QKV, P:121 BERT) */
  ELIS_EPI_BIAS_GELU_BF16 = 1, /* out bf16 [M,N] = GELU_erf(A W^T + bias)             (FFN1)            */
  ELIS_EPI_BIAS_RESID_F32 = 2  /* out f32  [M,N] = A W^T + bias + residual (f32 [M,N]) (out-proj, FFN2)  */
} elis_epilogue;

/* tcgen05/TMEM/TMA GEMM.  A bf16 [M, K] row-major, W bf16 [N, K] row-major (nn.Linear),
 * bias f32 [N]; M >= 1, N % 128 == 0, K % 64 == 0, all 16-byte aligned. */
elis_status elis_op_gemm(const uint16_t* A, const uint16_t* W, const float* bias, const float* residual,
                         void* out, int32_t M, int32_t N, int32_t K, int32_t epilogue, void* stream);

/* fp16 operand precision (elis_config.precision = ELIS_PREC_FP16, the library default at head dim 64):
 * the same tcgen05 GEMM with fp16 A [M, K] / W [N, K] and fp16 output.  epilogue ELIS_EPI_BIAS_BF16
 * (here: fp16 out = A W^T + bias; the QKV projection) or ELIS_EPI_BIAS_GELU_BF16 (fp16 GELU_erf; FFN1).
 * head_major = 1 (bias epilogue): out is written as the attention's head-major planes
 * [N / 64][M][64] (the predictor's QKV layout).  N % 256 == 0, K % 64 == 0. */
elis_status elis_op_gemm_f16(const uint16_t* A, const uint16_t* W, const float* bias, void* out, int32_t M, int32_t N,
                             int32_t K, int32_t epilogue, int32_t head_major, void* stream);

/* tcgen05 GEMM with the fused residual + LayerNorm epilogue (attention-output / FFN2 of a
 * post-LN BERT block): v = A W^T + bias + resid_inout; resid_inout <- LN(v; gamma, beta, eps)
 * (fp32, in place) and outb <- bf16(LN(v)).  N / (N % 256 ? 128 : 256) <= 4 (one cluster per row). */
elis_status elis_op_gemm_ln(const uint16_t* A, const uint16_t* W, const float* bias, float* resid_inout,
                            const float* gamma, const float* beta, float eps, uint16_t* outb, int32_t M, int32_t N,
                            int32_t K, void* stream);

/* FP8 weight preparation (R20): W f32 [rows, cols]
 * (cols % 4 == 0) -> q E4M3 bytes [rows, cols] = RNE-saturate(W[r, :] * 448 / amax_r) and
 * scale f32 [rows] = amax_r / 448 * post (1 * post for an all-zero row). */
elis_status elis_op_quant_rows_e4m3(const float* W, int32_t rows, int32_t cols, uint8_t* q, float* scale, float post,
                                   void* stream);

/* tcgen05 kind::f8f6f4 GEMM: A, W E4M3 bytes [M, K] / [N, K] row-major, fp32 accumulate;
 * v = (A W^T)[m, n] * colscale[n] + bias[n].  epilogue ELIS_EPI_BIAS_BF16: out bf16 [M, N] = v;
 * ELIS_EPI_BIAS_GELU_BF16: out E4M3 bytes [M, N] = E4M3(out_scale * GELU(v)).
 * N % 256 == 0, K % 128 == 0. */
elis_status elis_op_gemm_f8(const uint8_t* A, const uint8_t* W, const float* colscale, const float* bias, void* out,
                            int32_t M, int32_t N, int32_t K, int32_t epilogue, float out_scale, void* stream);

/* fp16 residual stream variant (elis_config.residual16, EPI_BIAS_RESID16_LN): fp16 operands A, W;
 * v = A W^T + bias + resid_inout (fp16 [M, N], read as fp32); resid_inout <- fp16(LN(v)) in place
 * (statistics and normalisation in fp32).  N a multiple of 256, at most 1024.  global_stats = 1
 * (K >= 2048): the row statistics go through global memory between CTA pairs that share no cluster
 * (the predictor's FFN2); the result is bit-identical to the cluster exchange. */
elis_status elis_op_gemm_ln16(const uint16_t* A, const uint16_t* W, const float* bias, uint16_t* resid_inout,
                              const float* gamma, const float* beta, float eps, int32_t M, int32_t N, int32_t K,
                              int32_t global_stats, void* stream);
/* FP8 variant of elis_op_gemm_ln: v = (A W^T) colscale + bias + resid_inout; resid_inout <- LN(v)
 * (fp32, in place), outb E4M3 bytes [M, N] = E4M3(out_scale * LN(v)).  N in {256, 512, 768, 1024}. */
elis_status elis_op_gemm_ln_f8(const uint8_t* A, const uint8_t* W, const float* colscale, const float* bias,
                               float* resid_inout, const float* gamma, const float* beta, float eps, uint8_t* outb,
                               float out_scale, int32_t M, int32_t N, int32_t K, void* stream);

/* Varlen bidirectional multi-head attention ("process tokens in parallel").
 * d = 64: qkv bf16 head-major planes [3 * num_heads][T][64] (plane h = Q of head h, plane
 *         num_heads + h = K, plane 2 num_heads + h = V) -- the layout the QKV GEMM writes;
 * d = 32: qkv bf16 [T, 3H] (Q | K | V, head h at columns h*d .. h*d+d-1 of each third).
 * lengths int32 [n] (sum == T, each in [1, 512]); ctx bf16 [T, H] = per request i and head h:
 * softmax(Q_h K_h^T / sqrt(d)) V_h over the request's own L_i tokens.  d = H / num_heads in {32, 64}. */
elis_status elis_op_attention(const uint16_t* qkv, const int32_t* lengths, int32_t n, int64_t T,
                              int32_t hidden, int32_t num_heads, uint16_t* ctx, void* stream);
/* The same with fp16 planes and fp16 ctx (elis_config.precision = ELIS_PREC_FP16; P rounded to
 * fp16).  d = 64 only. */
elis_status elis_op_attention_f16(const uint16_t* qkv, const int32_t* lengths, int32_t n, int64_t T,
                                  int32_t hidden, int32_t num_heads, uint16_t* ctx, void* stream);

/* Row LayerNorm: y = (u - mean) / sqrt(var + eps) * gamma + beta (population variance).
 * u f32 [rows, H] -> out_f32 [rows, H] and (if non-NULL) out_bf16 [rows, H]; H in {128, 768, 1024}. */
elis_status elis_op_layernorm(const float* u, const float* gamma, const float* beta, float eps,
                              int64_t rows, int32_t H, float* out_f32, uint16_t* out_bf16, void* stream);

/* Exact-fp32 FC layer of the regression head: Y f32 [n, N] = relu?(X f32 [n, K] W f32 [N, K]^T + b). */
elis_status elis_op_fc_f32(const float* X, const float* W, const float* b, float* Y, int32_t n,
                           int32_t N, int32_t K, int32_t relu, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ELIS_OPS_H_ */
