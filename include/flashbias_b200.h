/*
 * flashbias_b200.h — C ABI of the B200-native FlashBias attention path.
 *
 * This is the device boundary that sits directly below the reference's
 * L3 engine.  Every entry point is `extern "C"`, takes
 * plain pointers / sizes / a CUDA stream, never allocates, and is stream
 * ordered.  Tensors are described by `fb_tensor` (rank-4 [B, H, L, D] views;
 * a stride of 0 or a size-1 dim means broadcast along that dim).
 *
 * Reference interfaces each entry point replaces (paths relative to the
 * reference package root `pkg/src/flashbias/`):
 *
 *   fb_attn_fwd        flashbias_attention      attention.py:205-230
 *                      tiled_attention (Dense)  attention.py:140-202 (187-188)
 *                      tiled_attention (NoBias) attention.py:140-202
 *   fb_attn_bwd[_ex]   (no reference: SPEC.md:183) — gradient of the above,
 *                      restated in oracle/flashbias_oracle.py:attention_bwd
 *   fb_prepare_factors concat_cols(q, sqrt(C)*fq) / concat_cols(k, fk)
 *                      core.py:54-62 called at attention.py:227-228, plus the
 *                      bf16 k-way split
 *   fb_factor_alibi    decompose_alibi          decompose.py:37-52
 *   fb_factor_spatial  decompose_spatial        decompose.py:55-81
 *   fb_fold_factor_grads  chain rule from split columns back to logical
 *                      factors (inverse of fb_prepare_factors)
 *   fb_dense_from_factors  generate_bias (AlibiBias / SpatialDistanceBias)
 *                      bias.py:158-178 (dense-baseline input, K8)
 *
 * Error codes map onto the reference exception taxonomy (errors.py:4-25):
 *   FB_OK=0, FB_ESHAPE=1 (ShapeError), FB_EMASK=2 (MaskError),
 *   FB_ECONFIG=3 (ConfigError), FB_EVALUE=4 (ValidationError),
 *   FB_ECUDA=5 (RuntimeError).  Validation happens before any launch,
 *   exactly like the reference validates before compute
 *   (attention.py:77-93, 215-223).  fb_last_error() returns a thread-local
 *   message for the last failing call on the calling thread.
 */
#ifndef FLASHBIAS_B200_H
#define FLASHBIAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FB_ABI_VERSION 1

enum fb_status {
  FB_OK = 0,
  FB_ESHAPE = 1,
  FB_EMASK = 2,
  FB_ECONFIG = 3,
  FB_EVALUE = 4,
  FB_ECUDA = 5
};

enum fb_dtype { FB_F32 = 0, FB_BF16 = 1, FB_F16 = 2, FB_F64 = 3 };

enum fb_mask { FB_MASK_NONE = 0, FB_MASK_CAUSAL = 1 };

/* A strided rank-4 view [B, H, L, D] (element strides).  Rank-2 per-head
 * matrices of the reference are passed as [1, 1, L, D].  The last dim must
 * be contiguous (stride[3] == 1) for tensors that travel through TMA. */
typedef struct fb_tensor {
  void* data;
  int64_t shape[4];
  int64_t stride[4];
  int32_t dtype; /* enum fb_dtype */
} fb_tensor;

/* Forward attention with an optional factored and/or dense additive bias:
 *
 *   logits[b,h,i,j] = scale * ( q[b,h,i,:]·k[b,h,j,:] + uq[b,h,i,:]·uk[b,h,j,:] )
 *                     + bias[b,h,i,j]                  (+ -inf where j > i if causal)
 *   o = softmax_j(logits) · v,     lse[b,h,i] = logsumexp_j(logits)
 *
 * uq/uk are the device-ready factor panels produced by fb_prepare_factors
 * ([Bf,Hf,N,Rpad] / [Bf,Hf,M,Rpad], Rpad a multiple of 16, bf16|f16, Bf/Hf may
 * be 1 = broadcast).  With scale = 1/sqrt(C) and uq = sqrt(C)*fq this is
 * exactly the reference's widened contraction (attention.py:225-230).
 * Pass NULL for uq/uk (no factored bias) and/or bias (no dense bias).
 *
 * q,k,v,o: bf16 or f16 → tcgen05/TMEM/TMA kernel (head dim D in {32,64,128});
 *          f32         → SIMT fp32 kernel (any D <= 128, uq/uk f32, Rpad any).
 * lse: f32 [B,H,N] (may be NULL in inference). */
int fb_attn_fwd(const fb_tensor* q, const fb_tensor* k, const fb_tensor* v,
                const fb_tensor* uq, const fb_tensor* uk, const fb_tensor* bias,
                int mask, float scale, fb_tensor* o, fb_tensor* lse,
                void* stream);

/* Backward of fb_attn_fwd (bf16/f16 only).  Writes dq, dk, dv (same dtype as
 * q), and, when non-NULL, duq/duk: fp32 [B,H,N,Rpad]/[B,H,M,Rpad] gradients
 * of the *split* factor panels (not batch-reduced; fold with
 * fb_fold_factor_grads).  workspace must hold fb_bwd_workspace_bytes(). */
int fb_attn_bwd(const fb_tensor* q, const fb_tensor* k, const fb_tensor* v,
                const fb_tensor* uq, const fb_tensor* uk, const fb_tensor* bias,
                const fb_tensor* o, const fb_tensor* lse, const fb_tensor* dout,
                int mask, float scale, fb_tensor* dq, fb_tensor* dk,
                fb_tensor* dv, fb_tensor* duq, fb_tensor* duk,
                void* workspace, size_t workspace_bytes, void* stream);

/* fb_attn_bwd with a learnable dense bias and flags.
 * dbias (nullable; requires bias): dB = dlogits/dbias = dS, written as
 *   [B,H,N,M] in the bias dtype (rows contiguous, even row stride; the caller
 *   zero-fills it for causal masks -- blocks above the diagonal are not
 *   visited -- and sums it over dims the bias broadcasts).  Replaces the
 *   reference's learnable-bias route (attention.py:187-188 with a trainable
 *   DenseBias); head dim 64 / 128, fused backward only.
 * FB_BWD_DETERMINISTIC: the two-kernel backward (dK'/dV key-stationary + dQ'
 *   query-stationary, no atomics): bitwise reproducible run to run and across
 *   head shardings, at 7 GEMMs per tile instead of 5.  The default (flags = 0)
 *   accumulates dQ with fp32 L2 reduce-adds whose order varies between runs. */
#define FB_BWD_DETERMINISTIC 1
int fb_attn_bwd_ex(const fb_tensor* q, const fb_tensor* k, const fb_tensor* v,
                   const fb_tensor* uq, const fb_tensor* uk, const fb_tensor* bias,
                   const fb_tensor* o, const fb_tensor* lse, const fb_tensor* dout,
                   int mask, float scale, fb_tensor* dq, fb_tensor* dk,
                   fb_tensor* dv, fb_tensor* duq, fb_tensor* duk, fb_tensor* dbias,
                   int flags, void* workspace, size_t workspace_bytes, void* stream);

size_t fb_bwd_workspace_bytes(const fb_tensor* q, const fb_tensor* k);

/* Build device-ready factor panels from logical fp32 factors.
 *   f     : f32 [Bf,Hf,L,R] logical factor (fq or fk)
 *   side  : 0 = query side (multiplied by `premul`, e.g. sqrt(C)), 1 = key side
 *   split : k-way bf16 split level in {1,2,3}; the panels hold, for every
 *           logical rank r, one column per pair (a,b) with a+b <= split-1,
 *           query side carrying part a of premul*fq, key side part b of fk,
 *           so that sum_cols uq*uk == premul * fq·fk to ~2^(-8*split).
 *   out   : bf16|f16 [Bf,Hf,L,Rpad], Rpad = fb_factor_rpad(R, split), zero
 *           padded. */
int fb_prepare_factors(const fb_tensor* f, int side, int split, float premul,
                       fb_tensor* out, void* stream);
/* Both panels of a factor pair in one launch (uq = split(premul * fq), uk = split(fk));
 * same layout contract as two fb_prepare_factors calls. */
int fb_prepare_factor_pair(const fb_tensor* fq, const fb_tensor* fk, int split, float premul,
                           fb_tensor* uq, fb_tensor* uk, void* stream);
int64_t fb_factor_rpad(int64_t rank, int split);
int64_t fb_factor_cols(int64_t rank, int split);

/* Fused neural-factor prologue (replaces evaluating the reference's factor
 * networks, neural.py:44-47 / FactorNetworks.factors 76-77, and then
 * fb_prepare_factors): y = tanh(tanh(x W1 + b1) W2 + b2) W3 + b3 per token,
 * written straight into the split panel layout of fb_prepare_factors.
 *   x  : f32 [1,1,L,in] (in <= 8), w1 [1,1,in,h], b1 [1,1,1,h], w2 [1,1,h,h],
 *        b2 [1,1,1,h], w3 [1,1,h,R], b3 [1,1,1,R] (fp32, row-major, h <= 1024, R <= 128)
 *   out: bf16|f16 [1,1,L,Rpad]; factors: nullable fp32 [1,1,L,R] copy of y. */
int fb_mlp_factor_panels(const fb_tensor* x, const fb_tensor* w1, const fb_tensor* b1,
                         const fb_tensor* w2, const fb_tensor* b2, const fb_tensor* w3,
                         const fb_tensor* b3, int side, int split, float premul,
                         fb_tensor* out, fb_tensor* factors, void* stream);

/* Inverse of fb_prepare_factors for gradients: d(logical f)[b,h,l,r] =
 * postmul * sum over the split columns of rank r whose *partner* part is the
 * leading one, reduced over the batch dim when the factor was broadcast
 * (out Bf = 1 < in B).  in: f32 [B,H,L,Rpad], out: f32 [Bf,Hf,L,R]. */
int fb_fold_factor_grads(const fb_tensor* dpanel, int side, int split,
                         float postmul, fb_tensor* out, void* stream);

/* Closed-form exact factors on device (f32 out, logical rank):
 * ALiBi (decompose.py:37-52): fq[h,i] = slope_h*[1, i+1], fk[h,j] = [-(j+1), 1]
 *   slopes: f32 [H] device pointer; out fq [1,H,N,2], fk [1,H,M,2].
 * Spatial (decompose.py:55-81): R = 9; pos_q [.,.,N,3], pos_k [.,.,M,3] f32,
 *   row_weights f32 [.,H,N] or NULL. */
int fb_factor_alibi(const float* slopes, int64_t heads, int64_t n, int64_t m,
                    fb_tensor* fq, fb_tensor* fk, void* stream);
int fb_factor_spatial(const fb_tensor* pos_q, const fb_tensor* pos_k,
                      const fb_tensor* row_weights, fb_tensor* fq,
                      fb_tensor* fk, void* stream);

/* Dense bias materialisation (K8, bias.py:158-178): out[b,h,i,j] =
 * sum_r fq[b,h,i,r]*fk[b,h,j,r] evaluated in fp32 from logical factors,
 * written as bf16/f16/f32.  Used to build the dense-baseline input. */
int fb_dense_from_factors(const fb_tensor* fq, const fb_tensor* fk,
                          fb_tensor* out, void* stream);

/* D[b,h,i] = sum_c dout[b,h,i,c]*o[b,h,i,c] (fp32), the backward preprocess. */
int fb_bwd_preprocess(const fb_tensor* o, const fb_tensor* dout,
                      fb_tensor* delta, void* stream);

const char* fb_last_error(void);
int fb_abi_version(void);
/* Number of kernel launches issued by this library in this process (all
 * threads, including autograd's backward thread) since the last reset
 * (instrumentation for bench.py "gpu_launches"). */
int64_t fb_launch_count(int reset);

#ifdef __cplusplus
}
#endif

#endif /* FLASHBIAS_B200_H */
