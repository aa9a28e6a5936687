// fb_kernels.h — internal launch interfaces between the C ABI (fb_capi.cu)
// and the kernels.  Not part of the public boundary (include/flashbias_b200.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <type_traits>

namespace fb {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the
// attribute is per device, so a process driving several GPUs sets it on each.
inline cudaError_t smem_attr_once(std::atomic<uint64_t>& mask, const void* kern, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

struct FwdParams {
  int B, H, N, M;
  int causal;
  int num_pairs;      // ceil(N / 256): CTAs per (b,h)
  float scale_log2;   // softmax scale * log2(e)
  void* o;            // [B,H,N,D] output (element strides below)
  int64_t o_sb, o_sh, o_sn;
  float* lse;         // [B,H,N] contiguous, natural-log units (nullable)
  int uq_bb, uq_hb;   // factor / bias broadcast flags (size-1 dims)
  int uk_bb, uk_hb;
  int bias_bb, bias_hb;
  unsigned long long* trace; int trace_cta;  // FB_TRACE builds only
};

struct FwdMaps {
  CUtensorMap q, k, v, uq, uk, bias;
};

cudaError_t launch_fwd_sm100(int d, int rp, bool dense, bool bf16, const FwdMaps& maps,
                             const FwdParams& p, cudaStream_t s);

// ----- backward (tcgen05): dK'/dV (KV-stationary) and dQ' (Q-stationary)
struct BwdParams {
  int B, H, N, M;
  int causal;
  float scale;        // softmax scale
  float scale_log2;   // scale * log2(e)
  const float* lse;   // [B,H,N] natural-log
  const float* delta; // [B,H,N] rowsum(dO * O)
  void* dq; int64_t dq_sb, dq_sh, dq_sn;
  void* dk; int64_t dk_sb, dk_sh, dk_sn;
  void* dv; int64_t dv_sb, dv_sh, dv_sn;
  float* duq; int64_t duq_sb, duq_sh, duq_sn;  // nullable, fp32 [B,H,N,Rpad]
  float* duk; int64_t duk_sb, duk_sh, duk_sn;
  int uq_bb, uq_hb, uk_bb, uk_hb, bias_bb, bias_hb;
  void* dbias; int64_t db_sb, db_sh, db_sn;  // nullable: learnable dense bias gradient [B,H,N,M] (bias dtype)
  unsigned long long* trace; int trace_cta;  // FB_TRACE builds only
};

#ifdef __CUDACC__
// Learnable dense bias (K4): dB[b,h,q,kv] = dS[q,kv] (the bias enters the logits
// unscaled, ref attention.py:187-188).  pk[c2] holds the 16-bit dS of queries
// q0+2c2, q0+2c2+1 for this thread's key kv; neighbouring lanes hold
// neighbouring keys, so lane pairs swap halves and every lane stores one
// 4-byte (kv, kv+1) pair of one query row: a warp writes 64 contiguous bytes of
// two dB rows per store.  Rows are 4-byte aligned (db_sn even, host-padded).
__device__ __forceinline__ void store_dbias_rows(const BwdParams& p, int b, int h, int q0, int kv, int lane,
                                                 const uint32_t (&pk)[32]) {
  uint16_t* base = static_cast<uint16_t*>(p.dbias) + static_cast<int64_t>(b) * p.db_sb +
                   static_cast<int64_t>(h) * p.db_sh;
  const int odd = lane & 1, kve = kv & ~1;
#pragma unroll
  for (int c2 = 0; c2 < 32; ++c2) {
    const uint32_t mine = pk[c2], other = __shfl_xor_sync(0xffffffffu, pk[c2], 1);
    const uint32_t w = odd ? __byte_perm(other, mine, 0x7632) : __byte_perm(mine, other, 0x5410);
    const int q = q0 + 2 * c2 + odd;
    if (q < p.N && kve < p.M) {
      uint16_t* dst = base + static_cast<int64_t>(q) * p.db_sn + kve;
      if (kve + 1 < p.M) *reinterpret_cast<uint32_t*>(dst) = w;
      else *dst = static_cast<uint16_t>(w & 0xffffu);
    }
  }
}
#endif

struct BwdMaps {
  // dKV kernel: streamed 64-row query-side boxes, resident 128-row key side
  CUtensorMap q64, do64, uq64, biasT, k128, v128, uk128;
  // dQ kernel: resident 128-row query side, streamed 64-row key-side boxes
  CUtensorMap q128, do128, uq128, bias, k64, v64, uk64;
  // d=64 fused kernel: factor panels loaded as a second 64-column SW128 atom
  CUtensorMap uq64w, uk128w;
};

cudaError_t launch_bwd_sm100(int d, int rp, bool dense, bool bf16, bool factor_grads,
                             const BwdMaps& maps, const BwdParams& p, cudaStream_t s);
// single-pass backward for d = 128 without factor gradients: dQ reduced into
// an fp32 accumulator [B,H,N,128] through TMA bulk reductions, then converted
cudaError_t launch_bwd_fused_sm100(int rp, bool dense, bool bf16, const BwdMaps& maps, const CUtensorMap& dqacc,
                                   const BwdParams& p, cudaStream_t s);
// d = 128 on 128-key x 128-query tiles (every GEMM N = 128), Rpad <= 16 (factor gradients: Rpad == 16), no
// dense bias
bool bwd_t128_supported(int d, int rp, bool dense, bool factor_grads);
// fgrad: dUq reduce-added through `duq` (fp32 [B,H,N,16], box {16, 128}, 64-byte swizzle, zeroed by the
// caller), dUk written to p.duk
cudaError_t launch_bwd_t128_sm100(int rp, bool bf16, bool fgrad, const BwdMaps& maps, const CUtensorMap& dqacc,
                                  const CUtensorMap& duq, const BwdParams& p, cudaStream_t s);
// dq[b,h,n,:] = acc_t[b,h,:,n] (transposed fp32 accumulator [B,H,128,n4] of the 128x128-tile kernel)
cudaError_t launch_dq_convert(const float* acc, int d, const BwdParams& p, bool bf16, cudaStream_t s);
// single-pass backward for d = 64 (optionally with factor gradients, Rpad <= 64)
cudaError_t launch_bwd_fused64_sm100(int rp, bool dense, bool bf16, bool fgrad, const BwdMaps& maps,
                                     const CUtensorMap& dqacc, const CUtensorMap& duq, const BwdParams& p,
                                     cudaStream_t s);

// ----- SIMT fp32 path (K5)
struct SimtParams {
  int B, H, N, M, D, R;
  int causal;
  float scale;
  const float* q; int64_t q_sb, q_sh, q_sn;
  const float* k; int64_t k_sb, k_sh, k_sn;
  const float* v; int64_t v_sb, v_sh, v_sn;
  const float* uq; int64_t uq_sb, uq_sh, uq_sn;  // nullable (R == 0)
  const float* uk; int64_t uk_sb, uk_sh, uk_sn;
  const float* bias; int64_t bias_sb, bias_sh, bias_sn;  // nullable
  float* o; int64_t o_sb, o_sh, o_sn;
  float* lse;  // nullable, [B,H,N]
};
cudaError_t launch_fwd_simt_f32(const SimtParams& p, cudaStream_t s);

// ----- small kernels
struct Tensor4 {
  void* data;
  int64_t shape[4];
  int64_t stride[4];
  int dtype;
};
cudaError_t launch_prepare_factors(const Tensor4& f, int side, int split, float premul,
                                   const Tensor4& out, cudaStream_t s);
cudaError_t launch_prepare_factor_pair(const Tensor4& fq, const Tensor4& fk, int split, float premul,
                                       const Tensor4& uq, const Tensor4& uk, cudaStream_t s);
cudaError_t launch_fold_factor_grads(const Tensor4& dpanel, int side, int split, float postmul,
                                     const Tensor4& out, cudaStream_t s);
cudaError_t launch_factor_alibi(const float* slopes, int64_t heads, int64_t n, int64_t m,
                                const Tensor4& fq, const Tensor4& fk, cudaStream_t s);
cudaError_t launch_factor_spatial(const Tensor4& pq, const Tensor4& pk, const Tensor4* w,
                                  const Tensor4& fq, const Tensor4& fk, cudaStream_t s);
cudaError_t launch_dense_from_factors(const Tensor4& fq, const Tensor4& fk, const Tensor4& out,
                                      cudaStream_t s);
cudaError_t launch_bwd_preprocess(const Tensor4& o, const Tensor4& dout, const Tensor4& delta,
                                  cudaStream_t s);

int factor_pairs(int split);

// ----- fused neural-factor prologue (fb_neural.cu)
struct MlpParams {
  const float* x; int64_t x_stride;  // [L, in_dim] fp32 coordinates
  int L, in_dim, hidden, R;
  const float *w1, *b1, *w2, *b2, *w3, *b3;  // row-major [in,h] [h] [h,h] [h] [h,R] [R] fp32
  int side, split, rpad, out_dtype;  // panel layout of fb_prepare_factors
  float premul;
  void* out; int64_t out_stride;     // [L, rpad] bf16/f16 panel
  float* factors_out;                // nullable [L, R] fp32
};
cudaError_t launch_mlp_panels(const MlpParams& p, cudaStream_t s);

// debug timeline trace target (fb_debug_set_trace)
void trace_target(unsigned long long** buf, int* cta);

// launch accounting (fb_launch_count)
void note_launch(int n = 1);

}  // namespace fb
