// fb_neural.cu — fused neural-factor prologue: the three-layer MLP of the
// reference's factor networks (pkg/src/flashbias/neural.py:44-47: tanh(x W1 +
// b1) -> tanh(. W2 + b2) -> . W3 + b3) evaluated per token and written straight
// into the kernel's bf16/f16 k-way split factor-panel layout (the same columns
// fb_prepare_factors produces from materialised factors), so a learned bias
// reaches K1 without an fp32 factor tensor round trip.
//
// One CTA = 16 tokens x 256 threads.  Layer 1 (in_dim <= 8) and the hidden
// activations live in shared memory ([16][hidden] fp32 twice); layer 2, the
// h x h GEMV block, has thread j own output columns j, j+256, ... for all 16
// tokens (16 independent FMA chains per weight load, W2 read once per CTA
// through L1/L2); layer 3 likewise over the R outputs; the split epilogue is
// the prepare_factors arithmetic.  SIMT fp32: at AF3-style sizes (N ~ 10^3
// tokens, hidden 256) this is a few microseconds, far below K1.
#include "fb_kernels.h"
#include "fb_sm100.cuh"

namespace fb {

namespace {
constexpr int kTok = 16;

__device__ __forceinline__ float round_dt(float x, int dtype) {
  return dtype == 1 ? __bfloat162float(__float2bfloat16_rn(x)) : __half2float(__float2half_rn(x));
}
__device__ __forceinline__ float part_of(float x, int part, int dtype) {
  float rem = x, cur = 0.f;
  for (int i = 0; i <= part; ++i) {
    cur = round_dt(rem, dtype);
    rem = rem - cur;
  }
  return cur;
}
__device__ __forceinline__ void pair_of(int pidx, int& a, int& b) {
  int tot = 0, base = 0;
  while (pidx >= base + tot + 1) {
    base += tot + 1;
    ++tot;
  }
  a = pidx - base;
  b = tot - a;
}
}  // namespace

__global__ void __launch_bounds__(256) mlp_panels_kernel(MlpParams p) {
  extern __shared__ float sm[];
  float* xs = sm;                      // [kTok][in]
  float* h1 = xs + kTok * 8;           // [kTok][hidden]
  float* h2 = h1 + kTok * p.hidden;    // [kTok][hidden]
  float* ys = h2 + kTok * p.hidden;    // [kTok][R]
  const int t = threadIdx.x;
  const int l0 = blockIdx.x * kTok;
  const int ntok = min(kTok, p.L - l0);
  for (int i = t; i < kTok * p.in_dim; i += blockDim.x) {
    const int tok = i / p.in_dim, c = i % p.in_dim;
    xs[tok * 8 + c] = tok < ntok ? p.x[static_cast<int64_t>(l0 + tok) * p.x_stride + c] : 0.f;
  }
  __syncthreads();
  // layer 1: h1 = tanh(x W1 + b1)
  for (int j = t; j < p.hidden; j += blockDim.x) {
    float acc[kTok];
#pragma unroll
    for (int tok = 0; tok < kTok; ++tok) acc[tok] = p.b1[j];
    for (int c = 0; c < p.in_dim; ++c) {
      const float w = p.w1[c * p.hidden + j];
#pragma unroll
      for (int tok = 0; tok < kTok; ++tok) acc[tok] = fmaf(xs[tok * 8 + c], w, acc[tok]);
    }
#pragma unroll
    for (int tok = 0; tok < kTok; ++tok) h1[tok * p.hidden + j] = tanhf(acc[tok]);
  }
  __syncthreads();
  // layer 2: h2 = tanh(h1 W2 + b2)
  for (int j = t; j < p.hidden; j += blockDim.x) {
    float acc[kTok];
#pragma unroll
    for (int tok = 0; tok < kTok; ++tok) acc[tok] = p.b2[j];
    for (int k = 0; k < p.hidden; ++k) {
      const float w = __ldg(p.w2 + static_cast<int64_t>(k) * p.hidden + j);
#pragma unroll
      for (int tok = 0; tok < kTok; ++tok) acc[tok] = fmaf(h1[tok * p.hidden + k], w, acc[tok]);
    }
#pragma unroll
    for (int tok = 0; tok < kTok; ++tok) h2[tok * p.hidden + j] = tanhf(acc[tok]);
  }
  __syncthreads();
  // layer 3: y = h2 W3 + b3 (R outputs)
  for (int r = t; r < p.R; r += blockDim.x) {
    float acc[kTok];
#pragma unroll
    for (int tok = 0; tok < kTok; ++tok) acc[tok] = p.b3[r];
    for (int k = 0; k < p.hidden; ++k) {
      const float w = __ldg(p.w3 + static_cast<int64_t>(k) * p.R + r);
#pragma unroll
      for (int tok = 0; tok < kTok; ++tok) acc[tok] = fmaf(h2[tok * p.hidden + k], w, acc[tok]);
    }
#pragma unroll
    for (int tok = 0; tok < kTok; ++tok) ys[tok * p.R + r] = acc[tok];
  }
  __syncthreads();
  // split epilogue: panel column c = r * np + pair(a, b); side 0 takes part a of premul*y, side 1 part b of y
  const int np = p.split * (p.split + 1) / 2;
  for (int i = t; i < ntok * p.rpad; i += blockDim.x) {
    const int tok = i / p.rpad, c = i % p.rpad;
    float v = 0.f;
    if (c < p.R * np) {
      int a, b;
      pair_of(c % np, a, b);
      v = part_of(ys[tok * p.R + c / np] * p.premul, p.side == 0 ? a : b, p.out_dtype);
    }
    const int64_t o = static_cast<int64_t>(l0 + tok) * p.out_stride + c;
    if (p.out_dtype == 1) reinterpret_cast<__nv_bfloat16*>(p.out)[o] = __float2bfloat16_rn(v);
    else reinterpret_cast<__half*>(p.out)[o] = __float2half_rn(v);
  }
  if (p.factors_out != nullptr)  // optional fp32 copy of the logical factors (for reports / dense checks)
    for (int i = t; i < ntok * p.R; i += blockDim.x)
      p.factors_out[static_cast<int64_t>(l0 + i / p.R) * p.R + i % p.R] = ys[i];
}

cudaError_t launch_mlp_panels(const MlpParams& p, cudaStream_t s) {
  const size_t smem = (kTok * 8 + 2 * kTok * static_cast<size_t>(p.hidden) + kTok * static_cast<size_t>(p.R)) * 4;
  static std::atomic<uint64_t> attr_mask{0};
  cudaError_t e = smem_attr_once(attr_mask, reinterpret_cast<const void*>(mlp_panels_kernel), 200 * 1024);
  if (e != cudaSuccess) return e;
  mlp_panels_kernel<<<(p.L + kTok - 1) / kTok, 256, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace fb
