// mma_rate.cu — measured tcgen05.mma issue-to-completion throughput per SM for
// the instruction shapes the FlashBias kernels use (bf16, fp32 accumulate).
// Every SM runs one CTA that issues `iters` back-to-back MMAs into TMEM and
// waits for the commit; cycles/MMA = elapsed / iters.
#include <cuda.h>
#include <stdio.h>

#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"

using namespace fb;

__global__ void rate_kernel(int mode, int n, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t s0 = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 32) {  // one lane issues; descriptors precomputed, loop unrolled x16
    const uint32_t idesc_k = make_idesc(128, n, false, false, true);
    const uint32_t idesc_mn = make_idesc(128, n, true, true, true);
    const uint32_t idesc_ts = make_idesc(128, n, false, true, true);
    const uint64_t dk_a = kmajor_desc(s0, 128, 128, 0), dk_b = kmajor_desc(s0 + 65536, n, 128, 0);
    const uint64_t dm_a = mnmajor_desc(s0, 128, 128, 0), dm_b = mnmajor_desc(s0 + 65536, 128, 128, 0);
    const int m = mode % 10;
    const bool two = mode >= 10;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 16) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t d = tm + (two ? (u & 1) * 128 : 0);
        if (m == 0) mma_ss(d, dk_a + 2 * (u & 3), dk_b + 2 * (u & 3), idesc_k, 1u);
        else if (m == 1) mma_ss(d, dm_a + 128 * (u & 7), dm_b + 128 * (u & 7), idesc_mn, 1u);
        else mma_ts(d, tm + 256 + (u & 7) * 8, dm_b + 128 * (u & 7), idesc_ts, 1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[3] = {"SS K/K", "SS MN/MN", "TS A=tmem B=MN"};
  for (int mode : {0, 1, 2, 10, 12})
    for (int n : {64, 128, 256}) {
      if (n == 256 && (mode % 10) != 0) continue;
      const int iters = 4096;
      rate_kernel<<<148, 128, 200 * 1024>>>(mode, n, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      const double flops = 2.0 * 128 * n * 16;
      printf("%-16s acc=%d M=128 N=%3d K=16: %6.1f cycles/MMA (floor %d) -> %.0f FLOP/clk/SM\n", names[mode % 10],
             mode >= 10 ? 2 : 1, n,
             avg / iters, 128 * n / 256, flops / (avg / iters));
    }
  return 0;
}
