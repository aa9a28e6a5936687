// mma_rate2.cu — straight-line tcgen05.mma throughput (no per-MMA control flow):
// one thread issues REP unrolled MMAs with loop-invariant descriptors.
#include <cuda.h>
#include <stdio.h>
#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"
using namespace fb;

template <int MODE, int N>
__global__ void k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t s0 = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    constexpr uint32_t idk = make_idesc(128, N, false, false, true);
    constexpr uint32_t idt = make_idesc(128, N, false, true, true);
    const uint64_t a = kmajor_desc(s0, 128, 128, 0), b = kmajor_desc(s0 + 65536, N, 128, 0);
    const uint64_t bm = mnmajor_desc(s0 + 65536, 128, 128, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (MODE == 0) mma_ss(tm, a, b, idk, 1u);
        else mma_ts(tm, tm + 256, bm, idt, 1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <int MODE, int N>
void run(const char* nm) {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 512;
  k<MODE, N><<<148, 128, 200 * 1024>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-8s N=%3d: %6.1f cycles/MMA (floor %d)\n", nm, N, avg / (iters * 8), 128 * N / 256);
}

int main() {
  run<0, 64>("SS"); run<0, 128>("SS"); run<0, 256>("SS");
  run<1, 64>("TS"); run<1, 128>("TS"); run<1, 256>("TS");
  return 0;
}
