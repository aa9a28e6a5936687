// pair_rate.cu — issue rate of back-to-back tcgen05.mma.cta_group::2 (M=256,
// N=128 / 256, K=16, SS) from the leader CTA of a 2-CTA cluster, against the
// single-CTA M=128 floor measured by mma_rate2.cu (N=128: 64 cycles / MMA).
// 74 clusters = 148 SMs busy.
#include <cuda.h>
#include <stdio.h>
#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"
using namespace fb;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t / 32;
  const uint32_t s0 = (smem_u32(sm) + 1023) & ~1023u;
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (cta_rank() == 0 && t == 0) {
    const uint64_t a = kmajor_desc(s0, 128, 128, 0), b = kmajor_desc(s0 + 65536, N / 2, 128, 0);
    const uint32_t idesc = make_idesc(256, N, false, false, true);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm), "l"(a), "l"(b),
                     "r"(idesc), "r"(1u) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    mbar_wait(&bar, 0);
    out[blockIdx.x / 2] = clock64() - t0;
  } else if (t == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

template <int N>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 74 * 8);
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  const int iters = 512;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k<N>, iters, d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d: %s\n", N, cudaGetErrorString(e)); return; }
  unsigned long long h[74]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 74; ++i) avg += h[i]; avg /= 74;
  printf("pair SS M=256 N=%3d K=16: %6.1f cycles/MMA (= %d MACs per SM per cycle; single-CTA M=128 floor: 4096)\n",
         N, avg / (iters * 8), static_cast<int>(256.0 * N * 16 / 2 / (avg / (iters * 8))));
}

int main() { run<128>(); run<256>(); return 0; }
