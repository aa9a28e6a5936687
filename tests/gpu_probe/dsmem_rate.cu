// dsmem_rate.cu — distributed shared memory bandwidth between the two CTAs of a
// cluster (148 CTAs = 74 pairs, both directions at once), the channel a paired
// backward would use to pre-sum dQ halves:
//   mode 0: st.async.shared::cluster.v4.f32 with mbarrier complete_tx (each
//           of 128 threads streams 16-byte stores into the peer's 16 KB buffer)
//   mode 1: cp.async.bulk.shared::cluster.shared::cta (one thread, 8 KB bulk copies)
// Prints bytes/clk/SM sent (and received: symmetric).
#include <cuda.h>
#include <stdio.h>
#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"
using namespace fb;

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];  // [0,16K) receive ring 2 x 8 KB, [16K,32K) source
  __shared__ uint64_t full[2];                      // receive side: data landed (tx bytes)
  __shared__ uint64_t freeb[2];                     // send side: peer consumed my previous write
  const int t = threadIdx.x;
  const uint32_t me = cta_rank(), peer = me ^ 1;
  if (t == 0) {
    for (int i = 0; i < 2; ++i) { mbar_init(&full[i], 1); mbar_init(&freeb[i], 1); }
    fence_barrier_init();
  }
  for (int i = t; i < 4096; i += 128) reinterpret_cast<float*>(sm + 16384)[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cluster_sync();
  const uint32_t rbase = mapa(smem_u32(sm), peer);
  const uint32_t rfull = mapa(smem_u32(&full[0]), peer);
  const uint32_t rfree = mapa(smem_u32(&freeb[0]), peer);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it & 1, use = it >> 1;
    // wait until the peer has consumed what I wrote into its slot s last time
    if (use > 0) mbar_wait(&freeb[s], (use - 1) & 1);
    if (t == 0) {  // expect the peer's 8 KB into MY slot s
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(8192) : "memory");
    }
    if (MODE == 0) {
#pragma unroll 4
      for (int i = 0; i < 4; ++i) {  // 128 threads x 4 x 16 B = 8 KB
        const uint32_t off = s * 8192 + (i * 128 + t) * 16;
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                     ::"r"(rbase + off), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f), "r"(rfull + s * 8) : "memory");
      }
    } else if (t == 0) {
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(rbase + s * 8192), "r"(smem_u32(sm + 16384)), "r"(8192), "r"(rfull + s * 8) : "memory");
    }
    // consume the peer's data in my slot s, then tell the peer the slot is free
    mbar_wait(&full[s], use & 1);
    __syncthreads();
    if (t == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rfree + s * 8) : "memory");
  }
  long long t1 = clock64();
  cluster_sync();
  if (t == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* nm) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 32768 + 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  const int iters = 4000;
  cudaLaunchKernelEx(&cfg, k<MODE>, 100, d);
  cudaLaunchKernelEx(&cfg, k<MODE>, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", nm, cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-28s %.1f B/clk/SM each way (%.0f cycles per 8 KB)\n", nm, iters * 8192.0 / avg, avg / iters);
}

int main() {
  run<0>("st.async v4 (128 threads)");
  run<1>("cp.async.bulk 8 KB");
  return 0;
}
