// tma_mix.cu — is per-SM TMA throughput shared between bulk-tensor loads and
// bulk-tensor reduce-adds?  148 CTAs; warp 0 streams TMA loads (16 KB boxes,
// 4 buffers, L2-resident source) for a fixed number of boxes while
//   mode 0: nothing else
//   mode 1: warp 1 streams TMA reduce-adds (16 KB, 2 buffers) until loads finish
//   mode 2: warps 2-5 stream red.global.add.v4.f32 (coalesced) until loads finish
//   mode 3: warps 2-5 stream red.global.add.v4.f32, uncoalesced (lane = row, 16 B each)
// Prints load B/clk/SM and reduce B/clk/SM over the load window.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"
using namespace fb;

template <int MODE>
__global__ void __launch_bounds__(192, 1) k(const __grid_constant__ CUtensorMap lmap, const __grid_constant__ CUtensorMap rmap,
                                            float* g, int nloads, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[4];
  __shared__ volatile int done;
  __shared__ unsigned long long red_bytes;
  const int t = threadIdx.x, w = t / 32;
  float* st = reinterpret_cast<float*>(sm + 4 * 16384);
  for (int i = t; i < 2 * 4096; i += blockDim.x) st[i] = 1.f;
  if (t == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1); fence_barrier_init(); done = 0; red_bytes = 0; }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int rbase = blockIdx.x * 128;  // reduce region: 128 rows x 512 B per CTA
  long long t0 = clock64();
  if ((MODE == 4 || MODE == 5) && t == 0) {
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = 0; i < nloads; ++i) {
      const int b = i & 3;
      if (i >= 4) mbar_wait(&bars[b], ((i >> 2) - 1) & 1);
      mbar_arrive_expect_tx(&bars[b], 16384);
      // both CTAs must have freed buffer b before either multicasts into it: cluster barrier every 4 boxes
      if (b == 0) { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
      if ((i & 1) == (int)rank) {
        const int row = (((blockIdx.x >> 1) * 97 + i * 64) % 131072);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;"
                     ::"r"(smem_u32(sm + b * 16384)), "l"(reinterpret_cast<uint64_t>(&lmap)), "r"(0), "r"(row),
                     "r"(smem_u32(&bars[b])), "h"((uint16_t)3) : "memory");
      }
    }
    for (int b = 0; b < 4; ++b) mbar_wait(&bars[b], ((nloads - 4 + b) >> 2) & 1);
    long long t1 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    done = 1;
  } else if (t == 0) {
    for (int i = 0; i < nloads; ++i) {
      const int b = i & 3;
      if (i >= 4) mbar_wait(&bars[b], ((i >> 2) - 1) & 1);
      mbar_arrive_expect_tx(&bars[b], 16384);
      // source: 64-row x 128-col bf16 boxes from a 32 MB L2-resident tensor
      const int row = ((blockIdx.x * 97 + i * 64) % 131072);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm + b * 16384)), "l"(reinterpret_cast<uint64_t>(&lmap)), "r"(0), "r"(row),
                   "r"(smem_u32(&bars[b])) : "memory");
    }
    for (int b = 0; b < 4; ++b) mbar_wait(&bars[b], ((nloads - 4 + b) >> 2) & 1);
    long long t1 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    done = 1;
  } else if ((MODE == 1 || MODE == 5) && t == 32) {
    unsigned long long n = 0;
    int i = 0;
    while (!done) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(&rmap)), "r"(smem_u32(st + (i & 1) * 4096)), "r"(0), "r"(rbase + (i & 3) * 32) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      n += 16384; ++i;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    red_bytes = n;
  } else if ((MODE == 6 || MODE == 7) && w >= 2) {
    unsigned long long n = 0;
    const int tt = t - 64;  // 0..127: warp wq = tt>>5 handles rows 8*wq.. ; lane -> row (lane>>2), column group (lane&3)
    const int lane = tt & 31, wq = tt >> 5;
    while (!done) {
#pragma unroll 4
      for (int i = 0; i < 8; ++i) {
        if (MODE == 6) {
          float* p = g + static_cast<int64_t>(rbase + 8 * ((wq + 4 * i) & 15) + (lane >> 2)) * 128 + (lane & 3) * 4 + 16 * (i >> 2);
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
        } else {
          float* p = g + static_cast<int64_t>(rbase + 8 * ((wq + 4 * i) & 15) + (lane >> 2)) * 128 + (lane & 3) * 2 + 8 * (i >> 2);
          asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(1.f) : "memory");
        }
      }
      n += 8 * (MODE == 6 ? 16 : 8);
    }
    atomicAdd(&red_bytes, n);
  } else if ((MODE == 2 || MODE == 3) && w >= 2) {
    unsigned long long n = 0;
    const int tt = t - 64;  // 0..127
    while (!done) {
#pragma unroll 4
      for (int i = 0; i < 8; ++i) {
        float* p;
        if (MODE == 2) p = g + static_cast<int64_t>(rbase + (tt >> 5) + 4 * i) * 128 + (tt & 31) * 4;
        else p = g + static_cast<int64_t>(rbase + (tt & 31) + 32 * (i & 3)) * 128 + (tt >> 5) * 4 + (i >> 2) * 16;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
      n += 8 * 16;
    }
    atomicAdd(&red_bytes, n);
  }
  __syncthreads();
  if (t == 0) out[blockIdx.x * 2 + 1] = red_bytes;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE>
void run(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  void* src; cudaMalloc(&src, 131072 * 128 * 2); cudaMemset(src, 0, 131072 * 128 * 2);
  float* g; cudaMalloc(&g, 148 * 128 * 512); cudaMemset(g, 0, 148 * 128 * 512);
  CUtensorMap lmap, rmap;
  { cuuint64_t d[2] = {128, 131072}; cuuint64_t s[1] = {256}; cuuint32_t b[2] = {64, 128}; cuuint32_t e[2] = {1, 1};
    enc(&lmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  { cuuint64_t d[2] = {128, 148 * 128}; cuuint64_t s[1] = {512}; cuuint32_t b[2] = {128, 32}; cuuint32_t e[2] = {1, 1};
    enc(&rmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  unsigned long long* d; cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = 6 * 16384;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (MODE == 4 || MODE == 5) ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k<MODE>, lmap, rmap, g, 200, d);
  cudaLaunchKernelEx(&cfg, k<MODE>, lmap, rmap, g, 4000, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
  unsigned long long h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, rb = 0; for (int i = 0; i < 148; ++i) { cyc += h[2 * i]; rb += h[2 * i + 1]; }
  cyc /= 148; rb /= 148;
  printf("%-36s load %6.1f B/clk/SM   reduce %6.1f B/clk/SM\n", name, 4000.0 * 16384 / cyc, rb / cyc);
  cudaFree(src); cudaFree(g); cudaFree(d);
}

int main() {
  run<0>("TMA loads alone");
  run<1>("TMA loads + TMA reduce-add");
  run<2>("TMA loads + red.v4 coalesced");
  run<3>("TMA loads + red.v4 lane=row");
  run<6>("TMA loads + red.v4 8 rows x 64B");
  run<7>("TMA loads + red.v2 8 rows x 32B");
  return 0;
}
