// cta_pair_probe.cu — semantics of tcgen05.mma.cta_group::2 on B200 (groundwork
// for a paired backward that halves the dQ reduction traffic).
// Cluster of 2 CTAs; each holds A rows [128 r, 128 r + 128) (A[row][0] = row,
// other K columns 0) and B rows (= N columns) [64 r, 64 r + 64) (B[n][0] = n + 1).
// The leader issues one M=256, N=128, K=16 MMA; a multicast commit signals both
// CTAs; each CTA reads its TMEM accumulator and writes it out.  Expected if the
// pair semantics are "A split by M, B split by N, D split by M":
//   CTA r, lane i, column n  ==  (128 r + i) * (n + 1).
// mode 0: tcgen05.alloc.cta_group::2 in both CTAs; mode 1: cta_group::1 allocs.
#include <cuda.h>
#include <cuda_bf16.h>
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

template <int MODE, int MM = 256>
__global__ void __launch_bounds__(128, 1) k(float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t / 32;
  const uint32_t rank = cta_rank();
  // A: 128 rows x 16 bf16 (32-byte rows, SW32 K-major atom); B: 64 rows x 16 bf16 after it
  __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* Bm = reinterpret_cast<__nv_bfloat16*>(sm + 128 * 32);
  for (int i = t; i < 128 * 16; i += 128) A[i] = __float2bfloat16(0.f);
  for (int i = t; i < 64 * 16; i += 128) Bm[i] = __float2bfloat16(0.f);
  __syncthreads();
  // element (row, k=0) of a SW32 K-major tile: row r at r*32 bytes, 16-byte chunk 0 swizzled with (r>>2)&1
  {
    const int r = t;
    const int chunk = 0 ^ ((r >> 2) & 1);
    A[(r * 32 + chunk * 16) / 2] = __float2bfloat16(static_cast<float>(128 * rank + r));
    if (r < 64) {
      const int c2 = 0 ^ ((r >> 2) & 1);
      Bm[(r * 32 + c2 * 16) / 2] = __float2bfloat16(static_cast<float>(64 * rank + r + 1));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) {
    if (MODE != 1) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (MODE == 2) {  // stage A (this CTA's 128 rows x 16 bf16 = 8 packed columns) into TMEM columns [128, 136)
    uint32_t pk[8];
    for (int c = 0; c < 8; ++c) {
      const float lo = c == 0 ? static_cast<float>(128 * rank + t) : 0.f;
      __nv_bfloat162 v2 = __floats2bfloat162_rn(lo, 0.f);
      pk[c] = *reinterpret_cast<uint32_t*>(&v2);
    }
    const uint32_t lane_off0 = static_cast<uint32_t>((warp & 3) * 32) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lane_off0 + 128),
                 "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]) : "memory");
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
  }
  if (rank == 0 && t == 0 && MODE == 2) {
    const uint64_t bd = make_sdesc(smem_u32(Bm), 16, 256, 6);
    const uint32_t idesc = make_idesc(MM, 128, false, false, true);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
                 "r"(tmem + 128), "l"(bd), "r"(idesc), "r"(0u) : "memory");
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
  } else if (rank == 0 && t == 0) {
    const uint64_t ad = make_sdesc(smem_u32(A), 16, 256, 6);
    const uint64_t bd = make_sdesc(smem_u32(Bm), 16, 256, 6);
    const uint32_t idesc = make_idesc(MM, 128, false, false, true);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(0u) : "memory");
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + lane_off + c0, v);
    tmem_wait_ld();
    for (int c = 0; c < 32; ++c) out[(rank * 128 + t) * 128 + c0 + c] = __uint_as_float(v[c]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if (MODE != 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <int MODE, int MM = 256>
void run(const char* nm) {
  float* d;
  cudaMalloc(&d, 2 * 128 * 128 * 4);
  cudaMemset(d, 0xff, 2 * 128 * 128 * 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 16384;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k<MODE, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k<MODE, MM>, d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", nm, cudaGetErrorString(e)); cudaFree(d); return; }
  static float h[2 * 128 * 128];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (MM == 128) {  // report which (cta, lane) holds which A row: value / (n+1) at column 0
    printf("%s: M=128 pair MMA, value at column 0 (= A row id) per cta/lane:\n", nm);
    for (int r = 0; r < 2; ++r) {
      printf("  cta %d lanes 0..127 (every 16th):", r);
      for (int i = 0; i < 128; i += 16) printf(" %g", h[(r * 128 + i) * 128]);
      printf("\n");
    }
    cudaFree(d);
    return;
  }
  int bad = 0;
  for (int r = 0; r < 2; ++r)
    for (int i = 0; i < 128; ++i)
      for (int n = 0; n < 128; ++n) {
        const float want = static_cast<float>(128 * r + i) * static_cast<float>(n + 1);
        const float got = h[(r * 128 + i) * 128 + n];
        if (!(fabsf(got - want) <= 1e-3f * fmaxf(1.f, fabsf(want)))) {
          if (bad < 6) printf("  %s mismatch cta %d lane %d col %d: got %g want %g\n", nm, r, i, n, got, want);
          ++bad;
        }
      }
  printf("%s: %s (%d mismatches); samples cta0[1][1]=%g cta1[0][0]=%g cta1[5][100]=%g\n", nm,
         bad ? "UNEXPECTED" : "A split by M, B split by N, D rows on their own CTA", bad, h[1 * 128 + 1],
         h[128 * 128], h[(128 + 5) * 128 + 100]);
  cudaFree(d);
}

int main() {
  run<0>("alloc cta_group::2");
  run<1>("alloc cta_group::1");
  run<0, 128>("alloc cta_group::2");
  run<2>("TS pair MMA (A from TMEM)");
  return 0;
}
