// mma_sync_tf32_rate.cu — throughput of the warp-level mma.sync.m16n8k8 tf32 (and bf16 m16n8k16 for
// comparison) on sm_100a: 148 CTAs of W warps, 8 independent accumulators per warp.
// Prints MACs / clk / SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_sync_tf32_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(int iters, float* out, long long* cyc) {
  float acc[8][4] = {};
  uint32_t a[4] = {0x3f800000u, 0x3f800000u, 0x3f800000u, 0x3f800000u}, b[2] = {0x3f800000u, 0x3f800000u};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 16 * 512 * 4); cudaMalloc(&cyc, 8);
  for (int kind = 0; kind < 2; ++kind)
    for (int warps : {4, 8, 16}) {
      const int iters = 4096, blocks = 148;
      auto f = kind == 0 ? k<0> : k<1>;
      f<<<blocks, warps * 32>>>(16, out, cyc);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      f<<<blocks, warps * 32>>>(iters, out, cyc);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double macs = (kind == 0 ? 16.0 * 8 * 8 : 16.0 * 8 * 16) * 8 * iters * warps;  // per CTA
      printf("%s warps/SM=%2d: %.0f MACs/clk/SM (cta0 cycles %lld), chip %.1f TFLOP/s\n",
             kind == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16", warps, macs / c, c, 2 * macs * blocks / (ms * 1e-3) / 1e12);
    }
  return 0;
}
