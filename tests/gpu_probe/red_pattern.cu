// red_pattern.cu — fp32 reduce-add throughput into an L2-resident, row-pitched
// accumulator (the backward's transposed dQ accumulator [D, N]: row = head dim,
// 64 KB pitch) for access patterns a register-direct dQ drain could use, all
// 148 SMs active, 128 threads per CTA:
//   mode 0: red.global.add.v2.f32, warp = 16 rows x 32 B (the tcgen05.ld.16x256b
//           fragment: 4 lanes share a row, 2 consecutive columns each)
//   mode 1: red.global.add.v4.f32, warp = 512 contiguous bytes of one row (coalesced)
//   mode 2: red.global.add.v4.f32, warp = 32 rows x 16 B (tcgen05.ld.32x32b: lane = row)
//   mode 3: red.global.add.v2.f32, warp = 16 rows x 32 B with .L2::cache_hint-free plain red, 2 ops in a row
// Prints B/clk/SM (bytes added per SM per SM-clock) and the aggregate GB/s.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(float* g, int iters, int rows, long long pitch, unsigned long long* out) {
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  float* base = g + static_cast<long long>(blockIdx.x) * rows * pitch;  // this CTA's region (rows x pitch floats)
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // one "block" = 128 rows x 128 columns of fp32 (64 KB) per CTA, like one dQ^T tile
    const int col0 = (it * 128) % 512;  // 4 column windows: 256 KB touched per CTA (L2 resident)
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      if (MODE == 0 || MODE == 3) {
        // warp w covers rows [32w, 32w+32) in two 16-row halves; 16 column groups of 8
        const int half = i & 1, cg = i >> 1;
        const int row = 32 * w + 16 * half + (l >> 2);
        const int col = col0 + cg * 8 + 2 * (l & 3);
        float* p = base + row * pitch + col;
        asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(1.f) : "memory");
      } else if (MODE == 1) {
        const int row = 32 * w + i;
        float* p = base + row * pitch + col0 + 4 * l;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f),
                     "f"(1.f) : "memory");
      } else {
        const int row = 32 * w + l;
        float* p = base + row * pitch + col0 + 4 * i;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f),
                     "f"(1.f) : "memory");
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (t == 0) out[blockIdx.x] = clock64() - t0;
}

template <int MODE>
void run(const char* name) {
  const int ctas = 148, rows = 128;
  const long long pitch = 2048;  // floats per row in the region (8 KB): 128 rows x 8 KB = 1 MB per CTA... keep L2 resident
  float* g;
  cudaMalloc(&g, sizeof(float) * ctas * rows * pitch);
  cudaMemset(g, 0, sizeof(float) * ctas * rows * pitch);
  unsigned long long* d;
  cudaMalloc(&d, ctas * 8);
  const int iters = 200;
  k<MODE><<<ctas, 128>>>(g, 10, rows, pitch, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<ctas, 128>>>(g, iters, rows, pitch, d);
  cudaEventRecord(e1);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s failed\n", name); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < ctas; ++i) avg += h[i];
  avg /= ctas;
  const double bytes = static_cast<double>(iters) * 128 * 128 * 4;  // per CTA
  printf("%-44s %6.1f B/clk/SM, aggregate %7.1f GB/s\n", name, bytes / avg, bytes * ctas / (ms * 1e-3) / 1e9);
  cudaFree(g);
  cudaFree(d);
}

int main() {
  run<0>("red.v2 16 rows x 32 B per warp (16x256b)");
  run<1>("red.v4 512 B contiguous per warp");
  run<2>("red.v4 32 rows x 16 B per warp (32x32b)");
  run<0>("red.v2 16 rows x 32 B per warp (again)");
  return 0;
}
