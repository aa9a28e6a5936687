// tmem_rate.cu — tcgen05.ld / tcgen05.st throughput per SM (4 warps = 128 lanes).
#include <cuda.h>
#include <stdio.h>
#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"
using namespace fb;

template <int NW>
__global__ void k(int iters, int mode, unsigned long long* out, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tm + c * 32, r);
      tmem_wait_ld();
      acc += __uint_as_float(r[it & 31]);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st32(tm + c * 32, r);
      tmem_wait_st();
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int NW>
void run(int mode) {
  unsigned long long* d; float* s;
  cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 64);
  const int iters = 1000;
  k<NW><<<148, NW * 32>>>(iters, mode, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  const double bytes = (double)iters * NW * 32 * 128 * 4;  // each warp: 32 lanes x 128 cols x 4 B per iter
  printf("%s warps=%2d: %.1f cycles/iter, %.1f B/clk/SM\n", mode ? "st" : "ld", NW, avg / iters, bytes / avg);
}

int main() { run<4>(0); run<8>(0); run<4>(1); run<8>(1); return 0; }
