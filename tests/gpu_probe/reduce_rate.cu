// reduce_rate.cu — throughput of fp32 add-reductions into L2-resident global
// memory, per SM, all 148 SMs active (the backward's dQ accumulation):
//   mode 0: TMA bulk tensor reduce-add, 16 KB boxes, 1 in flight
//   mode 1: same, 4 in flight (4 stage buffers)
//   mode 2: red.global.add.v4.f32 from registers (128 threads)
//   mode 3: red.global.add.f32 from registers (128 threads)
//   mode 4: TMA bulk tensor store (no reduction), 4 in flight
//   mode 5: cp.reduce.async.bulk (non-tensor, 1-D) add.f32, 16 KB, 4 in flight
// Each CTA targets its own region of `span` bytes (wrapping), so traffic stays in L2.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap map, float* g, int iters, int rows_per_cta,
                                            unsigned long long* out) {
  extern __shared__ __align__(1024) float st[];  // 4 x 16 KB
  const int t = threadIdx.x;
  for (int i = t; i < 4 * 4096; i += 128) st[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int row0 = blockIdx.x * rows_per_cta;
  long long t0 = clock64();
  if (MODE == 6 || MODE == 7) {
    // sweep: 64 KB blocks b = 0.., each reduced 4x (4 chunks of 16 KB, REP passes) before moving on
    if (t == 0) {
      const int nblocks = rows_per_cta / 128;
      for (int it = 0; it < iters; ++it) {
        const int blk = (it / 16) % nblocks, pass = it % 16;
        const int r = row0 + blk * 128 + (pass & 3) * 32;
        if (MODE == 7 && pass < 4) {  // first touch: plain store of zeros-equivalent tile
          asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(st + (it & 3) * 4096)), "r"(0), "r"(r) : "memory");
        } else {
          asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
          asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(st + (it & 3) * 4096)), "r"(0), "r"(r) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else if (MODE == 0 || MODE == 1 || MODE == 4 || MODE == 5) {
    if (t == 0) {
      for (int it = 0; it < iters; ++it) {
        const int s = MODE == 0 ? 0 : (it & 3);
        const int r = row0 + (it * 32) % rows_per_cta;
        if (MODE == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        if (MODE == 4)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(st + s * 4096)), "r"(0), "r"(r) : "memory");
        else if (MODE == 5)
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 16384;" ::"l"(
                           g + static_cast<int64_t>(r) * 128), "r"(smem_u32(st + s * 4096)) : "memory");
        else
          asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(st + s * 4096)), "r"(0), "r"(r) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    // 16 KB per iteration = 32 rows x 128 floats; thread t covers column chunk (t & 31) * 4 of rows (t >> 5) + 4i
    for (int it = 0; it < iters; ++it) {
      const int r = row0 + (it * 32) % rows_per_cta;
      float* base = g + static_cast<int64_t>(r) * 128;
#pragma unroll 8
      for (int i = 0; i < 8; ++i) {
        float* p = base + ((t >> 5) + 4 * i) * 128 + (t & 31) * 4;
        if (MODE == 2) {
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                       : "memory");
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) atomicAdd(p + c, 1.f);
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
  if (t == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE>
void run(const char* name, int rows_per_cta, int ctas) {
  float* g;
  const int64_t rows = static_cast<int64_t>(rows_per_cta) * ctas;
  cudaMalloc(&g, rows * 128 * 4);
  cudaMemset(g, 0, rows * 128 * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {128, 32};
  cuuint32_t es[2] = {1, 1};
  reinterpret_cast<EncodeFn>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d;
  cudaMalloc(&d, ctas * 8);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 2000;
  k<MODE><<<ctas, 128, 65536>>>(map, g, 50, rows_per_cta, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<ctas, 128, 65536>>>(map, g, iters, rows_per_cta, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148]; cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < ctas; ++i) avg += h[i]; avg /= ctas;
  const double bytes = static_cast<double>(iters) * 16384;
  printf("%-34s ctas=%3d region=%5d KB/CTA: %6.1f B/clk/SM, aggregate %7.1f GB/s\n", name, ctas,
         rows_per_cta * 512 / 1024, bytes / avg, bytes * ctas / (ms * 1e-3) / 1e9);
  cudaFree(g); cudaFree(d);
}

int main() {
  run<6>("sweep: reduce into memset region", 16384, 148);
  run<7>("sweep: store first, then reduce", 16384, 148);
  for (int rows : {128, 2048}) {
    run<0>("tma reduce 16KB x1 in flight", rows, 148);
    run<1>("tma reduce 16KB x4 in flight", rows, 148);
    run<5>("bulk 1-D reduce 16KB x4", rows, 148);
    run<2>("red.global.add.v4.f32", rows, 148);
    run<3>("atomicAdd f32", rows, 148);
    run<4>("tma store 16KB x4 (no reduce)", rows, 148);
  }
  run<1>("tma reduce 16KB x4 in flight", 2048, 1);
  run<1>("tma reduce 16KB x4 in flight", 2048, 16);
  return 0;
}
