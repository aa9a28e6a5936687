// umma_probe.cu — single-CTA probes of the tcgen05 building blocks used by the
// FlashBias kernels (descriptor encodings, TMA swizzle layouts, A-from-TMEM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o umma_probe umma_probe.cu -lcuda
// Each probe computes D = A * B^T (fp32 accumulate) on the tensor core and
// compares with a host fp64 reference; prints the max abs error per probe.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"

using namespace fb;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

// mode 0: SS, A [M x K] K-major (swizzle sw), B [N x K] K-major
// mode 1: SS, A K-major, B given as [K x N] row-major (MN-major)
// mode 2: TS, A written to TMEM from registers, B [K x N] MN-major
// mode 3: SS with SW32 16-column panels for both (K = 16 * panels)
struct ProbeArgs {
  int mode, M, N, K, sw;
};

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                             const __nv_bfloat16* A, float* D, ProbeArgs a) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + (((smem_u32(raw) + 1023) & ~1023u) - smem_u32(raw));
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  const int atom_cols = a.sw / 2;
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + 128 * 256 * 2;  // A region up to 128 x 256
  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    int bytes = 0;
    if (a.mode == 3) {
      for (int p = 0; p < a.K / 16; ++p) {
        tma_load_4d(smem + p * a.M * 32, &tA, &bar_tma, p * 16, 0, 0, 0);
        tma_load_4d(smem + 128 * 256 * 2 + p * a.N * 32, &tB, &bar_tma, p * 16, 0, 0, 0);
      }
      bytes = a.M * a.K * 2 + a.N * a.K * 2;
    } else {
      if (a.mode != 2) {
        for (int at = 0; at < a.K / atom_cols; ++at)
          tma_load_4d(smem + at * a.M * a.sw, &tA, &bar_tma, at * atom_cols, 0, 0, 0);
        bytes += a.M * a.K * 2;
      }
      if (a.mode == 0) {
        for (int at = 0; at < a.K / atom_cols; ++at)
          tma_load_4d(smem + 128 * 256 * 2 + at * a.N * a.sw, &tB, &bar_tma, at * atom_cols, 0, 0, 0);
      } else {  // B stored [K rows x N cols]; boxes of atom_cols columns
        for (int at = 0; at < a.N / atom_cols; ++at)
          tma_load_4d(smem + 128 * 256 * 2 + at * a.K * a.sw, &tB, &bar_tma, at * atom_cols, 0, 0, 0);
      }
      bytes += a.N * a.K * 2;
    }
    mbar_arrive_expect_tx(&bar_tma, bytes);
  }
  if (a.mode == 2) {  // A row `tid` -> TMEM lanes, packed bf16 pairs at columns [256, 256 + K/2)
    for (int c0 = 0; c0 < a.K / 2; c0 += 16) {
      uint32_t r[16];
      for (int c = 0; c < 16; ++c) {
        __nv_bfloat162 v;
        v.x = A[tid * a.K + 2 * (c0 + c)];
        v.y = A[tid * a.K + 2 * (c0 + c) + 1];
        r[c] = *reinterpret_cast<uint32_t*>(&v);
      }
      tmem_st16(tm + (static_cast<uint32_t>(warp * 32) << 16) + 256 + c0, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_wait(&bar_tma, 0);
    tc_fence_after();
    const bool bmn = a.mode == 1 || a.mode == 2;
    const uint32_t idesc = make_idesc(a.M, a.N, false, bmn, true);
    for (int kk = 0; kk < a.K / 16; ++kk) {
      uint64_t bdesc;
      if (a.mode == 3) bdesc = make_sdesc(sB + kk * a.N * 32, 16, 256, 6);
      else if (bmn) bdesc = mnmajor_desc(sB, a.K, a.sw, kk * 16);
      else bdesc = kmajor_desc(sB, a.N, a.sw, kk * 16);
      if (a.mode == 2) {
        mma_ts(tm, tm + 256 + kk * 8, bdesc, idesc, kk > 0);
      } else {
        const uint64_t adesc = a.mode == 3 ? make_sdesc(sA + kk * a.M * 32, 16, 256, 6) : kmajor_desc(sA, a.M, a.sw, kk * 16);
        mma_ss(tm, adesc, bdesc, idesc, kk > 0);
      }
    }
    tc_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < a.N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16) + c0, r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) D[tid * a.N + c0 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void make_map(EncodeFn enc, CUtensorMap* m, void* ptr, int rows, int cols, int box_cols, int box_rows, int sw) {
  cuuint64_t dims[4] = {(cuuint64_t)cols, (cuuint64_t)rows, 1, 1};
  cuuint64_t strides[3] = {(cuuint64_t)cols * 2, (cuuint64_t)cols * 2 * rows, (cuuint64_t)cols * 2 * rows};
  cuuint32_t box[4] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMapSwizzle s = sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   s, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
}

static int run(EncodeFn enc, ProbeArgs a, const char* name) {
  const int M = a.M, N = a.N, K = a.K;
  std::vector<__nv_bfloat16> hA(M * K), hB(N * K), hBt(K * N);
  std::vector<float> fA(M * K), fB(N * K);
  srand(1234);
  for (int i = 0; i < M * K; ++i) {
    float x = (rand() % 17 - 8) / 8.0f;
    hA[i] = __float2bfloat16(x);
    fA[i] = __bfloat162float(hA[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    float x = (rand() % 13 - 6) / 4.0f;
    hB[i] = __float2bfloat16(x);
    fB[i] = __bfloat162float(hB[i]);
  }
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) hBt[k * N + n] = hB[n * K + k];
  __nv_bfloat16 *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, M * K * 2));
  CK(cudaMalloc(&dB, N * K * 2));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice));
  const bool bmn = a.mode == 1 || a.mode == 2;
  CK(cudaMemcpy(dB, bmn ? hBt.data() : hB.data(), N * K * 2, cudaMemcpyHostToDevice));
  CUtensorMap tA, tB;
  if (a.mode == 3) {
    make_map(enc, &tA, dA, M, K, 16, M, 32);
    make_map(enc, &tB, dB, N, K, 16, N, 32);
  } else {
    make_map(enc, &tA, dA, M, K, a.sw / 2, M, a.sw);
    if (bmn) make_map(enc, &tB, dB, K, N, a.sw / 2, K, a.sw);
    else make_map(enc, &tB, dB, N, K, a.sw / 2, N, a.sw);
  }
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  probe_kernel<<<1, 128, 200 * 1024>>>(tA, tB, dA, dD, a);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-40s FAILED: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  std::vector<float> hD(M * N);
  CK(cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)fA[m * K + k] * fB[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("%-40s M=%d N=%d K=%d sw=%d  max|err|=%.3e (max|ref|=%.3e) %s\n", name, M, N, K, a.sw, maxerr, maxref,
         maxerr < 1e-3 ? "OK" : "MISMATCH");
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return maxerr < 1e-3 ? 0 : 1;
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int idx = 0;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fn;
  int bad = 0;
  if (only < 0 || only == idx) bad += run(enc, {0, 128, 128, 64, 128}, "SS K/K sw128 K=64");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {0, 128, 128, 128, 128}, "SS K/K sw128 K=128");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {0, 128, 64, 128, 128}, "SS K/K sw128 N=64");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {0, 128, 128, 32, 64}, "SS K/K sw64 K=32");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {3, 128, 128, 32, 32}, "SS panels sw32 K=32");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {3, 128, 64, 16, 32}, "SS panels sw32 N=64");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {1, 128, 128, 128, 128}, "SS K/MN sw128 N=128 K=128");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {1, 128, 64, 128, 128}, "SS K/MN sw128 N=64 K=128");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {1, 128, 32, 128, 64}, "SS K/MN sw64 N=32 K=128");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {2, 128, 128, 128, 128}, "TS A-tmem / MN sw128 N=128 K=128");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {2, 128, 64, 128, 128}, "TS A-tmem / MN sw128 N=64 K=128");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {2, 128, 128, 64, 128}, "TS A-tmem / MN sw128 N=128 K=64");
  ++idx;
  if (only < 0 || only == idx) bad += run(enc, {2, 128, 32, 128, 64}, "TS A-tmem / MN sw64 N=32 K=128");
  ++idx;
  printf("%s\n", bad ? "PROBES FAILED" : "ALL PROBES OK");
  return bad;
}
