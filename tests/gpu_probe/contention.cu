// contention.cu — does a tcgen05.mma stream share shared-memory / TMEM bandwidth
// with thread-issued st.shared / tcgen05.ld traffic?  One thread issues MMAs
// (SS or TS, N = 64/128) while 8 other warps run a background load until the
// MMA stream finishes; prints MMA cycles per instruction and the background
// bytes per clock achieved during the window.
//   bg 0: none   1: st.shared.v4 (disjoint region)   2: tcgen05.ld 32x32b.x32
#include <cuda.h>
#include <stdio.h>
#include "../../paper_2505_12044_b200/csrc/fb_sm100.cuh"
using namespace fb;

template <int MODE, int N, int BG>
__global__ void k(int iters, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  __shared__ unsigned long long bg_bytes[8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t s0 = (smem_u32(smem) + 1023) & ~1023u;
  uint8_t* sp = smem + (s0 - smem_u32(smem));
  if (warp == 0) {
    if (lane == 0) {
      constexpr uint32_t idk = make_idesc(128, N, false, false, true);
      constexpr uint32_t idt = make_idesc(128, N, false, true, true);
      const uint64_t a = kmajor_desc(s0, 128, 128, 0), b = kmajor_desc(s0 + 32768, N, 128, 0);
      const uint64_t bm = mnmajor_desc(s0 + 32768, 128, 128, 0);
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
      long long t1 = clock64();
      done = 1;
      out[blockIdx.x * 2] = t1 - t0;
    }
  } else if (warp >= 4 && warp < 12 && BG != 0) {
    float acc = 0.f;
    unsigned long long nbytes = 0;
    long long t0 = clock64();
    if (BG == 1) {
      uint4* dst = reinterpret_cast<uint4*>(sp + 98304 + (warp - 4) * 8192);
      uint4 v = make_uint4(lane, 1, 2, 3);
      while (!done) {
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[(j * 32 + lane) & 511] = v;
        v.x += 1;
        nbytes += 16 * 32 * 16;
      }
    } else {
      const uint32_t ta = tm + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 384 + (warp >> 3) * 64;
      uint32_t r[32];
      while (!done) {
        tmem_ld32(ta, r);
        tmem_ld32(ta + 32, r);
        tmem_wait_ld();
        acc += __uint_as_float(r[lane & 31]);
        nbytes += 2 * 32 * 32 * 4;
      }
    }
    long long t1 = clock64();
    if (lane == 0) bg_bytes[warp - 4] = nbytes;
    if (lane == 0 && warp == 4) out[blockIdx.x * 2 + 1] = t1 - t0;
    if (acc == 1234.5f) sink[0] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0 && BG != 0) {
    unsigned long long s = 0;
    for (int i = 0; i < 8; ++i) s += bg_bytes[i];
    out[blockIdx.x * 2 + 1] = s;  // total bytes
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <int MODE, int N, int BG>
void run() {
  unsigned long long* d; float* s;
  cudaMalloc(&d, 148 * 16); cudaMalloc(&s, 64);
  cudaMemset(d, 0, 148 * 16);
  cudaFuncSetAttribute(k<MODE, N, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 2048;
  k<MODE, N, BG><<<148, 384, 200 * 1024>>>(iters, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, bytes = 0;
  for (int i = 0; i < 148; ++i) { cyc += h[2 * i]; bytes += h[2 * i + 1]; }
  cyc /= 148; bytes /= 148;
  printf("%s N=%3d bg=%s: %6.1f cycles/MMA (floor %d), bg %.1f B/clk\n", MODE ? "TS" : "SS", N,
         BG == 0 ? "none " : (BG == 1 ? "st.sh" : "ldtm "), cyc / (iters * 8), 128 * N / 256,
         BG ? bytes / cyc : 0.0);
}

int main() {
  run<0, 64, 0>(); run<0, 64, 1>(); run<0, 64, 2>();
  run<0, 128, 0>(); run<0, 128, 1>(); run<0, 128, 2>();
  run<1, 128, 0>(); run<1, 128, 1>(); run<1, 128, 2>();
  run<1, 64, 0>(); run<1, 64, 1>(); run<1, 64, 2>();
  return 0;
}
