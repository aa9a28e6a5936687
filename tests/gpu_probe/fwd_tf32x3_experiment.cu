// fwd_tf32x3_experiment.cu — EXPERIMENT (not built into the library): a 3xTF32 mma.sync variant of the
// fp32 forward (K5, C1).  Correct (rel. err 2.5e-6) but 0.219 ms vs 0.102 ms for the SIMT kernel on C1:
// one 4-warp CTA per SM (141 KB of split tiles) leaves the scalar-LDS-fed mma.sync chain latency-bound.
// Kept for reference; it compiles only inside the library tree (fb_kernels.h, fb_sm100.cuh).
//
// Same contract and numerics budget as the SIMT kernel in fb_small.cu (ref: attention.py:205-230, the
// reference's float64 streaming loop): logits = scale * (q.k^T + uq.uk^T) (+ dense bias) (+ causal -inf),
// online softmax, O = P.V, optional LSE.  The two contractions run as 3xTF32 on the warp-level tensor
// cores (mma.sync.m16n8k8.tf32, measured 510 MACs/clk/SM = 270 TFLOP/s on B200,
// tests/gpu_probe/mma_sync_tf32_rate.cu, against 74 TFLOP/s of FP32 FMA): every fp32 operand x is split
// into hi = x with the 13 low mantissa bits cleared (exactly representable in tf32) and lo = x - hi
// (exact in fp32; the tensor core reads its top 11 bits), and a.b = hi_a.hi_b + hi_a.lo_b + lo_a.hi_b
// drops only lo_a.lo_b and lo's truncation: ~2^-21 relative per product, fp32 accumulation.  The factor
// term uq.uk^T (and a dense bias) stays fp64 on the CUDA cores, as do the running max and the
// subtraction inside exp: an ALiBi term of ~500 would otherwise cost fp32 ulps of the exponent.
//
// CTA = 64 query rows x 4 warps, KV blocks of 64 keys.
//   Q.K^T: warp w computes S for all 64 rows x keys 16w..16w+15 (4 m-tiles x 2 n-tiles), so each warp
//          splits only its own 16 K rows (in place: sK <- hi, sKl <- lo); Q is split once per CTA.
//   softmax: row maxima are combined across the 4 warps through shared memory (fp64); P is written to
//          shared memory already split (sPh / sPl); each warp keeps partial row sums (combined at the end).
//   P.V:   warp w computes O rows 16w..16w+15 x all D columns; V is split in place by all threads.
// K(j+1) is in flight (cp.async) during softmax(j) and P.V(j), V(j+1) during Q.K(j+1) and softmax(j+1).
// Split-KV over a thread-block cluster for small grids, partials combined over DSMEM (as fb_small.cu).
#include "fb_kernels.h"
#include "fb_sm100.cuh"

namespace fb {
namespace {

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// d += a.b in 3xTF32 (hi.hi + hi.lo + lo.hi), small terms first
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     const uint32_t (&bh)[2], const uint32_t (&bl)[2]) {
  mma_tf32(d, al, bh);
  mma_tf32(d, ah, bl);
  mma_tf32(d, ah, bh);
}

__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace

template <int D, int SPLIT>
__global__ void __launch_bounds__(128, 1) fwd_tf32x3_kernel(const SimtParams p) {
  constexpr int BM = 64, BN = 64, TQ = D + 4, TV = D + 8, TP = BN + 4, C4 = D / 4, NTD = D / 8;
  extern __shared__ __align__(16) float sm[];
  const int R = p.R;
  float* sQh = sm;                 // [BM][TQ]
  float* sQl = sQh + BM * TQ;      // [BM][TQ]
  float* sK = sQl + BM * TQ;       // [BN][TQ]  raw, then hi (each warp splits its 16 rows)
  float* sKl = sK + BN * TQ;       // [BN][TQ]
  float* sV = sKl + BN * TQ;       // [BN][TV]  raw, then hi
  float* sVl = sV + BN * TV;       // [BN][TV]
  float* sPh = sVl + BN * TV;      // [BM][TP]
  float* sPl = sPh + BM * TP;      // [BM][TP]
  double* xmax = reinterpret_cast<double*>(sPl + BM * TP);  // [4][BM] per-warp row maxima / row sums
  double* sQf = xmax + 4 * BM;                               // [R][BM] fp64 factor columns
  double* sKf = sQf + R * BM;                                // [2][R][BN]

  const int b = blockIdx.z, h = blockIdx.y;
  const int rank = SPLIT > 1 ? static_cast<int>(blockIdx.x % SPLIT) : 0;
  const int q0 = (blockIdx.x / SPLIT) * BM;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31, g = lane >> 2, tq = lane & 3;
  const float* qb = p.q + b * p.q_sb + h * p.q_sh;
  const float* kb = p.k + b * p.k_sb + h * p.k_sh;
  const float* vb = p.v + b * p.v_sb + h * p.v_sh;
  const float* ukb = R > 0 ? p.uk + b * p.uk_sb + h * p.uk_sh : nullptr;

  const int kv_all = p.causal ? min(p.M, q0 + BM) : p.M;
  const int nkv = (kv_all + BN - 1) / BN;
  const int kb0 = nkv * rank / SPLIT, kb1 = nkv * (rank + 1) / SPLIT;
  auto load_k = [&](int kblk) {
#pragma unroll
    for (int it = 0; it < BN * C4 / 128; ++it) {
      const int idx = t + 128 * it, r = idx / C4, c4 = (idx % C4) * 4, j = kblk * BN + r;
      cp16(sK + r * TQ + c4, kb + static_cast<int64_t>(j < p.M ? j : 0) * p.k_sn + c4, j < p.M);
    }
  };
  auto load_v = [&](int kblk) {
#pragma unroll
    for (int it = 0; it < BN * C4 / 128; ++it) {
      const int idx = t + 128 * it, r = idx / C4, c4 = (idx % C4) * 4, j = kblk * BN + r;
      cp16(sV + r * TV + c4, vb + static_cast<int64_t>(j < p.M ? j : 0) * p.v_sn + c4, j < p.M);
    }
  };
  auto load_kf = [&](int kblk) {
    double* dst = sKf + (kblk & 1) * R * BN;
    for (int idx = t; idx < BN * R; idx += 128) {
      const int r = idx % BN, c = idx / BN, j = kblk * BN + r;
      dst[c * BN + r] = j < p.M ? static_cast<double>(ukb[static_cast<int64_t>(j) * p.uk_sn + c]) : 0.0;
    }
  };
  // ---- prologue: Q (raw into sQh), K(kb0), V(kb0); factor columns
#pragma unroll
  for (int it = 0; it < BM * C4 / 128; ++it) {
    const int idx = t + 128 * it, r = idx / C4, c4 = (idx % C4) * 4, row = q0 + r;
    cp16(sQh + r * TQ + c4, qb + static_cast<int64_t>(row < p.N ? row : 0) * p.q_sn + c4, row < p.N);
  }
  if (kb0 < kb1) {
    load_k(kb0);
    load_v(kb0);
  }
  cp_commit();
  for (int idx = t; idx < BM * R; idx += 128) {
    const int r = idx % BM, c = idx / BM, row = q0 + r;
    sQf[c * BM + r] =
        row < p.N ? static_cast<double>(p.uq[b * p.uq_sb + h * p.uq_sh + static_cast<int64_t>(row) * p.uq_sn + c])
                  : 0.0;
  }
  if (kb0 < kb1) load_kf(kb0);
  cp_wait<0>();
  __syncthreads();
  for (int idx = t; idx < BM * D; idx += 128) {  // split Q once
    const int r = idx / D, c = idx % D;
    const float x = sQh[r * TQ + c], hi = tf32_hi(x);
    sQh[r * TQ + c] = hi;
    sQl[r * TQ + c] = x - hi;
  }
  // (the first K/V split below is preceded by a barrier)

  // per-thread state: QK rows mt*16 + g (+8), mt = 0..3 -> 8 rows; the P.V rows are those of mt = w
  double m_run[8];
  float l_part[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    m_run[i] = -INFINITY;
    l_part[i] = 0.f;
  }
  float o[NTD][4];
#pragma unroll
  for (int n = 0; n < NTD; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[n][e] = 0.f;

  for (int kblk = kb0; kblk < kb1; ++kblk) {
    const int kv0 = kblk * BN;
    const bool more = kblk + 1 < kb1;
    const bool edge = kv0 + BN > p.M || (p.causal && kv0 + BN - 1 > q0) || q0 + BM > p.N;
    __syncthreads();  // Q split / previous block's V split and P reads done
    // split this warp's 16 K rows in place
#pragma unroll
    for (int it = 0; it < 16 * D / 32; ++it) {
      const int idx = lane + 32 * it, r = 16 * w + idx / D, c = idx % D;
      const float x = sK[r * TQ + c], hi = tf32_hi(x);
      sK[r * TQ + c] = hi;
      sKl[r * TQ + c] = x - hi;
    }
    __syncwarp();
    // ---- S = Q K^T for 64 rows x keys 16w .. 16w+15
    float s[4][2][4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[mt][nt][e] = 0.f;
#pragma unroll 2
    for (int k0 = 0; k0 < D; k0 += 8) {
      uint32_t bh[2][2], bl[2][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int n = 16 * w + 8 * nt + g;
        bh[nt][0] = __float_as_uint(sK[n * TQ + k0 + tq]);
        bh[nt][1] = __float_as_uint(sK[n * TQ + k0 + tq + 4]);
        bl[nt][0] = __float_as_uint(sKl[n * TQ + k0 + tq]);
        bl[nt][1] = __float_as_uint(sKl[n * TQ + k0 + tq + 4]);
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int r0 = 16 * mt + g;
        const uint32_t ah[4] = {__float_as_uint(sQh[r0 * TQ + k0 + tq]), __float_as_uint(sQh[(r0 + 8) * TQ + k0 + tq]),
                                __float_as_uint(sQh[r0 * TQ + k0 + tq + 4]),
                                __float_as_uint(sQh[(r0 + 8) * TQ + k0 + tq + 4])};
        const uint32_t al[4] = {__float_as_uint(sQl[r0 * TQ + k0 + tq]), __float_as_uint(sQl[(r0 + 8) * TQ + k0 + tq]),
                                __float_as_uint(sQl[r0 * TQ + k0 + tq + 4]),
                                __float_as_uint(sQl[(r0 + 8) * TQ + k0 + tq + 4])};
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) mma3(s[mt][nt], ah, al, bh[nt], bl[nt]);
      }
    }
    __syncthreads();  // every warp done with sK: K(j+1) may land there
    if (more) {
      load_k(kblk + 1);
      cp_commit();
    }
    // ---- logits in fp64, row maxima across the 4 warps
    const double* kf = sKf + (kblk & 1) * R * BN;
    double v[4][2][4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int rl = 16 * mt + g + 8 * hr, row = q0 + rl;
        double mx = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kl = 16 * w + 8 * nt + 2 * tq + e, j = kv0 + kl;
            double su = 0.0;
            for (int c = 0; c < R; ++c) su = fma(sQf[c * BM + rl], kf[c * BN + kl], su);
            double x = (static_cast<double>(s[mt][nt][2 * hr + e]) + su) * static_cast<double>(p.scale);
            if (p.bias && (!edge || (j < p.M && row < p.N)))
              x += p.bias[b * p.bias_sb + h * p.bias_sh + static_cast<int64_t>(row) * p.bias_sn + j];
            if (edge && (j >= p.M || (p.causal && j > row))) x = -INFINITY;
            v[mt][nt][2 * hr + e] = x;
            mx = fmax(mx, x);
          }
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        if (tq == 0) xmax[w * BM + rl] = mx;
      }
    if (more) load_kf(kblk + 1);  // the other buffer: its readers finished before this block's barriers
    __syncthreads();
    float alpha_pv[2] = {1.f, 1.f};
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int rl = 16 * mt + g + 8 * hr, i = 2 * mt + hr;
        const double mb = fmax(fmax(xmax[rl], xmax[BM + rl]), fmax(xmax[2 * BM + rl], xmax[3 * BM + rl]));
        const double m_new = fmax(m_run[i], mb);
        float alpha = 1.f;
        float pk[4] = {0.f, 0.f, 0.f, 0.f};
        if (m_new != -INFINITY) {
          alpha = expf(static_cast<float>(m_run[i] - m_new));
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) pk[2 * nt + e] = expf(static_cast<float>(v[mt][nt][2 * hr + e] - m_new));
          m_run[i] = m_new;
        }
        l_part[i] = l_part[i] * alpha + ((pk[0] + pk[1]) + (pk[2] + pk[3]));
        if (mt == w) alpha_pv[hr] = alpha;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int kl = 16 * w + 8 * nt + 2 * tq;
          const float h0 = tf32_hi(pk[2 * nt]), h1 = tf32_hi(pk[2 * nt + 1]);
          *reinterpret_cast<float2*>(sPh + rl * TP + kl) = make_float2(h0, h1);
          *reinterpret_cast<float2*>(sPl + rl * TP + kl) = make_float2(pk[2 * nt] - h0, pk[2 * nt + 1] - h1);
        }
      }
#pragma unroll
    for (int n = 0; n < NTD; ++n) {
      o[n][0] *= alpha_pv[0];
      o[n][1] *= alpha_pv[0];
      o[n][2] *= alpha_pv[1];
      o[n][3] *= alpha_pv[1];
    }
    if (more) cp_wait<1>();  // V(j) landed (K(j+1) may still be in flight)
    else cp_wait<0>();
    __syncthreads();  // P complete, V visible
    for (int idx = t; idx < BN * D; idx += 128) {  // split V in place
      const int r = idx / D, c = idx % D;
      const float x = sV[r * TV + c], hi = tf32_hi(x);
      sV[r * TV + c] = hi;
      sVl[r * TV + c] = x - hi;
    }
    __syncthreads();
    // ---- O(rows 16w..) += P V
#pragma unroll 2
    for (int k0 = 0; k0 < BN; k0 += 8) {
      const int r0 = 16 * w + g;
      const uint32_t ah[4] = {__float_as_uint(sPh[r0 * TP + k0 + tq]), __float_as_uint(sPh[(r0 + 8) * TP + k0 + tq]),
                              __float_as_uint(sPh[r0 * TP + k0 + tq + 4]),
                              __float_as_uint(sPh[(r0 + 8) * TP + k0 + tq + 4])};
      const uint32_t al[4] = {__float_as_uint(sPl[r0 * TP + k0 + tq]), __float_as_uint(sPl[(r0 + 8) * TP + k0 + tq]),
                              __float_as_uint(sPl[r0 * TP + k0 + tq + 4]),
                              __float_as_uint(sPl[(r0 + 8) * TP + k0 + tq + 4])};
#pragma unroll
      for (int n = 0; n < NTD; ++n) {
        const uint32_t bh[2] = {__float_as_uint(sV[(k0 + tq) * TV + 8 * n + g]),
                                __float_as_uint(sV[(k0 + tq + 4) * TV + 8 * n + g])};
        const uint32_t bl[2] = {__float_as_uint(sVl[(k0 + tq) * TV + 8 * n + g]),
                                __float_as_uint(sVl[(k0 + tq + 4) * TV + 8 * n + g])};
        mma3(o[n], ah, al, bh, bl);
      }
    }
    __syncthreads();  // every warp done with sV / sP
    if (more) {
      load_v(kblk + 1);
      cp_commit();
      cp_wait<1>();  // K(j+1) landed
    }
  }
  cp_wait<0>();
  // ---- row sums: quad, then across warps (through xmax)
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float l = l_part[i];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (tq == 0) xmax[w * BM + 16 * (i >> 1) + g + 8 * (i & 1)] = l;
  }
  __syncthreads();
  // this thread's output rows: 16w + g (+8) = QK row index i = 2w (+1)
  double m_out[2] = {-INFINITY, -INFINITY};
  float l_out[2];
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int rl = 16 * w + g + 8 * hr;
    l_out[hr] = static_cast<float>(((xmax[rl] + xmax[BM + rl]) + xmax[2 * BM + rl]) + xmax[3 * BM + rl]);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)  // m_run[2w + hr] without a dynamic index (keeps m_run in registers)
      if (mt == w) m_out[hr] = m_run[2 * mt + hr];
  }
  if constexpr (SPLIT > 1) {
    // partials -> smem (the K region): m (double) [BM], l [BM], acc [BM][D]
    double* pm = reinterpret_cast<double*>(sK);
    float* pl = reinterpret_cast<float*>(pm + BM);
    float* pa = pl + BM;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int rl = 16 * w + g + 8 * hr;
      if (tq == 0) {
        pm[rl] = m_out[hr];
        pl[rl] = l_out[hr];
      }
#pragma unroll
      for (int n = 0; n < NTD; ++n)
        *reinterpret_cast<float2*>(pa + rl * D + 8 * n + 2 * tq) = make_float2(o[n][2 * hr], o[n][2 * hr + 1]);
    }
    cluster_sync_all();
    constexpr int RS = BM / SPLIT;
    const uint32_t base = smem_u32(sK);
    for (int idx = t; idx < RS * C4; idx += 128) {
      const int r = rank * RS + idx / C4, c4 = (idx % C4) * 4, row = q0 + r;
      double mr[SPLIT];
      float lr[SPLIT];
      double m_all = -INFINITY;
#pragma unroll
      for (int k = 0; k < SPLIT; ++k) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base), "r"(k));
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(mr[k]) : "r"(ra + 8u * r));
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(lr[k]) : "r"(ra + 8u * BM + 4u * r));
        m_all = fmax(m_all, mr[k]);
      }
      float wsum = 0.f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < SPLIT; ++k) {
        const float wk = mr[k] == -INFINITY ? 0.f : expf(static_cast<float>(mr[k] - m_all));
        wsum += wk * lr[k];
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base), "r"(k));
        float4 x;
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                     : "r"(ra + 12u * BM + 4u * (r * D + c4)));
        acc.x = fmaf(wk, x.x, acc.x);
        acc.y = fmaf(wk, x.y, acc.y);
        acc.z = fmaf(wk, x.z, acc.z);
        acc.w = fmaf(wk, x.w, acc.w);
      }
      if (row < p.N) {
        const float inv = wsum > 0.f ? 1.0f / wsum : 0.f;
        *reinterpret_cast<float4*>(p.o + b * p.o_sb + h * p.o_sh + static_cast<int64_t>(row) * p.o_sn + c4) =
            make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        if (p.lse && c4 == 0)
          p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + row] =
              static_cast<float>(m_all + log(static_cast<double>(wsum)));
      }
    }
    cluster_sync_all();
    return;
  }
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int row = q0 + 16 * w + g + 8 * hr;
    if (row >= p.N) continue;
    const float inv = l_out[hr] > 0.f ? 1.0f / l_out[hr] : 0.f;
    float* orow = p.o + b * p.o_sb + h * p.o_sh + static_cast<int64_t>(row) * p.o_sn;
#pragma unroll
    for (int n = 0; n < NTD; ++n)
      *reinterpret_cast<float2*>(orow + 8 * n + 2 * tq) = make_float2(o[n][2 * hr] * inv, o[n][2 * hr + 1] * inv);
    if (p.lse && tq == 0)
      p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + row] =
          static_cast<float>(m_out[hr] + log(static_cast<double>(l_out[hr])));
  }
}

static size_t tf32_smem(int D, int R) {
  return sizeof(float) * (4 * 64 * static_cast<size_t>(D + 4) + 2 * 64 * static_cast<size_t>(D + 8) + 2 * 64 * 68) +
         sizeof(double) * (4 * 64 + static_cast<size_t>(R) * (64 + 128));
}

template <int D, int SPLIT>
static cudaError_t launch_tf32(const SimtParams& p, cudaStream_t s) {
  static std::atomic<uint64_t> attr_mask{0};
  auto kern = fwd_tf32x3_kernel<D, SPLIT>;
  cudaError_t e = smem_attr_once(attr_mask, reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(((p.N + 63) / 64) * SPLIT, p.H, p.B);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = tf32_smem(D, p.R);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = SPLIT;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int D>
static cudaError_t launch_tf32_d(const SimtParams& p, cudaStream_t s) {
  // one CTA per SM: split each row block's KV range over 2 / 4 / 8 CTAs until the grid covers the SMs
  const int64_t rowblocks = static_cast<int64_t>((p.N + 63) / 64) * p.H * p.B;
  const int kvb = (p.M + 63) / 64;
#ifndef FB_TF32_FORCE_SPLIT
  if (rowblocks * 4 <= 148 && kvb >= 16) return launch_tf32<D, 8>(p, s);
  if (rowblocks * 2 <= 148 && kvb >= 8) return launch_tf32<D, 4>(p, s);
  if (rowblocks <= 148 && kvb >= 4) return launch_tf32<D, 2>(p, s);
  return launch_tf32<D, 1>(p, s);
#else  // experiment builds
  if (FB_TF32_FORCE_SPLIT == 8) return launch_tf32<D, 8>(p, s);
  if (FB_TF32_FORCE_SPLIT == 4) return launch_tf32<D, 4>(p, s);
  if (FB_TF32_FORCE_SPLIT == 2) return launch_tf32<D, 2>(p, s);
  return launch_tf32<D, 1>(p, s);
#endif
}

bool fwd_tf32x3_supported(const SimtParams& p) {
  auto al16 = [](const float* ptr, int64_t sn) { return (reinterpret_cast<uintptr_t>(ptr) % 16) == 0 && sn % 4 == 0; };
  return (p.D == 32 || p.D == 64 || p.D == 128) && al16(p.q, p.q_sn) && al16(p.k, p.k_sn) && al16(p.v, p.v_sn) &&
         (reinterpret_cast<uintptr_t>(p.o) % 16) == 0 && p.o_sn % 4 == 0 && p.o_sb % 4 == 0 && p.o_sh % 4 == 0 &&
         p.q_sb % 4 == 0 && p.q_sh % 4 == 0 && p.k_sb % 4 == 0 && p.k_sh % 4 == 0 && p.v_sb % 4 == 0 &&
         p.v_sh % 4 == 0 && tf32_smem(p.D, p.R) <= 227 * 1024;
}

cudaError_t launch_fwd_tf32x3(const SimtParams& p, cudaStream_t s) {
  cudaError_t e = p.D == 32 ? launch_tf32_d<32>(p, s) : p.D == 64 ? launch_tf32_d<64>(p, s) : launch_tf32_d<128>(p, s);
  note_launch();
  return e;
}

}  // namespace fb
