// fb_bwd_sm100.cu — FlashBias backward on sm_100a (K2) and the dense-bias
// baseline backward (K4).  The reference has no backward; the
// math restated here is oracle/flashbias_oracle.py:attention_bwd:
//
//   s = scale * Q' K'^T (+ bias),  P = exp(s - lse),  dP = dO V^T,
//   dS = P * (dP - D),  D = rowsum(dO * O)
//   dV = P^T dO,  dQ' = scale dS K',  dK' = scale dS^T Q'
//
// with Q' = [Q | Uq], K' = [K | Uk]: the factor gradients dUq = scale dS Uk
// and dUk = scale dS^T Uq are the extra columns of the widened products
// (SURVEY §8(a) row a14), issued as extra N=16 UMMAs per panel.
//
// Two deterministic kernels (no atomics):
//   dKV: CTA owns 128 key rows, streams 64-row query blocks.
//        TMEM: S^T [0,64) dP^T [64,128) dV [128,128+D) dK [..+D) dUk [..+16RP)
//   dQ : CTA owns 128 query rows, streams 64-row key blocks, S/dP double
//        buffered.  TMEM: S_b [128b, 128b+64) dP_b [128b+64, 128b+128)
//        dQ [256, 256+D) dUq [256+D, +16RP)
// Both: warps 0-3 elementwise (thread = TMEM lane = row), warp 4 TMA,
// warp 5 TMEM alloc + single-thread MMA issue.  P^T / dS (bf16) overwrite the
// first 32 columns of their fp32 source and feed the next MMA from TMEM.
#include "fb_kernels.h"
#include "fb_sm100.cuh"

namespace fb {

constexpr float kLog2e = 1.4426950408889634f;

template <int D, int RP, bool DENSE>
struct BwdCfg {
  static constexpr int kSW = swizzle_bytes(D);
  static constexpr int kAtomCols = kSW / 2;
  static constexpr int kAtoms = D / kAtomCols;
  static constexpr int kBlk = 64;                 // streamed block length
  static constexpr int kTile128 = 128 * D * 2;    // resident 128-row operand
  static constexpr int kTile64 = 64 * D * 2;      // streamed 64-row operand
  static constexpr int kPanel128 = 128 * 32;
  static constexpr int kPanel64 = 64 * 32;
  static constexpr int kBarBytes = 512;
  static constexpr int kBudget = 232448 - 1024 - kBarBytes;
  static constexpr int kThreads = 192;
  static constexpr int kTmemCols = 512;
  // dKV kernel: resident K, Uk panels, V; ring item = Q, Uq panels, dO (+ bias^T 64x128)
  static constexpr int kKVRes = 2 * kTile128 + RP * kPanel128;
  static constexpr int kKVItem = 2 * kTile64 + RP * kPanel64 + (DENSE ? 64 * 128 * 2 : 0);
  static constexpr int kKVSlot = (kKVItem + 1023) / 1024 * 1024;
  static constexpr int kKVSlotsFit = (kBudget - kKVRes - 1024) / kKVSlot;
  static constexpr int kKVSlots = kKVSlotsFit > 6 ? 6 : kKVSlotsFit;
  static constexpr int kKVSmem = 1024 + kKVRes + kKVSlots * kKVSlot + 1024 + kBarBytes;
  // dQ kernel: resident Q, Uq panels, dO; ring item = K, Uk panels, V (+ bias 128x64)
  static constexpr int kQRes = 2 * kTile128 + RP * kPanel128;
  static constexpr int kQItem = 2 * kTile64 + RP * kPanel64 + (DENSE ? 128 * 64 * 2 : 0);
  static constexpr int kQSlot = (kQItem + 1023) / 1024 * 1024;
  static constexpr int kQSlotsFit = (kBudget - kQRes) / kQSlot;
  static constexpr int kQSlots = kQSlotsFit > 6 ? 6 : kQSlotsFit;
  static constexpr int kQSmem = 1024 + kQRes + kQSlots * kQSlot + kBarBytes;
  static_assert(kKVSlots >= 2 && kQSlots >= 2, "bwd smem ring too small");
};

struct BwdBars {
  uint64_t res_full;
  uint64_t s_full[2];
  uint64_t dp_full[2];
  uint64_t p_ready;
  uint64_t ds_ready[2];
  uint64_t final_;
  uint64_t slot_full[8];
  uint64_t slot_empty[8];
  uint32_t tmem_base;
};

template <typename T>
__device__ __forceinline__ T* row_ptr(void* base, int64_t sb, int64_t sh, int64_t sn, int b, int h, int r) {
  return reinterpret_cast<T*>(base) + static_cast<int64_t>(b) * sb + static_cast<int64_t>(h) * sh +
         static_cast<int64_t>(r) * sn;
}

// Store one TMEM row chunk (32 fp32 cols) scaled, as 16-bit elements.
template <bool BF16>
__device__ __forceinline__ void store_row32(void* dst, const uint32_t (&v)[32], float mul) {
  uint32_t pk[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) pk[c] = pack2<BF16>(__uint_as_float(v[2 * c]) * mul, __uint_as_float(v[2 * c + 1]) * mul);
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) d[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
}

// =====================================================================================
// dK' / dV kernel (KV-stationary)
// =====================================================================================
template <int D, int RP, bool DENSE, bool BF16, bool FGRAD>
__global__ void __launch_bounds__(192, 1)
    fb_bwd_dkv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_uq, const __grid_constant__ CUtensorMap tm_biasT,
                      const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                      const __grid_constant__ CUtensorMap tm_uk, const BwdParams p) {
  using Cfg = BwdCfg<D, RP, DENSE>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t k_base = sbase;
  const uint32_t v_base = sbase + Cfg::kTile128;
  const uint32_t uk_base = sbase + 2 * Cfg::kTile128;
  const uint32_t ring_base = sbase + Cfg::kKVRes;
  float* s_stats = reinterpret_cast<float*>(smem + Cfg::kKVRes + Cfg::kKVSlots * Cfg::kKVSlot);  // [2][2][64]
  BwdBars* bars = reinterpret_cast<BwdBars*>(smem + Cfg::kKVRes + Cfg::kKVSlots * Cfg::kKVSlot + 1024);

  const int warp = warp_id(), lane = lane_id();
  const int nkt = (p.M + 127) / 128;
  const int kt = blockIdx.x % nkt;  // ascending: causal-longest first within a head
  const int bh = blockIdx.x / nkt;  // head-major: resident CTAs share Q/dO via L2
  const int h = bh / p.B, b = bh % p.B;  // a head's batches adjacent (shared bias/L2)
  const int kv0 = kt * 128;
  const int nqb = (p.N + 63) / 64;
  const int i_start = p.causal ? kv0 / 64 : 0;
  const int nblk = nqb - i_start;

  if (warp == 4 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    if (RP > 0) {
      tma_prefetch(&tm_uq);
      tma_prefetch(&tm_uk);
    }
    if (DENSE) tma_prefetch(&tm_biasT);
    mbar_init(&bars->res_full, 1);
    mbar_init(&bars->s_full[0], 1);
    mbar_init(&bars->dp_full[0], 1);
    mbar_init(&bars->p_ready, 4);
    mbar_init(&bars->ds_ready[0], 4);
    mbar_init(&bars->final_, 1);
    for (int s = 0; s < Cfg::kKVSlots; ++s) {
      mbar_init(&bars->slot_full[s], 1);
      mbar_init(&bars->slot_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<Cfg::kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  constexpr uint32_t T_ST = 0, T_DPT = 64, T_DV = 128, T_DK = 128 + D, T_DUK = 128 + 2 * D;

  if (warp == 4) {
    if (lane == 0) {
      const int hq = p.uq_hb ? 0 : h, bq = p.uq_bb ? 0 : b;
      const int hk = p.uk_hb ? 0 : h, bk = p.uk_bb ? 0 : b;
      const int hb_ = p.bias_hb ? 0 : h, bb_ = p.bias_bb ? 0 : b;
      mbar_arrive_expect_tx(&bars->res_full, Cfg::kKVRes);
      for (int a = 0; a < Cfg::kAtoms; ++a) {
        tma_load_4d(smem + a * 128 * Cfg::kSW, &tm_k, &bars->res_full, a * Cfg::kAtomCols, kv0, h, b);
        tma_load_4d(smem + Cfg::kTile128 + a * 128 * Cfg::kSW, &tm_v, &bars->res_full, a * Cfg::kAtomCols, kv0, h, b);
      }
      for (int pn = 0; pn < RP; ++pn)
        tma_load_4d(smem + 2 * Cfg::kTile128 + pn * Cfg::kPanel128, &tm_uk, &bars->res_full, pn * 16, kv0, hk, bk);
      for (int c = 0; c < nblk; ++c) {
        const int q0 = (i_start + c) * 64;
        const int slot = c % Cfg::kKVSlots, use = c / Cfg::kKVSlots;
        if (use > 0) mbar_wait(&bars->slot_empty[slot], (use - 1) & 1);
        uint8_t* dst = smem + Cfg::kKVRes + slot * Cfg::kKVSlot;
        uint64_t* fb_ = &bars->slot_full[slot];
        mbar_arrive_expect_tx(fb_, Cfg::kKVItem);
        for (int a = 0; a < Cfg::kAtoms; ++a) {
          tma_load_4d(dst + a * 64 * Cfg::kSW, &tm_q, fb_, a * Cfg::kAtomCols, q0, h, b);
          tma_load_4d(dst + Cfg::kTile64 + a * 64 * Cfg::kSW, &tm_do, fb_, a * Cfg::kAtomCols, q0, h, b);
        }
        for (int pn = 0; pn < RP; ++pn)
          tma_load_4d(dst + 2 * Cfg::kTile64 + pn * Cfg::kPanel64, &tm_uq, fb_, pn * 16, q0, hq, bq);
        if (DENSE)
          for (int half = 0; half < 2; ++half)
            tma_load_4d(dst + 2 * Cfg::kTile64 + half * 64 * 128, &tm_biasT, fb_, kv0 + half * 64, q0, hb_, bb_);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t id_s = make_idesc(128, 64, false, false, BF16);
      constexpr uint32_t id_d = make_idesc(128, D, false, true, BF16);
      constexpr uint32_t id_u = make_idesc(128, 16, false, true, BF16);
      auto slot_addr = [&](int c) { return ring_base + (c % Cfg::kKVSlots) * Cfg::kKVSlot; };
      auto wait_slot = [&](int c) { mbar_wait(&bars->slot_full[c % Cfg::kKVSlots], (c / Cfg::kKVSlots) & 1); };
      auto issue_st = [&](int c) {
        const uint32_t qb = slot_addr(c);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + T_ST, kmajor_desc(k_base, 128, Cfg::kSW, kk * 16), kmajor_desc(qb, 64, Cfg::kSW, kk * 16), id_s,
                 kk > 0 ? 1u : 0u);
#pragma unroll
        for (int pn = 0; pn < RP; ++pn)
          mma_ss(tmem + T_ST, make_sdesc(uk_base + pn * Cfg::kPanel128, 16, 256, 6),
                 make_sdesc(qb + 2 * Cfg::kTile64 + pn * Cfg::kPanel64, 16, 256, 6), id_s, 1u);
        tc_commit(&bars->s_full[0]);
      };
      auto issue_dpt = [&](int c) {
        const uint32_t dob = slot_addr(c) + Cfg::kTile64;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + T_DPT, kmajor_desc(v_base, 128, Cfg::kSW, kk * 16), kmajor_desc(dob, 64, Cfg::kSW, kk * 16), id_s,
                 kk > 0 ? 1u : 0u);
        tc_commit(&bars->dp_full[0]);
      };
      mbar_wait(&bars->res_full, 0);
      wait_slot(0);
      tc_fence_after();
      issue_st(0);
      issue_dpt(0);
      for (int c = 0; c < nblk; ++c) {
        const uint32_t qb = slot_addr(c), dob = qb + Cfg::kTile64;
        mbar_wait(&bars->p_ready, c & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dV += P^T dO   (K = 64 query rows)
          mma_ts(tmem + T_DV, tmem + T_ST + kk * 8, mnmajor_desc(dob, 64, Cfg::kSW, kk * 16), id_d,
                 (c > 0 || kk > 0) ? 1u : 0u);
        if (c + 1 < nblk) {
          wait_slot(c + 1);
          tc_fence_after();
          issue_st(c + 1);
        }
        mbar_wait(&bars->ds_ready[0], c & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // dK += dS^T Q ; dUk += dS^T Uq
          mma_ts(tmem + T_DK, tmem + T_DPT + kk * 8, mnmajor_desc(qb, 64, Cfg::kSW, kk * 16), id_d,
                 (c > 0 || kk > 0) ? 1u : 0u);
          if constexpr (FGRAD) {
#pragma unroll
            for (int pn = 0; pn < RP; ++pn)
              mma_ts(tmem + T_DUK + pn * 16, tmem + T_DPT + kk * 8,
                     make_sdesc(qb + 2 * Cfg::kTile64 + pn * Cfg::kPanel64 + kk * 16 * 32, 64 * 32, 256, 6), id_u,
                     (c > 0 || kk > 0) ? 1u : 0u);
          }
        }
        tc_commit(&bars->slot_empty[c % Cfg::kKVSlots]);
        if (c + 1 < nblk) issue_dpt(c + 1);
      }
      tc_commit(&bars->final_);
    }
  } else {
    // ===================== elementwise warps: thread = key row
    const int r = threadIdx.x;  // 0..127
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const int kv = kv0 + r;
    const float* lse_g = p.lse + static_cast<int64_t>(b * p.H + h) * p.N;
    const float* dl_g = p.delta + static_cast<int64_t>(b * p.H + h) * p.N;
    for (int c = 0; c < nblk; ++c) {
      const int q0 = (i_start + c) * 64;
      float* st = s_stats + (c & 1) * 128;  // [lse*log2e (64) | delta (64)]
      {
        const int qq = r & 63;
        const int q = q0 + qq;
        if (r < 64) st[qq] = q < p.N ? lse_g[q] * kLog2e : INFINITY;
        else st[64 + qq] = q < p.N ? dl_g[q] : 0.f;
      }
      named_bar_sync(1, 128);
      float pr[64];
      mbar_wait(&bars->s_full[0], c & 1);
      tc_fence_after();
      {
        uint32_t u[64];
        tmem_ld32(tmem + lane_off + T_ST, *reinterpret_cast<uint32_t(*)[32]>(u));
        tmem_ld32(tmem + lane_off + T_ST + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
        tmem_wait_ld();
#pragma unroll
        for (int qq = 0; qq < 64; ++qq) pr[qq] = __uint_as_float(u[qq]) * p.scale_log2;
      }
      if constexpr (DENSE) {
        mbar_wait(&bars->slot_full[c % Cfg::kKVSlots], (c / Cfg::kKVSlots) & 1);
        const uint8_t* bt = smem + Cfg::kKVRes + (c % Cfg::kKVSlots) * Cfg::kKVSlot + 2 * Cfg::kTile64;
        const int half = r >> 6, cc = r & 63;
#pragma unroll
        for (int qq = 0; qq < 64; ++qq) {
          const uint16_t raw = *reinterpret_cast<const uint16_t*>(
              bt + half * 64 * 128 + qq * 128 + ((((cc >> 3) ^ (qq & 7))) << 4) + (cc & 7) * 2);
          float bv;
          if constexpr (BF16) bv = __bfloat162float(__ushort_as_bfloat16(raw));
          else bv = __half2float(__ushort_as_half(raw));
          pr[qq] = fmaf(bv, kLog2e, pr[qq]);
        }
      }
      const bool edge = p.causal ? (q0 < kv0 + 128) : false;
#pragma unroll
      for (int qq = 0; qq < 64; ++qq) {
        float x = pr[qq] - st[qq];
        if (edge && kv > q0 + qq) x = -INFINITY;
        pr[qq] = ex2(x);
      }
      {
        uint32_t pk[32];
#pragma unroll
        for (int c2 = 0; c2 < 32; ++c2) pk[c2] = pack2<BF16>(pr[2 * c2], pr[2 * c2 + 1]);
        tmem_st32(tmem + lane_off + T_ST, pk);
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_ready);
      mbar_wait(&bars->dp_full[0], c & 1);
      tc_fence_after();
      {
        uint32_t u[64];
        tmem_ld32(tmem + lane_off + T_DPT, *reinterpret_cast<uint32_t(*)[32]>(u));
        tmem_ld32(tmem + lane_off + T_DPT + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
        tmem_wait_ld();
        uint32_t pk[32];
#pragma unroll
        for (int c2 = 0; c2 < 32; ++c2) {
          const float d0 = pr[2 * c2] * (__uint_as_float(u[2 * c2]) - st[64 + 2 * c2]);
          const float d1 = pr[2 * c2 + 1] * (__uint_as_float(u[2 * c2 + 1]) - st[64 + 2 * c2 + 1]);
          pk[c2] = pack2<BF16>(d0, d1);
        }
        tmem_st32(tmem + lane_off + T_DPT, pk);
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->ds_ready[0]);
    }
    // ---- epilogue
    mbar_wait(&bars->final_, 0);
    tc_fence_after();
    const bool valid = kv < p.M;
    typedef typename std::conditional<BF16, __nv_bfloat16, __half>::type elem_t;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + T_DV + c0, v);
      tmem_wait_ld();
      if (valid) store_row32<BF16>(row_ptr<elem_t>(p.dv, p.dv_sb, p.dv_sh, p.dv_sn, b, h, kv) + c0, v, 1.0f);
      tmem_ld32(tmem + lane_off + T_DK + c0, v);
      tmem_wait_ld();
      if (valid) store_row32<BF16>(row_ptr<elem_t>(p.dk, p.dk_sb, p.dk_sh, p.dk_sn, b, h, kv) + c0, v, p.scale);
    }
    if constexpr (FGRAD) {
#pragma unroll
      for (int pn = 0; pn < RP; ++pn) {
        uint32_t v[16];
        tmem_ld16(tmem + lane_off + T_DUK + pn * 16, v);
        tmem_wait_ld();
        if (valid) {
          float* dst = row_ptr<float>(p.duk, p.duk_sb, p.duk_sh, p.duk_sn, b, h, kv) + pn * 16;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            reinterpret_cast<float4*>(dst)[q4] =
                make_float4(__uint_as_float(v[4 * q4]) * p.scale, __uint_as_float(v[4 * q4 + 1]) * p.scale,
                            __uint_as_float(v[4 * q4 + 2]) * p.scale, __uint_as_float(v[4 * q4 + 3]) * p.scale);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// =====================================================================================
// dQ' kernel (Q-stationary)
// =====================================================================================
template <int D, int RP, bool DENSE, bool BF16, bool FGRAD>
__global__ void __launch_bounds__(192, 1)
    fb_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                     const __grid_constant__ CUtensorMap tm_uq, const __grid_constant__ CUtensorMap tm_bias,
                     const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const __grid_constant__ CUtensorMap tm_uk, const BwdParams p) {
  using Cfg = BwdCfg<D, RP, DENSE>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t q_base = sbase;
  const uint32_t do_base = sbase + Cfg::kTile128;
  const uint32_t uq_base = sbase + 2 * Cfg::kTile128;
  const uint32_t ring_base = sbase + Cfg::kQRes;
  BwdBars* bars = reinterpret_cast<BwdBars*>(smem + Cfg::kQRes + Cfg::kQSlots * Cfg::kQSlot);

  const int warp = warp_id(), lane = lane_id();
  const int nqt = (p.N + 127) / 128;
  int qt = blockIdx.x % nqt;
  if (p.causal) qt = nqt - 1 - qt;  // longest first within a head
  const int bh = blockIdx.x / nqt;  // head-major: resident CTAs share K/V via L2
  const int h = bh / p.B, b = bh % p.B;  // a head's batches adjacent (shared bias/L2)
  const int q0 = qt * 128;
  const int nkb_all = (p.M + 63) / 64;
  const int nkb = p.causal ? min(nkb_all, (q0 + 127) / 64 + 1) : nkb_all;

  if (warp == 4 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    if (RP > 0) {
      tma_prefetch(&tm_uq);
      tma_prefetch(&tm_uk);
    }
    if (DENSE) tma_prefetch(&tm_bias);
    mbar_init(&bars->res_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->dp_full[i], 1);
      mbar_init(&bars->ds_ready[i], 4);
    }
    mbar_init(&bars->final_, 1);
    for (int s = 0; s < Cfg::kQSlots; ++s) {
      mbar_init(&bars->slot_full[s], 1);
      mbar_init(&bars->slot_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<Cfg::kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  constexpr uint32_t T_DQ = 256, T_DUQ = 256 + D;

  if (warp == 4) {
    if (lane == 0) {
      const int hq = p.uq_hb ? 0 : h, bq = p.uq_bb ? 0 : b;
      const int hk = p.uk_hb ? 0 : h, bk = p.uk_bb ? 0 : b;
      const int hb_ = p.bias_hb ? 0 : h, bb_ = p.bias_bb ? 0 : b;
      mbar_arrive_expect_tx(&bars->res_full, Cfg::kQRes);
      for (int a = 0; a < Cfg::kAtoms; ++a) {
        tma_load_4d(smem + a * 128 * Cfg::kSW, &tm_q, &bars->res_full, a * Cfg::kAtomCols, q0, h, b);
        tma_load_4d(smem + Cfg::kTile128 + a * 128 * Cfg::kSW, &tm_do, &bars->res_full, a * Cfg::kAtomCols, q0, h, b);
      }
      for (int pn = 0; pn < RP; ++pn)
        tma_load_4d(smem + 2 * Cfg::kTile128 + pn * Cfg::kPanel128, &tm_uq, &bars->res_full, pn * 16, q0, hq, bq);
      for (int j = 0; j < nkb; ++j) {
        const int k0 = j * 64;
        const int slot = j % Cfg::kQSlots, use = j / Cfg::kQSlots;
        if (use > 0) mbar_wait(&bars->slot_empty[slot], (use - 1) & 1);
        uint8_t* dst = smem + Cfg::kQRes + slot * Cfg::kQSlot;
        uint64_t* fb_ = &bars->slot_full[slot];
        mbar_arrive_expect_tx(fb_, Cfg::kQItem);
        for (int a = 0; a < Cfg::kAtoms; ++a) {
          tma_load_4d(dst + a * 64 * Cfg::kSW, &tm_k, fb_, a * Cfg::kAtomCols, k0, h, b);
          tma_load_4d(dst + Cfg::kTile64 + a * 64 * Cfg::kSW, &tm_v, fb_, a * Cfg::kAtomCols, k0, h, b);
        }
        for (int pn = 0; pn < RP; ++pn)
          tma_load_4d(dst + 2 * Cfg::kTile64 + pn * Cfg::kPanel64, &tm_uk, fb_, pn * 16, k0, hk, bk);
        if (DENSE) tma_load_4d(dst + 2 * Cfg::kTile64, &tm_bias, fb_, k0, q0, hb_, bb_);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t id_s = make_idesc(128, 64, false, false, BF16);
      constexpr uint32_t id_d = make_idesc(128, D, false, true, BF16);
      constexpr uint32_t id_u = make_idesc(128, 16, false, true, BF16);
      auto slot_addr = [&](int j) { return ring_base + (j % Cfg::kQSlots) * Cfg::kQSlot; };
      auto wait_slot = [&](int j) { mbar_wait(&bars->slot_full[j % Cfg::kQSlots], (j / Cfg::kQSlots) & 1); };
      auto issue_sdp = [&](int j) {
        const int buf = j & 1;
        const uint32_t kb = slot_addr(j), vb = kb + Cfg::kTile64;
        const uint32_t t_s = tmem + buf * 128, t_dp = tmem + buf * 128 + 64;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(t_s, kmajor_desc(q_base, 128, Cfg::kSW, kk * 16), kmajor_desc(kb, 64, Cfg::kSW, kk * 16), id_s,
                 kk > 0 ? 1u : 0u);
#pragma unroll
        for (int pn = 0; pn < RP; ++pn)
          mma_ss(t_s, make_sdesc(uq_base + pn * Cfg::kPanel128, 16, 256, 6),
                 make_sdesc(kb + 2 * Cfg::kTile64 + pn * Cfg::kPanel64, 16, 256, 6), id_s, 1u);
        tc_commit(&bars->s_full[buf]);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(t_dp, kmajor_desc(do_base, 128, Cfg::kSW, kk * 16), kmajor_desc(vb, 64, Cfg::kSW, kk * 16), id_s,
                 kk > 0 ? 1u : 0u);
        tc_commit(&bars->dp_full[buf]);
      };
      mbar_wait(&bars->res_full, 0);
      for (int j = 0; j < nkb && j < 2; ++j) {
        wait_slot(j);
        tc_fence_after();
        issue_sdp(j);
      }
      for (int j = 0; j < nkb; ++j) {
        const int buf = j & 1;
        const uint32_t kb = slot_addr(j);
        mbar_wait(&bars->ds_ready[buf], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t a_ds = tmem + buf * 128;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          mma_ts(tmem + T_DQ, a_ds + kk * 8, mnmajor_desc(kb, 64, Cfg::kSW, kk * 16), id_d, (j > 0 || kk > 0) ? 1u : 0u);
          if constexpr (FGRAD) {
#pragma unroll
            for (int pn = 0; pn < RP; ++pn)
              mma_ts(tmem + T_DUQ + pn * 16, a_ds + kk * 8,
                     make_sdesc(kb + 2 * Cfg::kTile64 + pn * Cfg::kPanel64 + kk * 16 * 32, 64 * 32, 256, 6), id_u,
                     (j > 0 || kk > 0) ? 1u : 0u);
          }
        }
        tc_commit(&bars->slot_empty[j % Cfg::kQSlots]);
        if (j + 2 < nkb) {
          wait_slot(j + 2);
          tc_fence_after();
          issue_sdp(j + 2);
        }
      }
      tc_commit(&bars->final_);
    }
  } else {
    const int r = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const int row = q0 + r;
    const bool valid = row < p.N;
    const float lse2 = valid ? p.lse[static_cast<int64_t>(b * p.H + h) * p.N + row] * kLog2e : INFINITY;
    const float dlt = valid ? p.delta[static_cast<int64_t>(b * p.H + h) * p.N + row] : 0.f;
    for (int j = 0; j < nkb; ++j) {
      const int buf = j & 1;
      const int k0 = j * 64;
      const uint32_t t_s = tmem + lane_off + buf * 128, t_dp = t_s + 64;
      float pr[64];
      mbar_wait(&bars->s_full[buf], (j >> 1) & 1);
      tc_fence_after();
      {
        uint32_t u[64];
        tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(u));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 64; ++c) pr[c] = fmaf(__uint_as_float(u[c]), p.scale_log2, -lse2);
      }
      if constexpr (DENSE) {
        mbar_wait(&bars->slot_full[j % Cfg::kQSlots], (j / Cfg::kQSlots) & 1);
        const uint8_t* bt = smem + Cfg::kQRes + (j % Cfg::kQSlots) * Cfg::kQSlot + 2 * Cfg::kTile64;
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const uint4 v = *reinterpret_cast<const uint4*>(bt + r * 128 + ((c8 ^ (r & 7)) << 4));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 bb = unpack2<BF16>(w[e]);
            pr[c8 * 8 + 2 * e] = fmaf(bb.x, kLog2e, pr[c8 * 8 + 2 * e]);
            pr[c8 * 8 + 2 * e + 1] = fmaf(bb.y, kLog2e, pr[c8 * 8 + 2 * e + 1]);
          }
        }
      }
      const bool edge = (k0 + 64 > p.M) || (p.causal && k0 + 64 > q0);
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        float x = pr[c];
        if (edge && (k0 + c >= p.M || (p.causal && k0 + c > row))) x = -INFINITY;
        pr[c] = ex2(x);
      }
      mbar_wait(&bars->dp_full[buf], (j >> 1) & 1);
      tc_fence_after();
      {
        uint32_t u[64];
        tmem_ld32(t_dp, *reinterpret_cast<uint32_t(*)[32]>(u));
        tmem_ld32(t_dp + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
        tmem_wait_ld();
        uint32_t pk[32];
#pragma unroll
        for (int c2 = 0; c2 < 32; ++c2)
          pk[c2] = pack2<BF16>(pr[2 * c2] * (__uint_as_float(u[2 * c2]) - dlt),
                               pr[2 * c2 + 1] * (__uint_as_float(u[2 * c2 + 1]) - dlt));
        tmem_st32(t_s, pk);
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->ds_ready[buf]);
    }
    mbar_wait(&bars->final_, 0);
    tc_fence_after();
    typedef typename std::conditional<BF16, __nv_bfloat16, __half>::type elem_t;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + T_DQ + c0, v);
      tmem_wait_ld();
      if (valid) store_row32<BF16>(row_ptr<elem_t>(p.dq, p.dq_sb, p.dq_sh, p.dq_sn, b, h, row) + c0, v, p.scale);
    }
    if constexpr (FGRAD) {
#pragma unroll
      for (int pn = 0; pn < RP; ++pn) {
        uint32_t v[16];
        tmem_ld16(tmem + lane_off + T_DUQ + pn * 16, v);
        tmem_wait_ld();
        if (valid) {
          float* dst = row_ptr<float>(p.duq, p.duq_sb, p.duq_sh, p.duq_sn, b, h, row) + pn * 16;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            reinterpret_cast<float4*>(dst)[q4] =
                make_float4(__uint_as_float(v[4 * q4]) * p.scale, __uint_as_float(v[4 * q4 + 1]) * p.scale,
                            __uint_as_float(v[4 * q4 + 2]) * p.scale, __uint_as_float(v[4 * q4 + 3]) * p.scale);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// ------------------------------------------------------------------ launch
template <int D, int RP, bool DENSE, bool BF16, bool FGRAD>
static cudaError_t launch_bwd_t(const BwdMaps& m, const BwdParams& p, cudaStream_t s) {
  using Cfg = BwdCfg<D, RP, DENSE>;
  auto kdkv = fb_bwd_dkv_kernel<D, RP, DENSE, BF16, FGRAD>;
  auto kdq = fb_bwd_dq_kernel<D, RP, DENSE, BF16, FGRAD>;
  static std::atomic<uint64_t> attr_kv{0}, attr_q{0};
  {
    cudaError_t e = smem_attr_once(attr_kv, reinterpret_cast<const void*>(kdkv), Cfg::kKVSmem);
    if (e != cudaSuccess) return e;
    e = smem_attr_once(attr_q, reinterpret_cast<const void*>(kdq), Cfg::kQSmem);
    if (e != cudaSuccess) return e;
  }
  const int bhc = p.B * p.H;
  kdkv<<<((p.M + 127) / 128) * bhc, Cfg::kThreads, Cfg::kKVSmem, s>>>(m.q64, m.do64, m.uq64, m.biasT, m.k128, m.v128,
                                                                       m.uk128, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  kdq<<<((p.N + 127) / 128) * bhc, Cfg::kThreads, Cfg::kQSmem, s>>>(m.q128, m.do128, m.uq128, m.bias, m.k64, m.v64,
                                                                     m.uk64, p);
  return cudaGetLastError();
}

template <int D, bool BF16>
static cudaError_t bwd_rp(int rp, bool dense, bool fgrad, const BwdMaps& m, const BwdParams& p, cudaStream_t s) {
  if (dense) return rp == 0 ? launch_bwd_t<D, 0, true, BF16, false>(m, p, s) : cudaErrorInvalidValue;
  if (rp == 0) return launch_bwd_t<D, 0, false, BF16, false>(m, p, s);
  if (fgrad) {
    switch (rp) {
      case 1: return launch_bwd_t<D, 1, false, BF16, true>(m, p, s);
      case 2: return launch_bwd_t<D, 2, false, BF16, true>(m, p, s);
      case 3: return launch_bwd_t<D, 3, false, BF16, true>(m, p, s);
      case 4: return launch_bwd_t<D, 4, false, BF16, true>(m, p, s);
    }
    if constexpr (D <= 64) {
      switch (rp) {
        case 5: return launch_bwd_t<D, 5, false, BF16, true>(m, p, s);
        case 6: return launch_bwd_t<D, 6, false, BF16, true>(m, p, s);
        case 7: return launch_bwd_t<D, 7, false, BF16, true>(m, p, s);
        case 8: return launch_bwd_t<D, 8, false, BF16, true>(m, p, s);
      }
    }
  } else {
    switch (rp) {
      case 1: return launch_bwd_t<D, 1, false, BF16, false>(m, p, s);
      case 2: return launch_bwd_t<D, 2, false, BF16, false>(m, p, s);
      case 3: return launch_bwd_t<D, 3, false, BF16, false>(m, p, s);
      case 4: return launch_bwd_t<D, 4, false, BF16, false>(m, p, s);
    }
    if constexpr (D <= 64) {
      switch (rp) {
        case 5: return launch_bwd_t<D, 5, false, BF16, false>(m, p, s);
        case 6: return launch_bwd_t<D, 6, false, BF16, false>(m, p, s);
        case 7: return launch_bwd_t<D, 7, false, BF16, false>(m, p, s);
        case 8: return launch_bwd_t<D, 8, false, BF16, false>(m, p, s);
      }
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwd_sm100(int d, int rp, bool dense, bool bf16, bool fgrad, const BwdMaps& m,
                             const BwdParams& p, cudaStream_t s) {
  if (bf16) {
    if (d == 32) return bwd_rp<32, true>(rp, dense, fgrad, m, p, s);
    if (d == 64) return bwd_rp<64, true>(rp, dense, fgrad, m, p, s);
    if (d == 128) return bwd_rp<128, true>(rp, dense, fgrad, m, p, s);
  } else {
    if (d == 32) return bwd_rp<32, false>(rp, dense, fgrad, m, p, s);
    if (d == 64) return bwd_rp<64, false>(rp, dense, fgrad, m, p, s);
    if (d == 128) return bwd_rp<128, false>(rp, dense, fgrad, m, p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace fb
