// fb_bwd_fused_sm100.cu — single-pass FlashBias backward for head dim 128
// (K2 fused / K4 fused): the 5-GEMM backward with dQ reduced through L2.
//
// Same math as fb_bwd_sm100.cu (oracle/flashbias_oracle.py:attention_bwd):
//   S^T = K' Q'^T, P^T = exp(scale S^T - lse), dP^T = V dO^T,
//   dS^T = P^T (dP^T - D), dV += P^T dO, dK += dS^T Q, dQ += scale dS K.
// CTA owns 128 key rows and streams 64-row query blocks c (causal: only the
// blocks at or below the diagonal).  dQ is produced transposed on the tensor
// core as dQ^T = K^T dS^T (M = d = 128, N = 64 queries); each 64x128 fp32 dQ
// tile is staged in shared memory and added into an fp32 accumulator in
// global memory with one TMA bulk reduction (cp.reduce.async.bulk.tensor
// .add) — the per-head accumulator (8 MB at N=16k) stays L2-resident under
// head-major scheduling.
//
// Two elementwise warpgroups ping-pong over the query blocks (EW0: even c,
// EW1: odd c) so the softmax-like work of one block overlaps the tensor-core
// work of the other.  TMEM (512 columns):
//   S^T_x [64x, 64x+64)   dP^T_x / dQ^T_x [128+64x, +64)   dV [256,384)   dK [384,512)
// P^T and dS^T (bf16) are written over the first 32 columns of their fp32
// source and consumed from TMEM as the A operand of dV / dK; dQ^T(c) reuses
// the dP^T_x columns once dK(c) has been issued (tcgen05 MMAs run in order).
// MMA order per block c (x = c & 1):
//   dV(c) | dP^T(c+1) | dK(c) dQ^T(c) | S^T(c+2)
//
// Warp roles (512 threads, 4 warpgroups for setmaxnreg):
//   warps 0-3 EW0, 4-7 EW1 (thread = key row = TMEM lane), 8-11 dQ drain
//   (thread = head-dim lane of dQ^T: TMEM -> smem -> TMA reduce), warp 12 TMA
//   producer, warp 13 TMEM alloc + MMA issuer, 14-15 idle.
#include "fb_kernels.h"
#include "fb_sm100.cuh"

namespace fb {

namespace {
constexpr float kLog2eF = 1.4426950408889634f;

__device__ __forceinline__ void tma_reduce_add_4d(const CUtensorMap* map, const void* smem, int c0, int c1, int c2,
                                                  int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
}  // namespace

template <int RP, bool DENSE>
struct FusedCfg {
  static constexpr int D = 128;
  static constexpr int kTile128 = 128 * D * 2;  // 32 KB
  static constexpr int kTile64 = 64 * D * 2;    // 16 KB
  static constexpr int kPanel128 = 128 * 32;
  static constexpr int kPanel64 = 64 * 32;
  static constexpr int kRes = 2 * kTile128 + RP * kPanel128;                             // K, V, Uk
  static constexpr int kItem = 2 * kTile64 + (DENSE ? 64 * 128 * 2 : RP * kPanel64);  // Q, dO, Uq | bias^T
  static constexpr int kSlot = (kItem + 1023) / 1024 * 1024;
  static constexpr int kDsBuf = 128 * 128;     // dS^T [128 keys][64 queries] bf16, SW128
  static constexpr int kDqStage = 32 * D * 4;  // 16 KB fp32: a dQ tile drains in two 32-query halves
  static constexpr int kMisc = 2048 + 512;     // stats [2 groups][2][128] + barriers
  static constexpr int kBudget = 232448 - 1024;
  static constexpr int kSlotsFit = (kBudget - kRes - 2 * kDsBuf - kDqStage - kMisc) / kSlot;
  static constexpr int kSlots = kSlotsFit > 4 ? 4 : kSlotsFit;
  static constexpr int kSmem = 1024 + kRes + kSlots * kSlot + 2 * kDsBuf + kDqStage + kMisc;
  static_assert(kSlots >= 2, "fused bwd ring too small");
};

struct FusedBars {
  uint64_t res_full, final_[2];
  uint64_t st_full[2], dpt_full[2], p_ready[2], ds_ready[2];
  uint64_t dq_full[2], dq_free[2], dsbuf_free[2];
  uint64_t slot_full[4], slot_empty[4];
  uint32_t tmem_base;
};

template <int RP, bool DENSE, bool BF16>
__global__ void __launch_bounds__(512, 1)
    fb_bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_uq, const __grid_constant__ CUtensorMap tm_biasT,
                        const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_uk, const __grid_constant__ CUtensorMap tm_dqacc,
                        const BwdParams p) {
  using Cfg = FusedCfg<RP, DENSE>;
  constexpr int D = 128;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t k_base = sbase, v_base = sbase + Cfg::kTile128, uk_base = sbase + 2 * Cfg::kTile128;
  const uint32_t ring_base = sbase + Cfg::kRes;
  uint8_t* ds_buf = smem + Cfg::kRes + Cfg::kSlots * Cfg::kSlot;  // 2 x 16 KB
  float* dq_stage = reinterpret_cast<float*>(ds_buf + 2 * Cfg::kDsBuf);
  float* s_stats = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(dq_stage) + Cfg::kDqStage);  // [2][2][128]
  FusedBars* bars = reinterpret_cast<FusedBars*>(reinterpret_cast<uint8_t*>(s_stats) + 2048);

  const int warp = warp_id(), lane = lane_id();
  const int nkt = (p.M + 127) / 128;
  const int kt = blockIdx.x % nkt;
  const int bh = blockIdx.x / nkt;
  const int h = bh / p.B, b = bh % p.B;
  const int kv0 = kt * 128;
  const int nqb = (p.N + 63) / 64;
  const int i_start = p.causal ? kv0 / 64 : 0;
  const int nblk = nqb - i_start;

  if (warp == 12 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_dqacc);
    if (RP > 0) {
      tma_prefetch(&tm_uq);
      tma_prefetch(&tm_uk);
    }
    if (DENSE) tma_prefetch(&tm_biasT);
    mbar_init(&bars->res_full, 1);
    mbar_init(&bars->final_[0], 1);
    mbar_init(&bars->final_[1], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->st_full[i], 1);
      mbar_init(&bars->dpt_full[i], 1);
      mbar_init(&bars->p_ready[i], 4);
      mbar_init(&bars->ds_ready[i], 4);
      mbar_init(&bars->dq_full[i], 1);
      mbar_init(&bars->dq_free[i], 4);
      mbar_init(&bars->dsbuf_free[i], 1);
    }
    for (int s = 0; s < Cfg::kSlots; ++s) {
      mbar_init(&bars->slot_full[s], 1);
      mbar_init(&bars->slot_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 13) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  constexpr uint32_t T_ST = 0, T_DPT = 128, T_DV = 256, T_DK = 384;

  if (warp >= 12) {
    regs_dec<96>();
    if (warp == 12 && lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const int hq = p.uq_hb ? 0 : h, bq = p.uq_bb ? 0 : b;
      const int hk = p.uk_hb ? 0 : h, bk = p.uk_bb ? 0 : b;
      const int hb_ = p.bias_hb ? 0 : h, bb_ = p.bias_bb ? 0 : b;
      mbar_arrive_expect_tx(&bars->res_full, Cfg::kRes);
      for (int a = 0; a < 2; ++a) {
        tma_load_4d(smem + a * 128 * 128, &tm_k, &bars->res_full, a * 64, kv0, h, b);
        tma_load_4d(smem + Cfg::kTile128 + a * 128 * 128, &tm_v, &bars->res_full, a * 64, kv0, h, b);
      }
      for (int pn = 0; pn < RP; ++pn)
        tma_load_4d(smem + 2 * Cfg::kTile128 + pn * Cfg::kPanel128, &tm_uk, &bars->res_full, pn * 16, kv0, hk, bk);
      for (int c = 0; c < nblk; ++c) {
        const int q0 = (i_start + c) * 64;
        const int slot = c % Cfg::kSlots, use = c / Cfg::kSlots;
        if (use > 0) mbar_wait(&bars->slot_empty[slot], (use - 1) & 1);
        trace(p.trace, p.trace_cta, 21, c);
        uint8_t* dst = smem + Cfg::kRes + slot * Cfg::kSlot;
        uint64_t* fb_ = &bars->slot_full[slot];
        mbar_arrive_expect_tx(fb_, Cfg::kItem);
        for (int a = 0; a < 2; ++a) {
          tma_load_4d(dst + a * 64 * 128, &tm_q, fb_, a * 64, q0, h, b);
          tma_load_4d(dst + Cfg::kTile64 + a * 64 * 128, &tm_do, fb_, a * 64, q0, h, b);
        }
        if (DENSE) {
          for (int half = 0; half < 2; ++half)
            tma_load_4d(dst + 2 * Cfg::kTile64 + half * 64 * 128, &tm_biasT, fb_, kv0 + half * 64, q0, hb_, bb_);
        } else {
          for (int pn = 0; pn < RP; ++pn)
            tma_load_4d(dst + 2 * Cfg::kTile64 + pn * Cfg::kPanel64, &tm_uq, fb_, pn * 16, q0, hq, bq);
        }
      }
    } else if ((warp == 13 || warp == 14) && lane == 0) {
      // ------------------------------------------------------------ MMA issuers
      // Two issuing threads, one per elementwise group x: each runs the chain of
      // its own blocks c = x, x+2, ... so a stall on one group never holds back
      // the other's tensor-core work (dV/dK accumulate from both; they are
      // zero-initialised by EW0 and every MMA into them accumulates).
      const int x = warp - 13;
      constexpr uint32_t id_s = make_idesc(128, 64, false, false, BF16);  // S^T, dP^T
      constexpr uint32_t id_d = make_idesc(128, D, false, true, BF16);    // dV, dK (A from TMEM)
      constexpr uint32_t id_q = make_idesc(128, 64, true, true, BF16);    // dQ^T = K^T dS^T
      // loop-invariant descriptors; per-K-step variants are constant adds to the
      // start-address field (addresses < 256 KB, so the 14-bit field never carries)
      const uint64_t dk_k = kmajor_desc(k_base, 128, 128, 0);   // K as A (K-major)
      const uint64_t dk_v = kmajor_desc(v_base, 128, 128, 0);   // V as A (K-major)
      const uint64_t dk_kt = mnmajor_desc(k_base, 128, 128, 0); // K^T as A (MN-major)
      const uint64_t dsb = mnmajor_desc(smem_u32(ds_buf) + x * Cfg::kDsBuf, 128, 128, 0);
      const uint32_t t_st = tmem + T_ST + 64 * x, t_dpt = tmem + T_DPT + 64 * x;
      auto slot_addr = [&](int c) { return ring_base + (c % Cfg::kSlots) * Cfg::kSlot; };
      auto kstep = [](int kk) -> uint64_t { return (kk >> 2) * (64 * 128 >> 4) + (kk & 3) * 2; };  // 64-row tile
      auto kstep128 = [](int kk) -> uint64_t { return (kk >> 2) * (128 * 128 >> 4) + (kk & 3) * 2; };
      auto wait_slot = [&](int c) {
        mbar_wait(&bars->slot_full[c % Cfg::kSlots], (c / Cfg::kSlots) & 1);
        tc_fence_after();
      };
      auto issue_st = [&](int c) {
        const uint32_t qb = slot_addr(c);
        const uint64_t dq = kmajor_desc(qb, 64, 128, 0);
        trace(p.trace, p.trace_cta, 11, c);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(t_st, dk_k + kstep128(kk), dq + kstep(kk), id_s, kk > 0 ? 1u : 0u);
        if constexpr (!DENSE) {
#pragma unroll
          for (int pn = 0; pn < RP; ++pn)
            mma_ss(t_st, make_sdesc(uk_base + pn * Cfg::kPanel128, 16, 256, 6),
                   make_sdesc(qb + 2 * Cfg::kTile64 + pn * Cfg::kPanel64, 16, 256, 6), id_s, 1u);
        }
        tc_commit(&bars->st_full[x]);
      };
      auto issue_dpt = [&](int c) {
        // dP^T_x last held dQ^T(c-2): wait for its drain
        if (c >= 2) mbar_wait(&bars->dq_free[x], ((c >> 1) - 1) & 1);
        tc_fence_after();
        trace(p.trace, p.trace_cta, 14, c);
        const uint64_t ddo = kmajor_desc(slot_addr(c) + Cfg::kTile64, 64, 128, 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(t_dpt, dk_v + kstep128(kk), ddo + kstep(kk), id_s, kk > 0 ? 1u : 0u);
        tc_commit(&bars->dpt_full[x]);
      };
      mbar_wait(&bars->res_full, 0);
      if (x < nblk) {
        wait_slot(x);
        issue_st(x);
        issue_dpt(x);
      }
      for (int c = x; c < nblk; c += 2) {
        const int u = c >> 1;
        const uint32_t qb = slot_addr(c);
        const uint64_t mq = mnmajor_desc(qb, 64, 128, 0), mdo = mnmajor_desc(qb + Cfg::kTile64, 64, 128, 0);
        mbar_wait(&bars->p_ready[x], u & 1);
        tc_fence_after();
        trace(p.trace, p.trace_cta, 10, c);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dV += P^T dO  (K = 64 queries)
          mma_ts(tmem + T_DV, t_st + kk * 8, mdo + kk * (16 * 128 >> 4), id_d, 1u);
        mbar_wait(&bars->ds_ready[x], u & 1);
        tc_fence_after();
        trace(p.trace, p.trace_cta, 12, c);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dK += dS^T Q
          mma_ts(tmem + T_DK, t_dpt + kk * 8, mq + kk * (16 * 128 >> 4), id_d, 1u);
        trace(p.trace, p.trace_cta, 13, c);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ^T = K^T dS^T (K = 128 keys), into the dP^T_x columns
          mma_ss(t_dpt, dk_kt + kk * (16 * 128 >> 4), dsb + kk * (16 * 128 >> 4), id_q, kk > 0 ? 1u : 0u);
        tc_commit(&bars->dq_full[x]);
        tc_commit(&bars->dsbuf_free[x]);
        tc_commit(&bars->slot_empty[c % Cfg::kSlots]);
        if (c + 2 < nblk) {
          wait_slot(c + 2);
          issue_st(c + 2);
          issue_dpt(c + 2);
        }
      }
      tc_commit(&bars->final_[x]);
    }
  } else if (warp < 8) {
    regs_inc<160>();
    // -------------------------------------------------------------- elementwise (thread = key row)
    const int g = warp >> 2;          // EW group: blocks c with c % 2 == g
    const int r = threadIdx.x & 127;  // key row within the tile == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_st = tmem + lane_off + T_ST + 64 * g;
    const uint32_t t_dpt = tmem + lane_off + T_DPT + 64 * g;
    const int kv = kv0 + r;
    const float* lse_g = p.lse + static_cast<int64_t>(b * p.H + h) * p.N;
    const float* dl_g = p.delta + static_cast<int64_t>(b * p.H + h) * p.N;
    {  // zero the dV / dK accumulators (every MMA into them accumulates); each group clears one
      uint32_t z[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) z[i] = 0u;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) tmem_st32(tmem + lane_off + (g == 0 ? T_DV : T_DK) + c0, z);
      tmem_wait_st();
      tc_fence_before();
    }
    named_bar_sync(4, 256);  // both accumulators cleared before any EW arrival (MMAs wait on those)
    tc_fence_after();
    for (int c = g; c < nblk; c += 2) {
      const int u = c >> 1;
      const int q0 = (i_start + c) * 64;
      float* st = s_stats + (g * 2 + (u & 1)) * 128;
      {
        const int qq = r & 63, q = q0 + qq;
        if (r < 64) st[qq] = q < p.N ? lse_g[q] * kLog2eF : INFINITY;
        else st[64 + qq] = q < p.N ? dl_g[q] : 0.f;
      }
      named_bar_sync(1 + g, 128);
      float pr[64];
      mbar_wait(&bars->st_full[g], u & 1);
      tc_fence_after();
      if (r == 0) trace(p.trace, p.trace_cta, 15, c);
      {
        uint32_t v[64];
        tmem_ld32(t_st, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32(t_st + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_wait_ld();
        const float2 mul = make_float2(p.scale_log2, p.scale_log2);
#pragma unroll
        for (int qq = 0; qq < 64; qq += 2) {
          const float2 r2 = ffma2(make_float2(__uint_as_float(v[qq]), __uint_as_float(v[qq + 1])), mul,
                                  make_float2(-st[qq], -st[qq + 1]));
          pr[qq] = r2.x;
          pr[qq + 1] = r2.y;
        }
      }
      if constexpr (DENSE) {
        mbar_wait(&bars->slot_full[c % Cfg::kSlots], (c / Cfg::kSlots) & 1);
        const uint8_t* bt = smem + Cfg::kRes + (c % Cfg::kSlots) * Cfg::kSlot + 2 * Cfg::kTile64;
        const int half = r >> 6, cc = r & 63;
#pragma unroll
        for (int qq = 0; qq < 64; ++qq) {
          const uint16_t raw = *reinterpret_cast<const uint16_t*>(bt + half * 64 * 128 + qq * 128 +
                                                                  (((cc >> 3) ^ (qq & 7)) << 4) + (cc & 7) * 2);
          float bv;
          if constexpr (BF16) bv = __bfloat162float(__ushort_as_bfloat16(raw));
          else bv = __half2float(__ushort_as_half(raw));
          pr[qq] = fmaf(bv, kLog2eF, pr[qq]);
        }
      }
      if (p.causal && (q0 < kv0 + 128)) {
#pragma unroll
        for (int qq = 0; qq < 64; ++qq)
          if (kv > q0 + qq) pr[qq] = -INFINITY;
      }
      {
        uint32_t pk[32];
#pragma unroll
        for (int c2 = 0; c2 < 32; ++c2) {
          if (poly_pair(c2)) {  // FB_POLY_NUM pairs in 8 on the FMA pipe (ex2_poly2), the rest on MUFU
            const float2 e2 = ex2_poly2(make_float2(pr[2 * c2], pr[2 * c2 + 1]));
            pr[2 * c2] = e2.x;
            pr[2 * c2 + 1] = e2.y;
          } else {
            pr[2 * c2] = ex2(pr[2 * c2]);
            pr[2 * c2 + 1] = ex2(pr[2 * c2 + 1]);
          }
          pk[c2] = pack2<BF16>(pr[2 * c2], pr[2 * c2 + 1]);
        }
        tmem_st32(t_st, pk);
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (r == 0) trace(p.trace, p.trace_cta, 16, c);
      if (lane == 0) mbar_arrive(&bars->p_ready[g]);
      mbar_wait(&bars->dpt_full[g], u & 1);
      tc_fence_after();
      if (r == 0) trace(p.trace, p.trace_cta, 17, c);
      uint32_t pk[32];
      {
        uint32_t v[64];
        tmem_ld32(t_dpt, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32(t_dpt + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_wait_ld();
#pragma unroll
        for (int c2 = 0; c2 < 32; ++c2) {
          const float2 dpd = fadd2(make_float2(__uint_as_float(v[2 * c2]), __uint_as_float(v[2 * c2 + 1])),
                                   make_float2(-st[64 + 2 * c2], -st[64 + 2 * c2 + 1]));
          const float2 ds = fmul2(make_float2(pr[2 * c2], pr[2 * c2 + 1]), dpd);
          pk[c2] = pack2<BF16>(ds.x, ds.y);
        }
      }
      if constexpr (DENSE) {
        if (p.dbias != nullptr) store_dbias_rows(p, b, h, q0, kv, lane, pk);
      }
      tmem_st32(t_dpt, pk);
      // dS^T row -> shared memory (B operand of dQ^T), SW128 MN-major: 16-byte
      // chunk ch of row r lives at chunk ch ^ (r & 7)
      if (u >= 1) mbar_wait(&bars->dsbuf_free[g], (u - 1) & 1);
      uint8_t* row = ds_buf + g * Cfg::kDsBuf + r * 128;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *reinterpret_cast<uint4*>(row + ((ch ^ (r & 7)) << 4)) =
            make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      fence_proxy_async();
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (r == 0) trace(p.trace, p.trace_cta, 18, c);
      if (lane == 0) mbar_arrive(&bars->ds_ready[g]);
    }
    if (g == 0) {
      // ---- epilogue (EW0): dV, dK rows, after both issuers' last MMAs
      mbar_wait(&bars->final_[0], 0);
      mbar_wait(&bars->final_[1], 0);
      tc_fence_after();
      const bool valid = kv < p.M;
      typedef typename std::conditional<BF16, __nv_bfloat16, __half>::type elem_t;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + T_DV + c0, v);
        tmem_wait_ld();
        if (valid) {
          elem_t* dst = reinterpret_cast<elem_t*>(p.dv) + static_cast<int64_t>(b) * p.dv_sb +
                        static_cast<int64_t>(h) * p.dv_sh + static_cast<int64_t>(kv) * p.dv_sn + c0;
          uint32_t o16[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) o16[c] = pack2<BF16>(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1]));
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            reinterpret_cast<uint4*>(dst)[q4] = make_uint4(o16[4 * q4], o16[4 * q4 + 1], o16[4 * q4 + 2], o16[4 * q4 + 3]);
        }
        tmem_ld32(tmem + lane_off + T_DK + c0, v);
        tmem_wait_ld();
        if (valid) {
          elem_t* dst = reinterpret_cast<elem_t*>(p.dk) + static_cast<int64_t>(b) * p.dk_sb +
                        static_cast<int64_t>(h) * p.dk_sh + static_cast<int64_t>(kv) * p.dk_sn + c0;
          uint32_t o16[16];
#pragma unroll
          for (int c = 0; c < 16; ++c)
            o16[c] = pack2<BF16>(__uint_as_float(v[2 * c]) * p.scale, __uint_as_float(v[2 * c + 1]) * p.scale);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            reinterpret_cast<uint4*>(dst)[q4] = make_uint4(o16[4 * q4], o16[4 * q4 + 1], o16[4 * q4 + 2], o16[4 * q4 + 3]);
        }
      }
    }
  } else {
    regs_dec<96>();
    // -------------------------------------------------------------- dQ drain (warps 8-11)
    const int dd = threadIdx.x - 256;  // head-dim index = TMEM lane of dQ^T
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const bool leader = dd == 0;
    for (int c = 0; c < nblk; ++c) {
      const int q0 = (i_start + c) * 64;
      const int x = c & 1, u = c >> 1;
      mbar_wait(&bars->dq_full[x], u & 1);
      tc_fence_after();
      if (leader) trace(p.trace, p.trace_cta, 19, c);
      uint32_t v[64];
      tmem_ld32(tmem + lane_off + T_DPT + 64 * x, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32(tmem + lane_off + T_DPT + 64 * x + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->dq_free[x]);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (leader) bulk_wait_read0();  // previous reduction finished reading the stage
        named_bar_sync(3, 128);
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) dq_stage[qq * D + dd] = __uint_as_float(v[32 * half + qq]) * p.scale;
        fence_proxy_async();
        named_bar_sync(3, 128);
        if (leader) {
          tma_reduce_add_4d(&tm_dqacc, dq_stage, 0, q0 + 32 * half, h, b);
          bulk_commit();
        }
      }
      if (leader) trace(p.trace, p.trace_cta, 20, c);
    }
    if (leader) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int RP, bool DENSE, bool BF16>
static cudaError_t launch_fused_t(const BwdMaps& m, const CUtensorMap& dqacc, const BwdParams& p, cudaStream_t s) {
  using Cfg = FusedCfg<RP, DENSE>;
  auto k = fb_bwd_fused_kernel<RP, DENSE, BF16>;
  static std::atomic<uint64_t> attr_mask{0};
  cudaError_t e = smem_attr_once(attr_mask, reinterpret_cast<const void*>(k), Cfg::kSmem);
  if (e != cudaSuccess) return e;
  k<<<((p.M + 127) / 128) * p.B * p.H, 512, Cfg::kSmem, s>>>(m.q64, m.do64, m.uq64, m.biasT, m.k128, m.v128,
                                                             m.uk128, dqacc, p);
  return cudaGetLastError();
}

template <bool BF16>
static cudaError_t fused_rp(int rp, bool dense, const BwdMaps& m, const CUtensorMap& dqacc, const BwdParams& p,
                            cudaStream_t s) {
  if (dense) return rp == 0 ? launch_fused_t<0, true, BF16>(m, dqacc, p, s) : cudaErrorInvalidValue;
  switch (rp) {
    case 0: return launch_fused_t<0, false, BF16>(m, dqacc, p, s);
    case 1: return launch_fused_t<1, false, BF16>(m, dqacc, p, s);
    case 2: return launch_fused_t<2, false, BF16>(m, dqacc, p, s);
    case 3: return launch_fused_t<3, false, BF16>(m, dqacc, p, s);
    case 4: return launch_fused_t<4, false, BF16>(m, dqacc, p, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwd_fused_sm100(int rp, bool dense, bool bf16, const BwdMaps& m, const CUtensorMap& dqacc,
                                   const BwdParams& p, cudaStream_t s) {
  return bf16 ? fused_rp<true>(rp, dense, m, dqacc, p, s) : fused_rp<false>(rp, dense, m, dqacc, p, s);
}

// dq[b,h,n,:] = dq_acc[b,h,n,:] (fp32 [B,H,N,d] -> bf16/f16); the scale is applied in the drain
template <bool BF16>
__global__ void dq_convert_kernel(const float* __restrict__ acc, void* dq, int B, int H, int N, int d, int64_t sb,
                                  int64_t sh, int64_t sn) {
  typedef typename std::conditional<BF16, __nv_bfloat16, __half>::type elem_t;
  const int64_t rows = static_cast<int64_t>(B) * H * N;
  const int per_row = d / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * per_row;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / per_row, c8 = (i % per_row) * 8;
    const int64_t n = row % N, hh = (row / N) % H, bb = row / (static_cast<int64_t>(N) * H);
    const float4 a = reinterpret_cast<const float4*>(acc + row * d + c8)[0];
    const float4 c = reinterpret_cast<const float4*>(acc + row * d + c8)[1];
    elem_t* dst = reinterpret_cast<elem_t*>(dq) + bb * sb + hh * sh + n * sn + c8;
    *reinterpret_cast<uint4*>(dst) =
        make_uint4(pack2<BF16>(a.x, a.y), pack2<BF16>(a.z, a.w), pack2<BF16>(c.x, c.y), pack2<BF16>(c.z, c.w));
  }
}

cudaError_t launch_dq_convert(const float* acc, int d, const BwdParams& p, bool bf16, cudaStream_t s) {
  const int64_t work = static_cast<int64_t>(p.B) * p.H * p.N * (d / 8);
  int64_t g = (work + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (bf16)
    dq_convert_kernel<true><<<static_cast<int>(g), 256, 0, s>>>(acc, p.dq, p.B, p.H, p.N, d, p.dq_sb, p.dq_sh, p.dq_sn);
  else
    dq_convert_kernel<false><<<static_cast<int>(g), 256, 0, s>>>(acc, p.dq, p.B, p.H, p.N, d, p.dq_sb, p.dq_sh, p.dq_sn);
  return cudaGetLastError();
}

}  // namespace fb
