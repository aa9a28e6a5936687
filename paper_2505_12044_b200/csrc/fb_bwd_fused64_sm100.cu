// fb_bwd_fused64_sm100.cu — single-pass FlashBias backward for head dim 64,
// including the factor gradients (learnable biases such as the Swin/PDE
// spatial weights).
//
// For d = 64 the factor panels ride in the SAME 128-byte-swizzled tiles as
// the head dim: K' = [K | Uk | 0] and Q' = [Q | Uq | 0] are two 64-column
// atoms each (the factor atom TMA-loaded from the [., ., L, Rpad] panel
// tensor with OOB zero fill, Rpad <= 64).  Then one MMA set yields
//   dK' = dS^T Q'   -> [dK | dUk]          (N = 128, TMEM [320, 448))
//   dQ'^T = K'^T dS^T -> [dQ^T ; dUq^T]    (M = 128 lanes: d rows 0-63, rank rows 64-127)
// and the drain reduces both halves into fp32 accumulators in global memory
// with TMA bulk reductions.  S^T = K' Q'^T only issues the K-steps that hold
// data (64 + 16 Rpad/16 columns).  Same pipeline otherwise as the d = 128
// kernel (fb_bwd_fused_sm100.cu): two elementwise warpgroups on alternating
// 64-query blocks, two MMA issuers, one drain warpgroup, one TMA producer.
// TMEM: S^T_x [64x,+64) dP^T_x / dQ'^T_x [128+64x,+64) dV [256,320) dK' [320,448)
#include "fb_kernels.h"
#include "fb_sm100.cuh"

namespace fb {

namespace {
constexpr float kLog2e64 = 1.4426950408889634f;

__device__ __forceinline__ void tma_reduce_add_4d_(const CUtensorMap* map, const void* smem, int c0, int c1, int c2,
                                                   int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit_() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0_() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0_() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
}  // namespace

template <int RP, bool DENSE, bool FGRAD>
struct Fused64Cfg {
  static constexpr int D = 64;
  static constexpr int kAtom128 = 128 * 128;  // [128 rows x 64 cols] bf16, SW128
  static constexpr int kAtom64 = 64 * 128;    // [64 rows x 64 cols]
  static constexpr int kRes = 2 * kAtom128 + kAtom128;  // K' (K | Uk), V
  static constexpr int kItem = 2 * kAtom64 + kAtom64 + (DENSE ? 64 * 128 * 2 : 0);  // Q' (Q | Uq), dO, bias^T
  static constexpr int kSlot = (kItem + 1023) / 1024 * 1024;
  static constexpr int kDsBuf = 128 * 128;
  static constexpr int kStage = 32 * 64 * 4;  // 8 KB each: dQ half-tile, dUq half-tile
  static constexpr int kMisc = 2048 + 512;
  static constexpr int kBudget = 232448 - 1024;
  static constexpr int kSlotsFit = (kBudget - kRes - 2 * kDsBuf - 2 * kStage - kMisc) / kSlot;
  static constexpr int kSlots = kSlotsFit > 4 ? 4 : kSlotsFit;
  static constexpr int kSmem = 1024 + kRes + kSlots * kSlot + 2 * kDsBuf + 2 * kStage + kMisc;
  static constexpr int kKCols = 64 + 16 * RP;  // contraction of S^T: head dim + factor panels
  static_assert(RP <= 4, "d=64 fused path carries at most 64 factor columns");
  static_assert(kSlots >= 2, "fused64 ring too small");
};

struct Fused64Bars {
  uint64_t res_full, final_[2];
  uint64_t st_full[2], dpt_full[2], p_ready[2], ds_ready[2];
  uint64_t dq_full[2], dq_free[2], dsbuf_free[2];
  uint64_t slot_full[4], slot_empty[4];
  uint32_t tmem_base;
};

template <int RP, bool DENSE, bool BF16, bool FGRAD>
__global__ void __launch_bounds__(512, 1)
    fb_bwd_fused64_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_uqw, const __grid_constant__ CUtensorMap tm_biasT,
                          const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                          const __grid_constant__ CUtensorMap tm_ukw, const __grid_constant__ CUtensorMap tm_dqacc,
                          const __grid_constant__ CUtensorMap tm_duq, const BwdParams p) {
  using Cfg = Fused64Cfg<RP, DENSE, FGRAD>;
  constexpr int D = 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t k_base = sbase, v_base = sbase + 2 * Cfg::kAtom128;
  const uint32_t ring_base = sbase + Cfg::kRes;
  uint8_t* ds_buf = smem + Cfg::kRes + Cfg::kSlots * Cfg::kSlot;
  float* stage_dq = reinterpret_cast<float*>(ds_buf + 2 * Cfg::kDsBuf);
  float* stage_du = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(stage_dq) + Cfg::kStage);
  float* s_stats = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(stage_du) + Cfg::kStage);
  Fused64Bars* bars = reinterpret_cast<Fused64Bars*>(reinterpret_cast<uint8_t*>(s_stats) + 2048);

  const int warp = warp_id(), lane = lane_id();
  const int nkt = (p.M + 127) / 128;
  const int kt = blockIdx.x % nkt;
  const int bh = blockIdx.x / nkt;
  const int h = bh / p.B, b = bh % p.B;
  const int kv0 = kt * 128;
  const int nqb = (p.N + 63) / 64;
  const int i_start = p.causal ? kv0 / 64 : 0;
  const int nblk = nqb - i_start;
  const int rpad = RP * 16;

  if (warp == 12 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_dqacc);
    if (RP > 0) {
      tma_prefetch(&tm_uqw);
      tma_prefetch(&tm_ukw);
    }
    if (FGRAD) tma_prefetch(&tm_duq);
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
  constexpr uint32_t T_ST = 0, T_DPT = 128, T_DV = 256, T_DK = 320;

  if (warp >= 12) {
    regs_dec<96>();
    if (warp == 12 && lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const int hq = p.uq_hb ? 0 : h, bq = p.uq_bb ? 0 : b;
      const int hk = p.uk_hb ? 0 : h, bk = p.uk_bb ? 0 : b;
      const int hb_ = p.bias_hb ? 0 : h, bb_ = p.bias_bb ? 0 : b;
      mbar_arrive_expect_tx(&bars->res_full, RP > 0 ? Cfg::kRes : Cfg::kRes - Cfg::kAtom128);
      tma_load_4d(smem, &tm_k, &bars->res_full, 0, kv0, h, b);
      if (RP > 0) tma_load_4d(smem + Cfg::kAtom128, &tm_ukw, &bars->res_full, 0, kv0, hk, bk);
      tma_load_4d(smem + 2 * Cfg::kAtom128, &tm_v, &bars->res_full, 0, kv0, h, b);
      constexpr int kItemBytes = (RP > 0 ? 2 : 1) * Cfg::kAtom64 + Cfg::kAtom64 + (DENSE ? 64 * 128 * 2 : 0);
      for (int c = 0; c < nblk; ++c) {
        const int q0 = (i_start + c) * 64;
        const int slot = c % Cfg::kSlots, use = c / Cfg::kSlots;
        if (use > 0) mbar_wait(&bars->slot_empty[slot], (use - 1) & 1);
        uint8_t* dst = smem + Cfg::kRes + slot * Cfg::kSlot;
        uint64_t* fb_ = &bars->slot_full[slot];
        mbar_arrive_expect_tx(fb_, kItemBytes);
        tma_load_4d(dst, &tm_q, fb_, 0, q0, h, b);
        if (RP > 0) tma_load_4d(dst + Cfg::kAtom64, &tm_uqw, fb_, 0, q0, hq, bq);
        tma_load_4d(dst + 2 * Cfg::kAtom64, &tm_do, fb_, 0, q0, h, b);
        if (DENSE)
          for (int half = 0; half < 2; ++half)
            tma_load_4d(dst + 3 * Cfg::kAtom64 + half * 64 * 128, &tm_biasT, fb_, kv0 + half * 64, q0, hb_, bb_);
      }
    } else if ((warp == 13 || warp == 14) && lane == 0) {
      // ------------------------------------------------------------ MMA issuers (one per EW group)
      const int x = warp - 13;
      constexpr uint32_t id_s = make_idesc(128, 64, false, false, BF16);              // S^T, dP^T
      constexpr uint32_t id_v = make_idesc(128, D, false, true, BF16);                // dV (A from TMEM)
      constexpr uint32_t id_k = make_idesc(128, FGRAD ? 128 : D, false, true, BF16);  // dK' (A from TMEM)
      constexpr uint32_t id_q = make_idesc(128, 64, true, true, BF16);                // dQ'^T = K'^T dS^T
      const uint64_t dk_kt = mnmajor_desc(k_base, 128, 128, 0);                       // K'^T as A (2 atoms)
      const uint64_t dsb = mnmajor_desc(smem_u32(ds_buf) + x * Cfg::kDsBuf, 128, 128, 0);
      const uint32_t t_st = tmem + T_ST + 64 * x, t_dpt = tmem + T_DPT + 64 * x;
      auto slot_addr = [&](int c) { return ring_base + (c % Cfg::kSlots) * Cfg::kSlot; };
      auto wait_slot = [&](int c) {
        mbar_wait(&bars->slot_full[c % Cfg::kSlots], (c / Cfg::kSlots) & 1);
        tc_fence_after();
      };
      auto issue_st = [&](int c) {
        const uint32_t qb = slot_addr(c);
#pragma unroll
        for (int kk = 0; kk < Cfg::kKCols / 16; ++kk)
          mma_ss(t_st, kmajor_desc(k_base, 128, 128, kk * 16), kmajor_desc(qb, 64, 128, kk * 16), id_s,
                 kk > 0 ? 1u : 0u);
        tc_commit(&bars->st_full[x]);
      };
      auto issue_dpt = [&](int c) {
        if (c >= 2) mbar_wait(&bars->dq_free[x], ((c >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dob = slot_addr(c) + 2 * Cfg::kAtom64;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(t_dpt, kmajor_desc(v_base, 128, 128, kk * 16), kmajor_desc(dob, 64, 128, kk * 16), id_s,
                 kk > 0 ? 1u : 0u);
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
        const uint64_t mq = mnmajor_desc(qb, 64, 128, 0), mdo = mnmajor_desc(qb + 2 * Cfg::kAtom64, 64, 128, 0);
        mbar_wait(&bars->p_ready[x], u & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dV += P^T dO
          mma_ts(tmem + T_DV, t_st + kk * 8, mdo + kk * (16 * 128 >> 4), id_v, 1u);
        mbar_wait(&bars->ds_ready[x], u & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dK' += dS^T Q'  ([dK | dUk] when FGRAD)
          mma_ts(tmem + T_DK, t_dpt + kk * 8, mq + kk * (16 * 128 >> 4), id_k, 1u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ'^T = K'^T dS^T (M = 128: [dQ^T ; dUq^T]), into dP^T_x
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
    const int g = warp >> 2;
    const int r = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_st = tmem + lane_off + T_ST + 64 * g;
    const uint32_t t_dpt = tmem + lane_off + T_DPT + 64 * g;
    const int kv = kv0 + r;
    const float* lse_g = p.lse + static_cast<int64_t>(b * p.H + h) * p.N;
    const float* dl_g = p.delta + static_cast<int64_t>(b * p.H + h) * p.N;
    {  // zero dV (group 0) / dK' (group 1): every MMA into them accumulates
      uint32_t z[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) z[i] = 0u;
      if (g == 0) {
        tmem_st32(tmem + lane_off + T_DV, z);
        tmem_st32(tmem + lane_off + T_DV + 32, z);
      } else {
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32) tmem_st32(tmem + lane_off + T_DK + c0, z);
      }
      tmem_wait_st();
      tc_fence_before();
    }
    named_bar_sync(4, 256);
    tc_fence_after();
    for (int c = g; c < nblk; c += 2) {
      const int u = c >> 1;
      const int q0 = (i_start + c) * 64;
      float* st = s_stats + (g * 2 + (u & 1)) * 128;
      {
        const int qq = r & 63, q = q0 + qq;
        if (r < 64) st[qq] = q < p.N ? lse_g[q] * kLog2e64 : INFINITY;
        else st[64 + qq] = q < p.N ? dl_g[q] : 0.f;
      }
      named_bar_sync(1 + g, 128);
      float pr[64];
      mbar_wait(&bars->st_full[g], u & 1);
      tc_fence_after();
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
        const uint8_t* bt = smem + Cfg::kRes + (c % Cfg::kSlots) * Cfg::kSlot + 3 * Cfg::kAtom64;
        const int half = r >> 6, cc = r & 63;
#pragma unroll
        for (int qq = 0; qq < 64; ++qq) {
          const uint16_t raw = *reinterpret_cast<const uint16_t*>(bt + half * 64 * 128 + qq * 128 +
                                                                  (((cc >> 3) ^ (qq & 7)) << 4) + (cc & 7) * 2);
          float bv;
          if constexpr (BF16) bv = __bfloat162float(__ushort_as_bfloat16(raw));
          else bv = __half2float(__ushort_as_half(raw));
          pr[qq] = fmaf(bv, kLog2e64, pr[qq]);
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
          if (poly_pair(c2)) {
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
      if (lane == 0) mbar_arrive(&bars->p_ready[g]);
      mbar_wait(&bars->dpt_full[g], u & 1);
      tc_fence_after();
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
      if (lane == 0) mbar_arrive(&bars->ds_ready[g]);
    }
    // ---- epilogue: group 0 writes dV, group 1 writes dK (+ dUk)
    mbar_wait(&bars->final_[0], 0);
    mbar_wait(&bars->final_[1], 0);
    tc_fence_after();
    const bool valid = kv < p.M;
    typedef typename std::conditional<BF16, __nv_bfloat16, __half>::type elem_t;
    const uint32_t src = tmem + lane_off + (g == 0 ? T_DV : T_DK);
    const float mul = g == 0 ? 1.0f : p.scale;
    elem_t* dst = g == 0 ? reinterpret_cast<elem_t*>(p.dv) + static_cast<int64_t>(b) * p.dv_sb +
                               static_cast<int64_t>(h) * p.dv_sh + static_cast<int64_t>(kv) * p.dv_sn
                         : reinterpret_cast<elem_t*>(p.dk) + static_cast<int64_t>(b) * p.dk_sb +
                               static_cast<int64_t>(h) * p.dk_sh + static_cast<int64_t>(kv) * p.dk_sn;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(src + c0, v);
      tmem_wait_ld();
      if (valid) {
        uint32_t o16[16];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          o16[c] = pack2<BF16>(__uint_as_float(v[2 * c]) * mul, __uint_as_float(v[2 * c + 1]) * mul);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          reinterpret_cast<uint4*>(dst + c0)[q4] = make_uint4(o16[4 * q4], o16[4 * q4 + 1], o16[4 * q4 + 2], o16[4 * q4 + 3]);
      }
    }
    if constexpr (FGRAD) {
      if (g == 1) {
        float* du = p.duk + static_cast<int64_t>(b) * p.duk_sb + static_cast<int64_t>(h) * p.duk_sh +
                    static_cast<int64_t>(kv) * p.duk_sn;
#pragma unroll
        for (int pn = 0; pn < RP; ++pn) {
          uint32_t v[16];
          tmem_ld16(tmem + lane_off + T_DK + 64 + pn * 16, v);
          tmem_wait_ld();
          if (valid)
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              reinterpret_cast<float4*>(du + pn * 16)[q4] =
                  make_float4(__uint_as_float(v[4 * q4]) * p.scale, __uint_as_float(v[4 * q4 + 1]) * p.scale,
                              __uint_as_float(v[4 * q4 + 2]) * p.scale, __uint_as_float(v[4 * q4 + 3]) * p.scale);
        }
      }
    }
  } else {
    regs_dec<96>();
    // -------------------------------------------------------------- drain (warps 8-11)
    // TMEM lane L of dQ'^T: L < 64 -> dQ column L; L >= 64 -> factor rank L - 64
    const int L = threadIdx.x - 256;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const bool is_dq = L < 64;
    const bool lead_q = L == 0, lead_u = L == 64;
    for (int c = 0; c < nblk; ++c) {
      const int q0 = (i_start + c) * 64;
      const int x = c & 1, u = c >> 1;
      mbar_wait(&bars->dq_full[x], u & 1);
      tc_fence_after();
      uint32_t v[64];
      tmem_ld32(tmem + lane_off + T_DPT + 64 * x, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32(tmem + lane_off + T_DPT + 64 * x + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->dq_free[x]);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (lead_q || (FGRAD && lead_u)) bulk_wait_read0_();
        named_bar_sync(3, 128);
        if (is_dq) {
#pragma unroll
          for (int qq = 0; qq < 32; ++qq) stage_dq[qq * 64 + L] = __uint_as_float(v[32 * half + qq]) * p.scale;
        } else if (FGRAD && L - 64 < rpad) {
#pragma unroll
          for (int qq = 0; qq < 32; ++qq) stage_du[qq * rpad + (L - 64)] = __uint_as_float(v[32 * half + qq]) * p.scale;
        }
        fence_proxy_async();
        named_bar_sync(3, 128);
        if (lead_q) {
          tma_reduce_add_4d_(&tm_dqacc, stage_dq, 0, q0 + 32 * half, h, b);
          bulk_commit_();
        }
        if (FGRAD && lead_u) {
          tma_reduce_add_4d_(&tm_duq, stage_du, 0, q0 + 32 * half, h, b);
          bulk_commit_();
        }
      }
    }
    if (lead_q || lead_u) bulk_wait0_();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int RP, bool DENSE, bool BF16, bool FGRAD>
static cudaError_t launch64_t(const BwdMaps& m, const CUtensorMap& dqacc, const CUtensorMap& duq, const BwdParams& p,
                              cudaStream_t s) {
  using Cfg = Fused64Cfg<RP, DENSE, FGRAD>;
  auto k = fb_bwd_fused64_kernel<RP, DENSE, BF16, FGRAD>;
  static std::atomic<uint64_t> attr_mask{0};
  cudaError_t e = smem_attr_once(attr_mask, reinterpret_cast<const void*>(k), Cfg::kSmem);
  if (e != cudaSuccess) return e;
  k<<<((p.M + 127) / 128) * p.B * p.H, 512, Cfg::kSmem, s>>>(m.q64, m.do64, m.uq64w, m.biasT, m.k128, m.v128,
                                                             m.uk128w, dqacc, duq, p);
  return cudaGetLastError();
}

template <bool BF16>
static cudaError_t f64_rp(int rp, bool dense, bool fgrad, const BwdMaps& m, const CUtensorMap& dqacc,
                          const CUtensorMap& duq, const BwdParams& p, cudaStream_t s) {
  if (dense) return rp == 0 ? launch64_t<0, true, BF16, false>(m, dqacc, duq, p, s) : cudaErrorInvalidValue;
  if (fgrad) {
    switch (rp) {
      case 1: return launch64_t<1, false, BF16, true>(m, dqacc, duq, p, s);
      case 2: return launch64_t<2, false, BF16, true>(m, dqacc, duq, p, s);
      case 3: return launch64_t<3, false, BF16, true>(m, dqacc, duq, p, s);
      case 4: return launch64_t<4, false, BF16, true>(m, dqacc, duq, p, s);
    }
    return cudaErrorInvalidValue;
  }
  switch (rp) {
    case 0: return launch64_t<0, false, BF16, false>(m, dqacc, duq, p, s);
    case 1: return launch64_t<1, false, BF16, false>(m, dqacc, duq, p, s);
    case 2: return launch64_t<2, false, BF16, false>(m, dqacc, duq, p, s);
    case 3: return launch64_t<3, false, BF16, false>(m, dqacc, duq, p, s);
    case 4: return launch64_t<4, false, BF16, false>(m, dqacc, duq, p, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwd_fused64_sm100(int rp, bool dense, bool bf16, bool fgrad, const BwdMaps& m,
                                     const CUtensorMap& dqacc, const CUtensorMap& duq, const BwdParams& p,
                                     cudaStream_t s) {
  return bf16 ? f64_rp<true>(rp, dense, fgrad, m, dqacc, duq, p, s)
              : f64_rp<false>(rp, dense, fgrad, m, dqacc, duq, p, s);
}

}  // namespace fb
