// fb_bwd_t128_sm100.cu — single-pass FlashBias backward for head dim 128 on
// 128-key x 128-query tiles (K2 fused, no factor gradients, Rpad <= 16).
//
// Same math as fb_bwd_fused_sm100.cu (oracle/flashbias_oracle.py:attention_bwd):
//   S^T = K' Q'^T, P^T = exp(scale S^T - lse), dP^T = V dO^T,
//   dS^T = P^T (dP^T - D), dV += P^T dO, dK += dS^T Q, dQ^T = K^T dS^T.
// Why a second d=128 kernel: tcgen05.mma with N = 64 costs ~45 cycles per
// K-step against a 32-cycle floor (tests/gpu_probe/contention.cu, SS and TS
// alike), so the 64-query kernel tops out near 80% of the tensor pipe.  Here
// every GEMM is M = 128, N = 128 (64 cycles per K-step, at the floor).
//
// TMEM (512 columns): S^T/P^T [0,128) | dP^T, then dQ^T [128,256) | dV | dK.
// dS^T goes to shared memory only (SW128, rows = keys): it is the K-major A
// operand of dK (SS) and the MN-major B operand of dQ^T, so the dP^T columns
// are free as soon as the elementwise warps have loaded dP^T, and dQ^T(j)
// lands there while dK(j) runs; its drain (TMEM -> regs) overlaps dK(j).
// P^T (bf16) is written back over the S^T columns each group read (group g:
// queries [64g, 64g+64) -> columns [64g, 64g+32)) and feeds dV as a TS MMA.
//
// MMA order (single issuing thread; tcgen05 MMAs of one CTA run in order):
//   prologue: S(0) dP(0) dV(0)
//   block j:  S(j+1) | dQ^T(j) dK(j) | dP(j+1) dV(j+1)
// Windows per 2624-cycle iteration: P(j+1) has dQ+dK+dP (~1536 cycles) after
// S(j+1) lands; dS(j+1) has dV+S (~1088); the dQ drain has dK (512).
//
// Warp roles (512 threads): warps 0-3 / 4-7 elementwise for query columns
// [0,64) / [64,128) (thread = key row = TMEM lane), 8-11 dQ drain (thread =
// head-dim lane of dQ^T: TMEM -> smem -> TMA reduce-add into the fp32 dQ
// accumulator), warp 12 TMA producer, warp 13 TMEM alloc + MMA issuer.
//
// MC (cluster multicast) variant: a cluster of two CTAs owns two adjacent key
// tiles of one head and streams the SAME query blocks in lockstep, so each
// Q / dO / Uq tile is read from L2 once for both SMs: each CTA's producer
// loads one 64-column atom and multicasts it to both CTAs (the full barriers
// expect the whole tile), and a slot is refilled only after BOTH CTAs' MMAs
// have released it (multicast commits, empty barriers count 2).  L2 is the
// shared bottleneck of this kernel (the dQ reduce-adds and these loads go
// through the same slices: tests/gpu_probe/reduce_rate.cu), so halving the
// load traffic leaves more of it to the reductions.  Causal: both CTAs start
// at the even tile's diagonal block; for the odd tile that first block is
// fully masked (P = dS = 0) and its dQ reduction is skipped.
//
// LEARN variant (learnable factors, one 16-column panel): the factor gradients
// dUk = scale dS^T Uq and dUq = scale dS Uk are two extra N = 16 MMAs per block.
// TMEM has no free columns for a dUk accumulator (S^T | dP^T | dV | dK fill all
// 512), so both land in the dP^T columns once the elementwise warps have read
// dP^T: the drain adds the 16 dUk columns into registers (written at the end,
// one fp32 row per key) and reduce-adds the 128 x 16 dUq block into the fp32
// dUq output like a 9th dQ chunk.  MMA order per block becomes
//   S(j+1) | dUk(j) dUq(j) dK(j) | dQ^T(j) | dP(j+1) dV(j+1)
// with dQ^T(j) issued once the drain has read the factor columns.
#include "fb_kernels.h"
#include "fb_sm100.cuh"

#ifndef T128_REG_EW
#define T128_REG_EW 144
#endif
#ifndef T128_REG_DR
#define T128_REG_DR 152
#endif
#ifndef T128_REG_OT
#define T128_REG_OT 72
#endif
// dQ drain: TMA reduce-add from a swizzled smem stage.  Measured alternatives: per-warp
// 2 KB boxes without cross-warp barriers (equal), red.global.add.v4.f32 after a per-warp smem transpose
// (C3 bwd 25.1-25.4 ms vs 23.1), plain TMA stores (same time).
#ifndef T128_QCHUNK
#define T128_QCHUNK 16  // queries per dQ reduce-add box (16 KB of stages: 16 -> 2 x 8 KB SW64, 8 -> 4 x 4 KB SW32)
#endif
static_assert(2 * T128_REG_EW + T128_REG_DR + T128_REG_OT <= 512, "t128 register pool");

namespace fb {

namespace {
constexpr float kLog2eT = 1.4426950408889634f;

__device__ __forceinline__ void t128_reduce_add(const CUtensorMap* map, const void* smem, int c0, int c1, int c2,
                                                int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void t128_bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void t128_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
template <int N>
__device__ __forceinline__ void t128_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void t128_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
}  // namespace

template <int RP>
struct T128Cfg {
  static constexpr int kTile = 128 * 128 * 2;  // 32 KB: 128 rows x 128 bf16, two SW128 atoms
  static constexpr int kPanel = 128 * 32;      // 16 factor columns, SW32
  static constexpr int kK = 0, kV = kTile, kUk = 2 * kTile;
  static constexpr int kRes = (2 * kTile + RP * kPanel + 1023) / 1024 * 1024;
  static constexpr int kQSlot = (kTile + RP * kPanel + 1023) / 1024 * 1024;
  static constexpr int kQ0 = kRes;
  static constexpr int kDO = kQ0 + 2 * kQSlot;
  static constexpr int kDS = kDO + kTile;
  static constexpr int kStage = kDS + kTile;   // 2 x 8 KB fp32: 16 queries x 128 dims (dUq chunk: SW64 rows)
  static constexpr int kStats = kStage + 32 * 128 * 4;
  static constexpr int kBars = kStats + 2 * 2 * 128 * 4;
  static constexpr int kSmem = 1024 + kBars + 256;
  static_assert(kSmem <= 232448, "t128 backward: shared memory budget");
};

struct T128Bars {
  uint64_t res_full;
  uint64_t q_full[2], q_empty[2];
  uint64_t do_full, do_empty;
  uint64_t s_full, p_ready, dp_full, ds_ready, ds_free, dq_full, dq_free, final_;
  uint64_t fg_full, fg_free;  // LEARN: factor-gradient columns written / read out of the dP^T region
  uint32_t tmem_base;
};

template <int RP, bool BF16, bool MC, bool LEARN>
__global__ void __launch_bounds__(512, 1)
    fb_bwd_t128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_uq, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_uk,
                       const __grid_constant__ CUtensorMap tm_dqacc, const __grid_constant__ CUtensorMap tm_duq,
                       const BwdParams p) {
  static_assert(!LEARN || RP == 1, "factor gradients: one 16-column panel");
  using Cfg = T128Cfg<RP>;
  constexpr int D = 128;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  const uint32_t sbase = smem_u32(smem);
  uint8_t* ds_buf = smem + Cfg::kDS;
  float* dq_stage = reinterpret_cast<float*>(smem + Cfg::kStage);
  float* s_stats = reinterpret_cast<float*>(smem + Cfg::kStats);  // [2 buf][lse | delta][128]
  T128Bars* bars = reinterpret_cast<T128Bars*>(smem + Cfg::kBars);

  const int warp = warp_id(), lane = lane_id();
  const int nkt = (p.M + 127) / 128;
  const int kt = blockIdx.x % nkt;
  const int bh = blockIdx.x / nkt;
  const int h = bh / p.B, b = bh % p.B;
  const int kv0 = kt * 128;
  const int nqb = (p.N + 127) / 128;
  // MC: the pair (even tile, odd tile) shares one query-block stream starting at the even tile's diagonal
  const uint32_t crank = MC ? cluster_ctarank() : 0u;
  const int i_start = p.causal ? (MC ? (kt & ~1) : kt) : 0;
  const int nblk = nqb > i_start ? nqb - i_start : 0;
  constexpr uint16_t kPair = 3;

  if (warp == 12 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_dqacc);
    if (LEARN) tma_prefetch(&tm_duq);
    if (RP > 0) {
      tma_prefetch(&tm_uq);
      tma_prefetch(&tm_uk);
    }
    mbar_init(&bars->res_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], MC ? 2 : 1);  // MC: released by both CTAs' MMAs
    }
    mbar_init(&bars->do_full, 1);
    mbar_init(&bars->do_empty, MC ? 2 : 1);
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->p_ready, 8);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->ds_ready, 8);
    mbar_init(&bars->ds_free, 1);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->dq_free, 4);
    mbar_init(&bars->final_, 1);
    mbar_init(&bars->fg_full, 1);
    mbar_init(&bars->fg_free, 4);
    fence_barrier_init();
  }
  if (warp == 13) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync_all();  // both CTAs' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  constexpr uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 384;

  if (warp >= 12) {
    regs_dec<T128_REG_OT>();
    if (warp == 12 && lane == 0 && nblk > 0) {
      // ------------------------------------------------------------ TMA producer
      const int hq = p.uq_hb ? 0 : h, bq = p.uq_bb ? 0 : b;
      const int hk = p.uk_hb ? 0 : h, bk = p.uk_bb ? 0 : b;
      mbar_arrive_expect_tx(&bars->res_full, 2 * Cfg::kTile + RP * Cfg::kPanel);
      for (int a = 0; a < 2; ++a) {
        tma_load_4d(smem + Cfg::kK + a * 16384, &tm_k, &bars->res_full, a * 64, kv0, h, b);
        tma_load_4d(smem + Cfg::kV + a * 16384, &tm_v, &bars->res_full, a * 64, kv0, h, b);
      }
      for (int pn = 0; pn < RP; ++pn)
        tma_load_4d(smem + Cfg::kUk + pn * Cfg::kPanel, &tm_uk, &bars->res_full, pn * 16, kv0, hk, bk);
      for (int j = 0; j < nblk; ++j) {
        const int q0 = (i_start + j) * 128;
        const int slot = j & 1, use = j >> 1;
        if (use > 0) mbar_wait(&bars->q_empty[slot], (use - 1) & 1);
        uint8_t* qd = smem + Cfg::kQ0 + slot * Cfg::kQSlot;
        mbar_arrive_expect_tx(&bars->q_full[slot], Cfg::kTile + RP * Cfg::kPanel);
        if constexpr (MC) {  // this CTA's atom (and CTA 0: the factor panels) to both CTAs
          tma_load_4d_mc(qd + crank * 16384, &tm_q, &bars->q_full[slot], crank * 64, q0, h, b, kPair);
          if (crank == 0)
            for (int pn = 0; pn < RP; ++pn)
              tma_load_4d_mc(qd + Cfg::kTile + pn * Cfg::kPanel, &tm_uq, &bars->q_full[slot], pn * 16, q0, hq, bq,
                             kPair);
        } else {
          for (int a = 0; a < 2; ++a) tma_load_4d(qd + a * 16384, &tm_q, &bars->q_full[slot], a * 64, q0, h, b);
          for (int pn = 0; pn < RP; ++pn)
            tma_load_4d(qd + Cfg::kTile + pn * Cfg::kPanel, &tm_uq, &bars->q_full[slot], pn * 16, q0, hq, bq);
        }
        if (j > 0) mbar_wait(&bars->do_empty, (j - 1) & 1);
        trace(p.trace, p.trace_cta, 21, j);
        mbar_arrive_expect_tx(&bars->do_full, Cfg::kTile);
        if constexpr (MC) {
          tma_load_4d_mc(smem + Cfg::kDO + crank * 16384, &tm_do, &bars->do_full, crank * 64, q0, h, b, kPair);
        } else {
          for (int a = 0; a < 2; ++a)
            tma_load_4d(smem + Cfg::kDO + a * 16384, &tm_do, &bars->do_full, a * 64, q0, h, b);
        }
      }
    } else if (warp == 13 && lane == 0 && nblk > 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t id_s = make_idesc(128, 128, false, false, BF16);  // S^T, dP^T (K-major A, B)
      constexpr uint32_t id_d = make_idesc(128, D, false, true, BF16);     // dV (A TMEM), dK (A smem K-major)
      constexpr uint32_t id_q = make_idesc(128, 128, true, true, BF16);    // dQ^T = K^T dS^T
      // Descriptors are rebuilt from an opaque copy of the smem base inside each
      // issue step: otherwise the compiler hoists all 8 K-step variants of every
      // operand out of the block loop and the issuing thread spills.
      auto desc = [&](int off, bool mn) {
        const uint32_t a = opaque_u32(sbase) + off;
        return mn ? mnmajor_desc(a, 128, 128, 0) : kmajor_desc(a, 128, 128, 0);
      };
      // K-step kk of a 128-row SW128 K-major tile: atom (kk / 4), 32-byte column step (kk % 4)
      auto ks = [](int kk) -> uint64_t { return (kk >> 2) * (128 * 128 >> 4) + (kk & 3) * 2; };
      constexpr uint64_t kRow16 = 16 * 128 >> 4;  // 16 rows of an MN-major SW128 tile
      auto qslot = [&](int j) { return Cfg::kQ0 + (j & 1) * Cfg::kQSlot; };
      auto issue_s = [&](int j) {
        mbar_wait(&bars->q_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        trace(p.trace, p.trace_cta, 11, j);
        const uint64_t dq = desc(qslot(j), false), dk_k = desc(Cfg::kK, false);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) mma_ss(tmem + T_S, dk_k + ks(kk), dq + ks(kk), id_s, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int pn = 0; pn < RP; ++pn)
          mma_ss(tmem + T_S, make_sdesc(opaque_u32(sbase) + Cfg::kUk + pn * Cfg::kPanel, 16, 256, 6),
                 make_sdesc(opaque_u32(sbase) + qslot(j) + Cfg::kTile + pn * Cfg::kPanel, 16, 256, 6), id_s, 1u);
        tc_commit(&bars->s_full);
      };
      auto issue_dp = [&](int j) {
        mbar_wait(&bars->do_full, j & 1);
        if (j > 0) mbar_wait(&bars->dq_free, (j - 1) & 1);  // dQ^T(j-1) drained out of these columns
        tc_fence_after();
        trace(p.trace, p.trace_cta, 14, j);
        const uint64_t dk_v = desc(Cfg::kV, false), dk_do = desc(Cfg::kDO, false);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + T_DP, dk_v + ks(kk), dk_do + ks(kk), id_s, kk > 0 ? 1u : 0u);
        tc_commit(&bars->dp_full);
      };
      auto issue_dv = [&](int j) {
        mbar_wait(&bars->p_ready, j & 1);
        tc_fence_after();
        trace(p.trace, p.trace_cta, 10, j);
        const uint64_t dm_do = desc(Cfg::kDO, true);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // K = 128 queries; P^T of group g sits at columns [64g, 64g+32)
          mma_ts(tmem + T_DV, tmem + T_S + (kk >> 2) * 64 + (kk & 3) * 8, dm_do + kk * kRow16, id_d,
                 (j > 0 || kk > 0) ? 1u : 0u);
        if constexpr (MC) tc_commit_mc(&bars->do_empty, kPair);
        else tc_commit(&bars->do_empty);
      };
      // 16-column factor panel (rows = K index, SW32) as an MN-major operand: K-step = 16 rows x 32 B
      auto panel_mn = [&](int off) { return make_sdesc(opaque_u32(sbase) + off, 128 * 32, 8 * 32, 6); };
      constexpr uint64_t kPanelRow16 = 16 * 32 >> 4;
      auto issue_dq = [&](int j) {
        const uint64_t dm_kt = desc(Cfg::kK, true), dm_ds = desc(Cfg::kDS, true);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ^T = K^T dS^T (K = 128 keys) into the dP^T columns
          mma_ss(tmem + T_DP, dm_kt + kk * kRow16, dm_ds + kk * kRow16, id_q, kk > 0 ? 1u : 0u);
        tc_commit(&bars->dq_full);
        (void)j;
      };
      auto issue_dk = [&](int j) {
        trace(p.trace, p.trace_cta, 12, j);
        const uint64_t dm_q = desc(qslot(j), true), dk_ds = desc(Cfg::kDS, false);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dK += dS^T Q (K = 128 queries)
          mma_ss(tmem + T_DK, dk_ds + ks(kk), dm_q + kk * kRow16, id_d, (j > 0 || kk > 0) ? 1u : 0u);
      };
      auto issue_dqk = [&](int j) {
        mbar_wait(&bars->ds_ready, j & 1);
        tc_fence_after();
        trace(p.trace, p.trace_cta, 13, j);
        if constexpr (LEARN) {
          constexpr uint32_t id_fk = make_idesc(128, 16, false, true, BF16);  // dUk part = dS^T Uq
          constexpr uint32_t id_fq = make_idesc(128, 16, true, true, BF16);   // dUq = dS Uk (A = dS^T read MN-major)
          const uint64_t dk_ds = desc(Cfg::kDS, false), dm_ds = desc(Cfg::kDS, true);
          const uint64_t uq_mn = panel_mn(qslot(j) + Cfg::kTile), uk_mn = panel_mn(Cfg::kUk);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(tmem + T_DP, dk_ds + ks(kk), uq_mn + kk * kPanelRow16, id_fk, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(tmem + T_DP + 16, dm_ds + kk * kRow16, uk_mn + kk * kPanelRow16, id_fq, kk > 0 ? 1u : 0u);
          tc_commit(&bars->fg_full);
          issue_dk(j);
          if constexpr (MC) tc_commit_mc(&bars->q_empty[j & 1], kPair);
          else tc_commit(&bars->q_empty[j & 1]);
          mbar_wait(&bars->fg_free, j & 1);  // the drain has read the factor columns out of the dP^T region
          tc_fence_after();
          issue_dq(j);
        } else {
          issue_dq(j);
          issue_dk(j);
          if constexpr (MC) tc_commit_mc(&bars->q_empty[j & 1], kPair);
          else tc_commit(&bars->q_empty[j & 1]);
        }
        tc_commit(&bars->ds_free);
      };
      mbar_wait(&bars->res_full, 0);
      issue_s(0);
      issue_dp(0);
      issue_dv(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) issue_s(j + 1);
        issue_dqk(j);
        if (j + 1 < nblk) {
          issue_dp(j + 1);
          issue_dv(j + 1);
        }
      }
      tc_commit(&bars->final_);
    }
  } else if (warp < 8) {
    regs_inc<T128_REG_EW>();
    // -------------------------------------------------------------- elementwise (thread = key row)
    const int g = warp >> 2;           // query columns [64g, 64g+64) of each block
    const int r = threadIdx.x & 127;   // key row within the tile == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_off + T_S + 64 * g;
    const uint32_t t_dp = tmem + lane_off + T_DP + 64 * g;
    const int kv = kv0 + r;
    const float* lse_g = p.lse + static_cast<int64_t>(b * p.H + h) * p.N;
    const float* dl_g = p.delta + static_cast<int64_t>(b * p.H + h) * p.N;
    uint8_t* ds_row = ds_buf + g * 16384 + r * 128;
    // LSE / delta of block j are fetched from global during block j - 1
    const int tq = threadIdx.x & 127;
    const float* src_g = threadIdx.x < 128 ? lse_g : dl_g;
    const float pad = threadIdx.x < 128 ? INFINITY : 0.f, mul = threadIdx.x < 128 ? kLog2eT : 1.f;
    float pre = (i_start * 128 + tq) < p.N ? src_g[i_start * 128 + tq] * mul : pad;
    for (int j = 0; j < nblk; ++j) {
      const int q0 = (i_start + j) * 128;
      float* st = s_stats + (j & 1) * 256;
      st[threadIdx.x] = pre;
      if (j + 1 < nblk) pre = (q0 + 128 + tq) < p.N ? src_g[q0 + 128 + tq] * mul : pad;
      named_bar_sync(1, 256);
      const float* lse2 = st + 64 * g;
      const float* dlt = st + 128 + 64 * g;
      float pr[64];
      mbar_wait(&bars->s_full, j & 1);
      tc_fence_after();
      if (r == 0) trace(p.trace, p.trace_cta, 15 + g * 7, j);
      {
        uint32_t v[64];
        tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_wait_ld();
        const float2 mul = make_float2(p.scale_log2, p.scale_log2);
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 x = ffma2(make_float2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])), mul,
                                 make_float2(-lse2[c], -lse2[c + 1]));
          pr[c] = x.x;
          pr[c + 1] = x.y;
        }
      }
      if (p.causal && q0 <= kv0) {  // diagonal block (MC odd tile: also the fully masked block before it)
        const int qb = q0 + 64 * g;
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (kv > qb + c) pr[c] = -INFINITY;
      }
      {
        uint32_t pk[32];
#pragma unroll
        for (int c2 = 0; c2 < 32; ++c2) {
          if (poly_pair(c2)) {  // FB_POLY_NUM pairs in 8 on the FMA pipe
            const float2 e2 = ex2_poly2(make_float2(pr[2 * c2], pr[2 * c2 + 1]));
            pr[2 * c2] = e2.x;
            pr[2 * c2 + 1] = e2.y;
          } else {
            pr[2 * c2] = ex2(pr[2 * c2]);
            pr[2 * c2 + 1] = ex2(pr[2 * c2 + 1]);
          }
          pk[c2] = pack2<BF16>(pr[2 * c2], pr[2 * c2 + 1]);
        }
        tmem_st32(t_s, pk);  // P^T over the first 32 of this group's S^T columns
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (r == 0) trace(p.trace, p.trace_cta, 16 + g * 7, j);
      if (lane == 0) mbar_arrive(&bars->p_ready);
      mbar_wait(&bars->dp_full, j & 1);
      tc_fence_after();
      if (r == 0) trace(p.trace, p.trace_cta, 17 + g * 7, j);
      if (j > 0) mbar_wait(&bars->ds_free, (j - 1) & 1);  // dK(j-1) finished reading dS^T
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t v[32];
        tmem_ld32(t_dp + 32 * hf, v);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int c2 = 0; c2 < 16; ++c2) {
          const int c = 32 * hf + 2 * c2;
          const float2 dpd = fadd2(make_float2(__uint_as_float(v[2 * c2]), __uint_as_float(v[2 * c2 + 1])),
                                   make_float2(-dlt[c], -dlt[c + 1]));
          const float2 ds = fmul2(make_float2(pr[c], pr[c + 1]), dpd);
          pk[c2] = pack2<BF16>(ds.x, ds.y);
        }
        // dS^T row r, queries [64g + 32hf, +32): 16-byte chunks ch = 4hf..4hf+3 of the
        // 128-byte swizzled line, chunk ch stored at ch ^ (r & 7)
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int ch = 4 * hf + c4;
          *reinterpret_cast<uint4*>(ds_row + ((ch ^ (r & 7)) << 4)) =
              make_uint4(pk[4 * c4], pk[4 * c4 + 1], pk[4 * c4 + 2], pk[4 * c4 + 3]);
        }
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (r == 0) trace(p.trace, p.trace_cta, 18 + g * 7, j);
      if (lane == 0) mbar_arrive(&bars->ds_ready);
    }
    // ---- epilogue: group 0 writes dV rows, group 1 dK rows (scaled)
    typedef typename std::conditional<BF16, __nv_bfloat16, __half>::type elem_t;
    const bool valid = kv < p.M;
    elem_t* dst = g == 0 ? reinterpret_cast<elem_t*>(p.dv) + static_cast<int64_t>(b) * p.dv_sb +
                               static_cast<int64_t>(h) * p.dv_sh + static_cast<int64_t>(kv) * p.dv_sn
                         : reinterpret_cast<elem_t*>(p.dk) + static_cast<int64_t>(b) * p.dk_sb +
                               static_cast<int64_t>(h) * p.dk_sh + static_cast<int64_t>(kv) * p.dk_sn;
    const float osc = g == 0 ? 1.f : p.scale;
    if (nblk > 0) {
      mbar_wait(&bars->final_, 0);
      tc_fence_after();
    }
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t v[32];
      if (nblk > 0) {
        tmem_ld32(tmem + lane_off + (g == 0 ? T_DV : T_DK) + c0, v);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0u;
      }
      if (valid) {
        uint32_t o16[16];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          o16[c] = pack2<BF16>(__uint_as_float(v[2 * c]) * osc, __uint_as_float(v[2 * c + 1]) * osc);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          reinterpret_cast<uint4*>(dst + c0)[q4] =
              make_uint4(o16[4 * q4], o16[4 * q4 + 1], o16[4 * q4 + 2], o16[4 * q4 + 3]);
      }
    }
  } else {
    regs_inc<T128_REG_DR>();
    // -------------------------------------------------------------- dQ drain (warps 8-11)
    // dQ^T (lane = head dim) is reduce-added into the fp32 accumulator [B,H,N,128]
    // (head dims contiguous) in 16-query x 128-dim boxes: thread dd writes column
    // dd of each query row of the stage (a warp writes 128 contiguous bytes per
    // query: conflict-free), so each box row the L2 reduces is a full 512-byte
    // line.  Two 8 KB stages, one reduction in flight while the next is written.
    const int dd = threadIdx.x - 256;  // head-dim index = TMEM lane of dQ^T
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const bool leader = dd == 0;
    int chunk = 0;
    constexpr int QC = T128_QCHUNK, RB = QC * 4, NST = 16384 / (128 * RB);  // row bytes, stages
    float duk[LEARN ? 16 : 1];
#pragma unroll
    for (int c = 0; c < (LEARN ? 16 : 1); ++c) duk[c] = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int q0 = (i_start + j) * 128;
      // MC odd tile, causal: the first shared block lies entirely above this tile's diagonal (dQ^T = 0)
      const bool skip = MC && p.causal && q0 + 128 <= kv0;
      if constexpr (LEARN) {
        static_assert(!LEARN || RB == 64, "the dUq chunk reuses the 64-byte-row stage geometry");
        mbar_wait(&bars->fg_full, j & 1);
        tc_fence_after();
        uint32_t f[32];  // [0,16): dUk part (lane = key), [16,32): dUq (lane = query)
        tmem_ld32(tmem + lane_off + T_DP, f);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->fg_free);
#pragma unroll
        for (int c = 0; c < 16; ++c) duk[c] += __uint_as_float(f[c]);
        if (!skip) {  // the 128 x 16 dUq block: one more 8 KB chunk through the dQ stages
          uint8_t* stg = reinterpret_cast<uint8_t*>(dq_stage) + (chunk % NST) * (128 * RB);
          if (leader) t128_wait_read<NST - 1>();
          named_bar_sync(3, 128);
          const float sc = p.scale;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4)
            *reinterpret_cast<float4*>(stg + dd * RB + ((c4 ^ ((dd * RB >> 7) & (RB / 16 - 1))) << 4)) =
                make_float4(__uint_as_float(f[16 + 4 * c4]) * sc, __uint_as_float(f[17 + 4 * c4]) * sc,
                            __uint_as_float(f[18 + 4 * c4]) * sc, __uint_as_float(f[19 + 4 * c4]) * sc);
          fence_proxy_async();
          named_bar_sync(3, 128);
          if (leader) {
            t128_reduce_add(&tm_duq, stg, 0, q0, h, b);
            t128_bulk_commit();
          }
          ++chunk;
        }
      }
      mbar_wait(&bars->dq_full, j & 1);
      tc_fence_after();
      if (leader) trace(p.trace, p.trace_cta, 19, j);
      uint32_t v[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_ld32(tmem + lane_off + T_DP + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->dq_free);
#pragma unroll
      for (int c = 0; c < (skip ? 0 : 128 / QC); ++c, ++chunk) {
        // stage = [16 queries][128 dims] fp32: thread dd writes column dd (consecutive words per query row)
        float* stg = dq_stage + (chunk % NST) * (QC * 128);
        if (leader) trace(p.trace, p.trace_cta, 26, j * 8 + c);
        if (leader) t128_wait_read<NST - 1>();  // the reduction that last read this stage has finished reading
        if (leader) trace(p.trace, p.trace_cta, 27, j * 8 + c);
        named_bar_sync(3, 128);
        const float sc = p.scale;
#pragma unroll
        for (int qq = 0; qq < QC; ++qq) stg[qq * 128 + dd] = __uint_as_float(v[QC * c + qq]) * sc;
        if (leader) trace(p.trace, p.trace_cta, 28, j * 8 + c);
        fence_proxy_async();
        if (leader) trace(p.trace, p.trace_cta, 29, j * 8 + c);
        named_bar_sync(3, 128);
        if (leader) {
          trace(p.trace, p.trace_cta, 30, j * 8 + c);
          t128_reduce_add(&tm_dqacc, stg, 0, q0 + QC * c, h, b);
          t128_bulk_commit();
        }
      }
      if (leader) trace(p.trace, p.trace_cta, 20, j);
    }
    if (leader) t128_wait_all();
    if constexpr (LEARN) {  // dUk rows (lane dd = key kv0 + dd), fp32, scaled like dK
      const int kv = kv0 + dd;
      if (kv < p.M) {
        float* dst = p.duk + static_cast<int64_t>(b) * p.duk_sb + static_cast<int64_t>(h) * p.duk_sh +
                     static_cast<int64_t>(kv) * p.duk_sn;
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4)
          reinterpret_cast<float4*>(dst)[c4] = make_float4(duk[4 * c4] * p.scale, duk[4 * c4 + 1] * p.scale,
                                                           duk[4 * c4 + 2] * p.scale, duk[4 * c4 + 3] * p.scale);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  // MC: the peer's last multicast commits / loads target this CTA's smem: exit together
  if constexpr (MC) cluster_sync_all();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

#ifndef T128_MULTICAST
#define T128_MULTICAST 1
#endif

template <int RP, bool BF16, bool MC, bool LEARN>
static cudaError_t launch_t128_mc(const BwdMaps& m, const CUtensorMap& dqacc, const CUtensorMap& duq,
                                  const BwdParams& p, cudaStream_t s) {
  using Cfg = T128Cfg<RP>;
  auto k = fb_bwd_t128_kernel<RP, BF16, MC, LEARN>;
  static std::atomic<uint64_t> attr_mask{0};
  cudaError_t e = smem_attr_once(attr_mask, reinterpret_cast<const void*>(k), Cfg::kSmem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(((p.M + 127) / 128) * p.B * p.H);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MC ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k, m.q128, m.do128, m.uq128, m.k128, m.v128, m.uk128, dqacc, duq, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// cluster pairs need an even number of key tiles per head (adjacent tiles of one head)
template <int RP, bool BF16, bool LEARN>
static cudaError_t launch_t128_t(const BwdMaps& m, const CUtensorMap& dqacc, const CUtensorMap& duq,
                                 const BwdParams& p, cudaStream_t s) {
  const int nkt = (p.M + 127) / 128;
  if (T128_MULTICAST && nkt % 2 == 0) return launch_t128_mc<RP, BF16, true, LEARN>(m, dqacc, duq, p, s);
  return launch_t128_mc<RP, BF16, false, LEARN>(m, dqacc, duq, p, s);
}

bool bwd_t128_supported(int d, int rp, bool dense, bool factor_grads) {
  return d == 128 && !dense && (factor_grads ? rp == 1 : rp <= 1);
}

cudaError_t launch_bwd_t128_sm100(int rp, bool bf16, bool fgrad, const BwdMaps& m, const CUtensorMap& dqacc,
                                  const CUtensorMap& duq, const BwdParams& p, cudaStream_t s) {
  if (fgrad) {
    if (rp != 1) return cudaErrorInvalidValue;
    return bf16 ? launch_t128_t<1, true, true>(m, dqacc, duq, p, s) : launch_t128_t<1, false, true>(m, dqacc, duq, p, s);
  }
  if (rp == 0)
    return bf16 ? launch_t128_t<0, true, false>(m, dqacc, duq, p, s) : launch_t128_t<0, false, false>(m, dqacc, duq, p, s);
  if (rp == 1)
    return bf16 ? launch_t128_t<1, true, false>(m, dqacc, duq, p, s) : launch_t128_t<1, false, false>(m, dqacc, duq, p, s);
  return cudaErrorInvalidValue;
}

}  // namespace fb
