// fb_fwd_sm100.cu — FlashBias forward on sm_100a (K1), dense-bias baseline
// (K3) and the no-bias variant, all from one warp-specialised pipeline.
//
// Restates the reference streaming loop (pkg/src/flashbias/attention.py:174-201)
// on tcgen05: the factored bias enters as extra UMMA K-steps from a second
// shared-memory descriptor (the widened contraction [q | sqrt(C) fq][k | fk]^T
// of attention.py:225-230 without materialising anything), the dense bias as
// a TMA-staged tile added in the softmax stage (attention.py:187-188).
//
// CTA = two 128-row query tiles (t = 0, 1) sharing one K/V stream.
//   warps 0-3  softmax for tile 0 (thread = query row = TMEM lane)
//   warps 4-7  softmax for tile 1
//   warp  8    TMA producer (Q, U once; K(+fk), bias, V ring per KV block)
//   warp  9    TMEM allocator + single-thread tcgen05.mma issuer
//   warps 10-11 idle (complete the third warpgroup for setmaxnreg)
// Register budget: softmax warpgroups 208 regs/thread, the rest 80 (8*208 + 4*80 <= 384*168, the launch pool).
// TMEM columns: S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// P_t (bf16/f16 pairs) overwrites the first 64 columns of S_t and feeds the
// PV MMA directly from TMEM (A operand), so P never touches shared memory.
// Online softmax with lazy rescaling: the running max only moves when it
// grows by more than 8 (log2 units), bounding p <= 256.
#include "fb_kernels.h"
#include "fb_sm100.cuh"

namespace fb {

template <int D, int RP, bool DENSE, bool BF16>
struct FwdCfg {
  static constexpr int kRows = kTileRows;
  static constexpr int kSW = swizzle_bytes(D);
  static constexpr int kAtomCols = kSW / 2;
  static constexpr int kAtoms = D / kAtomCols;
  static constexpr int kQBytes = kRows * D * 2;
  static constexpr int kPanelBytes = kRows * 32;  // 16 columns, SW32
  static constexpr int kUBytes = RP * kPanelBytes;
  static constexpr int kKBytes = kQBytes + kUBytes;
  static constexpr int kVBytes = kQBytes;
  static constexpr int kBiasBytes = DENSE ? kRows * 128 * 2 : 0;
  static constexpr int kSlotRaw =
      kKBytes > kVBytes ? (kKBytes > kBiasBytes ? kKBytes : kBiasBytes)
                        : (kVBytes > kBiasBytes ? kVBytes : kBiasBytes);
  static constexpr int kSlotBytes = (kSlotRaw + 1023) / 1024 * 1024;
  static constexpr int kIPS = DENSE ? 4 : 2;  // ring items per KV step
  static constexpr int kQRegion = (2 * (kQBytes + kUBytes) + 1023) / 1024 * 1024;
  static constexpr int kBarBytes = 256;
  static constexpr int kBudget = 232448 - 1024 - kBarBytes;
  static constexpr int kSlotsFit = (kBudget - kQRegion) / kSlotBytes;
  static constexpr int kSlots = kSlotsFit > 8 ? 8 : kSlotsFit;
  static constexpr int kSmemBytes = 1024 + kQRegion + kSlots * kSlotBytes + kBarBytes;
  static constexpr int kThreads = 384;
  static constexpr int kTmemCols = 512;
  static_assert(D == 32 || D == 64 || D == 128, "head dim");
  static_assert(kSlots >= 2, "shared memory ring too small");
};

// P split: the first kSplitPairs packed columns (96 keys) feed PV K-steps 0..kSplitSteps-1
constexpr int kSplitPairs = 48, kSplitSteps = 6;

struct FwdBars {
  uint64_t q_full;
  uint64_t s_full[2];
  uint64_t p_ready[2];
  uint64_t p_part[2];  // first kSplitPairs bf16 pairs of P written (PV K-steps 0..5 may start)
  uint64_t o_final[2];
  uint64_t slot_full[8];
  uint64_t slot_empty[8];
  uint32_t tmem_base;
};

// Blocks processed by the two tiles of query pair `pair`.
__device__ __forceinline__ void fwd_block_counts(const FwdParams& p, int pair, int& n0, int& n1) {
  const int nkv = (p.M + kTileRows - 1) / kTileRows;
  if (p.causal) {
    const int r0 = pair * 2 * kTileRows;
    n0 = min(nkv, r0 / kTileRows + 1);
    n1 = min(nkv, r0 / kTileRows + 2);
  } else {
    n0 = n1 = nkv;
  }
}

template <int D, int RP, bool DENSE, bool BF16>
__global__ void __launch_bounds__(384, 1)
    fb_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_uq,
                  const __grid_constant__ CUtensorMap tm_uk,
                  const __grid_constant__ CUtensorMap tm_bias, const FwdParams p) {
  using Cfg = FwdCfg<D, RP, DENSE, BF16>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t q_base = sbase;                             // Q0 | Q1
  const uint32_t u_base = sbase + 2 * Cfg::kQBytes;          // U0 | U1
  const uint32_t ring_base = sbase + Cfg::kQRegion;          // slots
  FwdBars* bars = reinterpret_cast<FwdBars*>(smem + Cfg::kQRegion + Cfg::kSlots * Cfg::kSlotBytes);

  const int warp = warp_id();
  const int lane = lane_id();

  // ---- work decomposition: head-major so the ~148 resident CTAs share the
  // K/V of 2-3 heads through L2; within a head, longest (causal) pairs first.
  const int bh = blockIdx.x / p.num_pairs;
  int pair = blockIdx.x % p.num_pairs;
  if (p.causal) pair = p.num_pairs - 1 - pair;
  const int h = bh / p.B;  // (head, batch) order: a head's batches are adjacent
  const int b = bh % p.B;
  const int row0 = pair * 2 * kTileRows;
  int n0, n1;
  fwd_block_counts(p, pair, n0, n1);

  // ---- setup
  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    if (RP > 0) {
      tma_prefetch(&tm_uq);
      tma_prefetch(&tm_uk);
    }
    if (DENSE) tma_prefetch(&tm_bias);
    mbar_init(&bars->q_full, 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bars->s_full[t], 1);
      mbar_init(&bars->p_ready[t], 4);
      mbar_init(&bars->p_part[t], 4);
      mbar_init(&bars->o_final[t], 1);
    }
    for (int s = 0; s < Cfg::kSlots; ++s) {
      mbar_init(&bars->slot_full[s], 1);
      mbar_init(&bars->slot_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<Cfg::kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  // KV blocks are visited in REVERSE order (step s -> block j = n1-1-s): for a
  // causal ALiBi-style bias the diagonal block holds the row max, so the lazy
  // rescale almost never fires afterwards.  Tile 1 can own one more block than
  // tile 0 (causal); tile 0 joins at step d = n1 - n0.
  // Ring items of step s: K, [B0 if s >= d], B1, V (dense) or K, V.
  const int dlt = n1 - n0;
  auto step_base = [&](int st) { return DENSE ? st * Cfg::kIPS - min(st, dlt) : st * Cfg::kIPS; };
  auto step_items = [&](int st) { return (DENSE && st < dlt) ? Cfg::kIPS - 1 : Cfg::kIPS; };

  if (warp >= 8) {
  regs_dec<80>();
  if (warp == 8) {
    // =========================== TMA producer
    if (lane == 0) {
      const int hq = p.uq_hb ? 0 : h, bq = p.uq_bb ? 0 : b;
      const int hk = p.uk_hb ? 0 : h, bk = p.uk_bb ? 0 : b;
      const int hb_ = p.bias_hb ? 0 : h, bb_ = p.bias_bb ? 0 : b;
      mbar_arrive_expect_tx(&bars->q_full, 2 * (Cfg::kQBytes + Cfg::kUBytes));
      for (int t = 0; t < 2; ++t) {
        for (int a = 0; a < Cfg::kAtoms; ++a)
          tma_load_4d(smem + t * Cfg::kQBytes + a * kTileRows * Cfg::kSW, &tm_q, &bars->q_full,
                      a * Cfg::kAtomCols, row0 + t * kTileRows, h, b);
        for (int pn = 0; pn < RP; ++pn)
          tma_load_4d(smem + 2 * Cfg::kQBytes + t * Cfg::kUBytes + pn * Cfg::kPanelBytes, &tm_uq,
                      &bars->q_full, pn * 16, row0 + t * kTileRows, hq, bq);
      }
      int item = 0;
      for (int st = 0; st < n1; ++st) {
        const int kv0 = (n1 - 1 - st) * kTileRows;
        const int npos = step_items(st);
        for (int pos = 0; pos < npos; ++pos, ++item) {
          const int slot = item % Cfg::kSlots;
          const int use = item / Cfg::kSlots;
          if (use > 0) mbar_wait(&bars->slot_empty[slot], (use - 1) & 1);
          trace(p.trace, p.trace_cta, 4, item);
          uint8_t* dst = smem + Cfg::kQRegion + slot * Cfg::kSlotBytes;
          uint64_t* fb_ = &bars->slot_full[slot];
          if (pos == 0) {  // K (+ fk panels)
            mbar_arrive_expect_tx(fb_, Cfg::kKBytes);
            for (int a = 0; a < Cfg::kAtoms; ++a)
              tma_load_4d(dst + a * kTileRows * Cfg::kSW, &tm_k, fb_, a * Cfg::kAtomCols, kv0, h, b);
            for (int pn = 0; pn < RP; ++pn)
              tma_load_4d(dst + Cfg::kQBytes + pn * Cfg::kPanelBytes, &tm_uk, fb_, pn * 16, kv0, hk, bk);
          } else if (pos == npos - 1) {  // V
            mbar_arrive_expect_tx(fb_, Cfg::kVBytes);
            for (int a = 0; a < Cfg::kAtoms; ++a)
              tma_load_4d(dst + a * kTileRows * Cfg::kSW, &tm_v, fb_, a * Cfg::kAtomCols, kv0, h, b);
          } else {  // dense bias tile for tile t
            const int t = (npos == Cfg::kIPS) ? pos - 1 : 1;
            mbar_arrive_expect_tx(fb_, Cfg::kBiasBytes);
            for (int half = 0; half < 2; ++half)
              tma_load_4d(dst + half * kTileRows * 128, &tm_bias, fb_, kv0 + half * 64,
                          row0 + t * kTileRows, hb_, bb_);
          }
        }
      }
    }
  } else if (warp == 9) {
    // =========================== MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc(128, 128, false, false, BF16);
      constexpr uint32_t idesc_pv = make_idesc(128, D, false, true, BF16);
      auto slot_addr = [&](int item) { return ring_base + (item % Cfg::kSlots) * Cfg::kSlotBytes; };
      auto wait_full = [&](int item) {
        mbar_wait(&bars->slot_full[item % Cfg::kSlots], (item / Cfg::kSlots) & 1);
        tc_fence_after();
      };
      auto release = [&](int item) {
        uint64_t* e = &bars->slot_empty[item % Cfg::kSlots];
        mbar_arrive_cnt(e, 3);
        tc_commit(e);
      };
      auto issue_s = [&](int t, int st) {
        trace(p.trace, p.trace_cta, 2, t * 1024 + st);
        const uint32_t d_s = tmem + t * 128;
        const uint32_t qa = q_base + t * Cfg::kQBytes;
        const uint32_t kb = slot_addr(step_base(st));
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(d_s, kmajor_desc(qa, kTileRows, Cfg::kSW, kk * 16),
                 kmajor_desc(kb, kTileRows, Cfg::kSW, kk * 16), idesc_qk, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int pn = 0; pn < RP; ++pn)
          mma_ss(d_s, make_sdesc(u_base + t * Cfg::kUBytes + pn * Cfg::kPanelBytes, 16, 256, 6),
                 make_sdesc(kb + Cfg::kQBytes + pn * Cfg::kPanelBytes, 16, 256, 6), idesc_qk, 1u);
        tc_commit(&bars->s_full[t]);
      };
      // PV in two parts (FA4-style split arrive): K-steps over the first 96 keys
      // start once the softmax has written that part of P, the last 32 after p_ready
      auto issue_pv = [&](int t, int vitem, bool acc, uint32_t parity) {
        const uint32_t d_o = tmem + 256 + t * D;
        const uint32_t a_p = tmem + t * 128;
        const uint32_t vb = slot_addr(vitem);
        mbar_wait(&bars->p_part[t], parity);
        tc_fence_after();
        trace(p.trace, p.trace_cta, 3, t * 1024 + vitem);
#pragma unroll
        for (int kk = 0; kk < kSplitSteps; ++kk)
          mma_ts(d_o, a_p + kk * 8, mnmajor_desc(vb, kTileRows, Cfg::kSW, kk * 16), idesc_pv,
                 (acc || kk > 0) ? 1u : 0u);
        mbar_wait(&bars->p_ready[t], parity);
        tc_fence_after();
#pragma unroll
        for (int kk = kSplitSteps; kk < kTileRows / 16; ++kk)
          mma_ts(d_o, a_p + kk * 8, mnmajor_desc(vb, kTileRows, Cfg::kSW, kk * 16), idesc_pv, 1u);
      };
      auto v_item = [&](int st) { return step_base(st) + step_items(st) - 1; };

      mbar_wait(&bars->q_full, 0);
      tc_fence_after();
      // prologue: tile 1's first S, and tile 0's first S (same step when d == 0)
      wait_full(step_base(0));
      if (dlt == 0) issue_s(0, 0);
      issue_s(1, 0);
      release(step_base(0));
      if (dlt == 1 && n1 > 1) {
        wait_full(step_base(1));
        issue_s(0, 1);
      }
      for (int st = 0; st < n1; ++st) {
        const int vi = v_item(st);
        wait_full(vi);
        if (st >= dlt) {
          issue_pv(0, vi, st > dlt, (st - dlt) & 1);
          if (st + 1 < n1) {
            wait_full(step_base(st + 1));
            issue_s(0, st + 1);
          } else {
            tc_commit(&bars->o_final[0]);
          }
        }
        issue_pv(1, vi, st > 0, st & 1);
        release(vi);
        if (st + 1 < n1) {
          wait_full(step_base(st + 1));
          issue_s(1, st + 1);
          release(step_base(st + 1));
        } else {
          tc_commit(&bars->o_final[1]);
        }
      }
    }
  }
  } else {
    regs_inc<208>();
    // =========================== softmax / correction / epilogue (warps 0..7)
    const int t = warp >> 2;
    const int r = threadIdx.x & 127;  // row within tile == TMEM lane
    const int n_t = t == 0 ? n0 : n1;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_off + t * 128;
    const uint32_t t_o = tmem + lane_off + 256 + t * D;
    const int row = row0 + t * kTileRows + r;
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;

    for (int it = 0; it < n_t; ++it) {
      const int st = it + (t == 0 ? dlt : 0);  // global step
      const int kv0 = (n1 - 1 - st) * kTileRows;
      float x[128];
      mbar_wait(&bars->s_full[t], it & 1);
      tc_fence_after();
      if (r == 0) trace(p.trace, p.trace_cta, 5, t * 1024 + it);
      {
        uint32_t* xr = reinterpret_cast<uint32_t*>(x);
        tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(xr + 0));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(xr + 32));
        tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(xr + 64));
        tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(xr + 96));
        tmem_wait_ld();
      }
      // x holds raw Q'K'^T (DENSE: already scaled to log2 units with the bias added)
      if constexpr (DENSE) {
        const int item = step_base(st) + 1 + (t == 1 && st >= dlt ? 1 : 0);
        const int slot = item % Cfg::kSlots;
        mbar_wait(&bars->slot_full[slot], (item / Cfg::kSlots) & 1);
        const uint8_t* bt = smem + Cfg::kQRegion + slot * Cfg::kSlotBytes;
        constexpr float kLog2e = 1.4426950408889634f;
#pragma unroll
        for (int c8 = 0; c8 < 16; ++c8) {  // 16-byte chunks of the 256-byte bias row
          const int half = c8 >> 3, ch = c8 & 7;
          const uint4 v = *reinterpret_cast<const uint4*>(bt + half * kTileRows * 128 + r * 128 +
                                                          ((ch ^ (r & 7)) << 4));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 bb = unpack2<BF16>(w[e]);
            const int c = c8 * 8 + e * 2;
            const float2 r2 = ffma2(make_float2(x[c], x[c + 1]), make_float2(sl2, sl2),
                                    make_float2(bb.x * kLog2e, bb.y * kLog2e));
            x[c] = r2.x;
            x[c + 1] = r2.y;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->slot_empty[slot]);
      }
      const bool edge = (kv0 + kTileRows > p.M) || (p.causal && kv0 + kTileRows > row0 + t * kTileRows);
      if (edge) {
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          const int col = kv0 + c;
          if (col >= p.M || (p.causal && col > row)) x[c] = -INFINITY;
        }
      }
      // row max: a 3-input max tree over independent partials
      float mx;
      {
        float m4[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float a = x[32 * g];
#pragma unroll
          for (int c = 1; c < 31; c += 2) a = fmax3(a, x[32 * g + c], x[32 * g + c + 1]);
          m4[g] = fmaxf(a, x[32 * g + 31]);
        }
        mx = fmax3(fmaxf(m4[0], m4[1]), m4[2], m4[3]);
      }
      const float m_new = DENSE ? fmaxf(m_run, mx) : fmaxf(m_run, mx * sl2);
      // lazy rescale: move the running max only when it grows by > 8 (log2 units)
      bool need = false;
      float alpha = 1.0f;
      if (it == 0) {
        m_run = m_new;
      } else if (m_new > m_run + 8.0f) {
        need = true;
        alpha = ex2(m_run - m_new);
        m_run = m_new;
      }
      // O_t was last written by PV_t(previous), which completed before S_t(this)
      // (commit order): rescale it now, before any part of P is released to PV_t(this)
      if (__any_sync(0xffffffffu, need)) {
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(t_o + c0, o);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 v2 = fmul2(make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])),
                                    make_float2(alpha, alpha));
            o[c] = __float_as_uint(v2.x);
            o[c + 1] = __float_as_uint(v2.y);
          }
          tmem_st32(t_o + c0, o);
        }
        tmem_wait_st();
      }
      // p = 2^(x*sl2 - m): packed FFMA2, MUFU ex2, packed FADD2 partial sums
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      {
        const float2 mul = DENSE ? make_float2(1.f, 1.f) : make_float2(sl2, sl2);
        // a row whose keys so far are all -inf (dense bias masking whole trailing key
        // blocks, visited first) has m_run = -inf: subtract 0 so p = 2^-inf = 0, not NaN
        const float m_use = m_run == -INFINITY ? 0.f : m_run;
        const float2 neg = make_float2(-m_use, -m_use);
        uint32_t pk[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const float2 e2 = ffma2(make_float2(x[2 * c], x[2 * c + 1]), mul, neg);
          // FB_POLY_NUM pairs in 8 go through the FMA-pipe polynomial, the rest through MUFU
          const float2 p2 = poly_pair_fwd<D>(c) ? ex2_poly2(e2) : make_float2(ex2(e2.x), ex2(e2.y));
          acc[c & 3] = fadd2(acc[c & 3], p2);
          pk[c] = pack2<BF16>(p2.x, p2.y);
          if (c == kSplitPairs - 1) {  // first 3/4 of P -> TMEM, release PV K-steps 0..5
            tmem_st32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(pk + 0));
            tmem_st16(t_s + 32, *reinterpret_cast<uint32_t(*)[16]>(pk + 32));
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->p_part[t]);
          }
        }
        tmem_st16(t_s + 48, *reinterpret_cast<uint32_t(*)[16]>(pk + 48));
      }
      const float2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
      const float2 s4 = fadd2(s01, s23);
      l_run = l_run * alpha + (s4.x + s4.y);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (r == 0) trace(p.trace, p.trace_cta, 6, t * 1024 + it);
      if (lane == 0) trace(p.trace, p.trace_cta, 22 + (warp & 3), t * 1024 + it);
      if (lane == 0) mbar_arrive(&bars->p_ready[t]);
    }

    // ---- epilogue: O / l -> global, LSE
    if (n_t > 0) {
      mbar_wait(&bars->o_final[t], 0);
      tc_fence_after();
    }
    const float inv_l = l_run > 0.f ? 1.0f / l_run : 0.f;
    const bool valid = row < p.N;
    typedef typename std::conditional<BF16, __nv_bfloat16, __half>::type elem_t;
    elem_t* orow = reinterpret_cast<elem_t*>(p.o) + static_cast<int64_t>(b) * p.o_sb +
                   static_cast<int64_t>(h) * p.o_sh + static_cast<int64_t>(row) * p.o_sn;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t o[32];
      tmem_ld32(t_o + c0, o);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        pk[c] = pack2<BF16>(__uint_as_float(o[2 * c]) * inv_l, __uint_as_float(o[2 * c + 1]) * inv_l);
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          dst[q4] = make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
      }
    }
    if (valid && p.lse != nullptr) {
      // fully masked row: LSE = +inf makes the backward's p = exp(s - lse) exactly 0
      const float lse = l_run > 0.f ? (m_run + __log2f(l_run)) * 0.6931471805599453f : INFINITY;
      p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + row] = lse;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// ------------------------------------------------------------------ launch
template <int D, int RP, bool DENSE, bool BF16>
static cudaError_t launch_fwd_t(const FwdMaps& maps, const FwdParams& p, cudaStream_t stream) {
  using Cfg = FwdCfg<D, RP, DENSE, BF16>;
  auto kern = fb_fwd_kernel<D, RP, DENSE, BF16>;
  static std::atomic<uint64_t> attr_mask{0};
  cudaError_t e = smem_attr_once(attr_mask, reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  const int grid = p.num_pairs * p.B * p.H;
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, stream>>>(maps.q, maps.k, maps.v, maps.uq, maps.uk,
                                                          maps.bias, p);
  return cudaGetLastError();
}

template <int D, bool BF16>
static cudaError_t dispatch_rp(int rp, bool dense, const FwdMaps& maps, const FwdParams& p,
                               cudaStream_t s) {
  if (dense) {
    if (rp != 0) return cudaErrorInvalidValue;
    return launch_fwd_t<D, 0, true, BF16>(maps, p, s);
  }
  switch (rp) {
    case 0: return launch_fwd_t<D, 0, false, BF16>(maps, p, s);
    case 1: return launch_fwd_t<D, 1, false, BF16>(maps, p, s);
    case 2: return launch_fwd_t<D, 2, false, BF16>(maps, p, s);
    case 3: return launch_fwd_t<D, 3, false, BF16>(maps, p, s);
    case 4: return launch_fwd_t<D, 4, false, BF16>(maps, p, s);
  }
  if constexpr (D <= 64) {  // wider factor panels (up to 128 split columns) fit next to small heads
    switch (rp) {
      case 5: return launch_fwd_t<D, 5, false, BF16>(maps, p, s);
      case 6: return launch_fwd_t<D, 6, false, BF16>(maps, p, s);
      case 7: return launch_fwd_t<D, 7, false, BF16>(maps, p, s);
      case 8: return launch_fwd_t<D, 8, false, BF16>(maps, p, s);
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fwd_sm100(int d, int rp, bool dense, bool bf16, const FwdMaps& maps,
                             const FwdParams& p, cudaStream_t s) {
  if (bf16) {
    if (d == 32) return dispatch_rp<32, true>(rp, dense, maps, p, s);
    if (d == 64) return dispatch_rp<64, true>(rp, dense, maps, p, s);
    if (d == 128) return dispatch_rp<128, true>(rp, dense, maps, p, s);
  } else {
    if (d == 32) return dispatch_rp<32, false>(rp, dense, maps, p, s);
    if (d == 64) return dispatch_rp<64, false>(rp, dense, maps, p, s);
    if (d == 128) return dispatch_rp<128, false>(rp, dense, maps, p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace fb
