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

struct FwdBars {
  uint64_t q_full;
  uint64_t s_full[2];
  uint64_t p_ready[2];
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

  // item bookkeeping shared by all roles: step j holds K, [B0 if j<n0], B1, V (dense)
  // or K, V (otherwise).  Only the last step of tile 0 can be missing.
  auto step_base = [&](int j) { return j <= n0 ? j * Cfg::kIPS : n0 * Cfg::kIPS + (j - n0) * (Cfg::kIPS - 1); };

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
      for (int j = 0; j < n1; ++j) {
        const int kv0 = j * kTileRows;
        const int npos = (DENSE && j >= n0) ? Cfg::kIPS - 1 : Cfg::kIPS;
        for (int pos = 0; pos < npos; ++pos, ++item) {
          const int slot = item % Cfg::kSlots;
          const int use = item / Cfg::kSlots;
          if (use > 0) mbar_wait(&bars->slot_empty[slot], (use - 1) & 1);
          trace(p.trace, p.trace_cta, 20, item);
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
      };
      auto release = [&](int item) {
        uint64_t* e = &bars->slot_empty[item % Cfg::kSlots];
        mbar_arrive_cnt(e, 3);
        tc_commit(e);
      };
      auto issue_s = [&](int t, int kitem) {
        trace(p.trace, p.trace_cta, 2, t * 4096 + kitem);
        const uint32_t d_s = tmem + t * 128;
        const uint32_t qa = q_base + t * Cfg::kQBytes;
        const uint32_t kb = slot_addr(kitem);
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
      auto issue_pv = [&](int t, int vitem, int j) {
        trace(p.trace, p.trace_cta, 3, t * 4096 + j);
        const uint32_t d_o = tmem + 256 + t * D;
        const uint32_t a_p = tmem + t * 128;
        const uint32_t vb = slot_addr(vitem);
#pragma unroll
        for (int kk = 0; kk < kTileRows / 16; ++kk)
          mma_ts(d_o, a_p + kk * 8, mnmajor_desc(vb, kTileRows, Cfg::kSW, kk * 16), idesc_pv,
                 (j > 0 || kk > 0) ? 1u : 0u);
      };
      auto k_item = [&](int j) { return step_base(j); };
      auto v_item = [&](int j) {
        const int npos = (DENSE && j >= n0) ? Cfg::kIPS - 1 : Cfg::kIPS;
        return step_base(j) + npos - 1;
      };

      mbar_wait(&bars->q_full, 0);
      tc_fence_after();
      // prologue: S0(0), S1(0)
      wait_full(k_item(0));
      tc_fence_after();
      if (n0 > 0) issue_s(0, k_item(0));
      issue_s(1, k_item(0));
      release(k_item(0));
      for (int j = 0; j < n1; ++j) {
        const int vi = v_item(j);
        wait_full(vi);
        tc_fence_after();
        if (j < n0) {
          mbar_wait(&bars->p_ready[0], j & 1);
          tc_fence_after();
          issue_pv(0, vi, j);
          if (j + 1 < n0) {
            wait_full(k_item(j + 1));
            tc_fence_after();
            issue_s(0, k_item(j + 1));
          } else {
            tc_commit(&bars->o_final[0]);
          }
        }
        mbar_wait(&bars->p_ready[1], j & 1);
        tc_fence_after();
        issue_pv(1, vi, j);
        release(vi);
        if (j + 1 < n1) {
          wait_full(k_item(j + 1));
          tc_fence_after();
          issue_s(1, k_item(j + 1));
          release(k_item(j + 1));
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

    for (int j = 0; j < n_t; ++j) {
      const int kv0 = j * kTileRows;
      float x[128];
      mbar_wait(&bars->s_full[t], j & 1);
      tc_fence_after();
      if (r == 0) trace(p.trace, p.trace_cta, 10, t * 4096 + j);
      {
        uint32_t* xr = reinterpret_cast<uint32_t*>(x);
        tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(xr + 0));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(xr + 32));
        tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(xr + 64));
        tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(xr + 96));
        tmem_wait_ld();
      }
      if constexpr (DENSE) {
        // this tile's bias item for step j
        const int item = step_base(j) + 1 + (t == 1 && j < n0 ? 1 : 0);
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
            x[c] = fmaf(x[c], sl2, bb.x * kLog2e);
            x[c + 1] = fmaf(x[c + 1], sl2, bb.y * kLog2e);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->slot_empty[slot]);
      } else {
#pragma unroll
        for (int c = 0; c < 128; ++c) x[c] *= sl2;
      }
      const bool edge = (kv0 + kTileRows > p.M) || (p.causal && kv0 + kTileRows > row0 + t * kTileRows);
      if (edge) {
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          const int col = kv0 + c;
          if (col >= p.M || (p.causal && col > row)) x[c] = -INFINITY;
        }
      }
      float mx = x[0];
#pragma unroll
      for (int c = 1; c < 128; ++c) mx = fmaxf(mx, x[c]);
      const float m_new = fmaxf(m_run, mx);
      // lazy rescale: move the running max only when it grows by > 8 (log2 units)
      bool need = false;
      float alpha = 1.0f;
      if (j == 0) {
        m_run = m_new;
      } else if (m_new > m_run + 8.0f) {
        need = true;
        alpha = ex2(m_run - m_new);
        m_run = m_new;
      }
      float sum = 0.f;
      {
        uint32_t pk[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const float p0 = ex2(x[2 * c] - m_run);
          const float p1 = ex2(x[2 * c + 1] - m_run);
          sum += p0 + p1;
          pk[c] = pack2<BF16>(p0, p1);
        }
        tmem_st32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(pk + 0));
        tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(pk + 32));
      }
      l_run = l_run * alpha + sum;
      // O_t was last written by PV_t(j-1), which completed before S_t(j) (commit order)
      if (__any_sync(0xffffffffu, need)) {
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(t_o + c0, o);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
          tmem_st32(t_o + c0, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (r == 0) trace(p.trace, p.trace_cta, 11, t * 4096 + j);
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
      const float lse = (m_run + __log2f(l_run)) * 0.6931471805599453f;
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
  static bool attr_done = false;  // set once per instantiation (host-side, benign race)
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
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
