// attn_bwd.cu — block-diagonal varlen attention backward for sm_100a.
//
// Gradients of vlasim::packed_attention — the reference has no
// backward; the closed form is SURVEY.md §8(c):
//   P = exp(S·scale − LSE), dV = Pᵀ dO, dP = dO Vᵀ, dS = P ∘ (dP − D), D = rowsum(dO ∘ O),
//   dQ = scale · dS K, dK = scale · dSᵀ Q.
//
// Launches:
//   memset      zero the fp32 dQ accumulator
//   k_bwd_pre   D = rowsum(dO∘O), LSE → log2 domain, per-token visible spans    [HBM-bound]
//   k_bwd_main  persistent: each CTA loops over work items = (128-key tile on the global grid,
//               KV head).  Per item, K and V stay in smem; the q heads of the group × the
//               128-row Q tiles of the tile's visible query range stream through a TMA ring
//               (tile skipping: queries outside [q_lo, q_hi) are never loaded or multiplied).
//   k_bwd_post  dQ = bf16(scale · dQacc), optionally scattered through row_map
//
// k_bwd_main warp roles (448 threads):
//   warps 0-7   "softmax": warp w owns key rows 32·(w%4).. (TMEM lane quadrant w%4) and query
//               columns [64·(w/4), +64).  Phase A: S → Pᵀ (bf16, written back into the S
//               columns it read).  Phase B: dP → dSᵀ (bf16, SWIZZLE_128B smem, read back as the
//               K-major A of dK and the MN-major A of dQ).  Item end: dK/dV epilogue.
//   warps 8-11  dQ drain: TMEM dQ rows → red.global.add.v4.f32 into the fp32 accumulator.
//   warp 12     TMA producer.   warp 13  TMEM allocator + tcgen05.mma issuer.
// TMEM (512 columns): S/P [0,128) · dP/dQ [128,256) · dV [256,256+HD) · dK after dV.
// Issue order per iteration (FA4-style): dV, dK, S(next), dQ, dP(next) — the next S is
// computed while the drain warps empty dQ and the softmax warps run phase A of the next
// iteration.  The P→S and dP→dQ column aliasing relies on tcgen05.mma executing in issue
// order.
#include <cfloat>
#include <climits>

#include "attn_common.cuh"
#include "common.hpp"
#include "sm100.cuh"

using namespace vlasim_dev;

namespace vlasim_host {
int validate_attn_args(const vlasim_attn_args* a, bool fp8);
}

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// ------------------------------------------------------------------ pre / post
// D[h][t] = Σ_c dO·O (fp32) and LSE → log2 domain; 16-byte loads, HD/8 lanes per (t, h) row.
// Lane 0 of every (t, head 0) row also writes the token's visible spans (attn_common.cuh):
// rows[t] = visible keys of query t, cols[t] = queries that see key t.
template <int HD>
__global__ void k_bwd_pre(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                          const float* __restrict__ lse, float* __restrict__ lse2, float* __restrict__ dsum,
                          int2* __restrict__ rows_span, int2* __restrict__ cols_span, const int32_t* __restrict__ cu,
                          const int32_t* __restrict__ prefix, int nseq, int mask, int T, int Tp, int H) {
  constexpr int LPR = HD / 8;  // lanes per row (8 bf16 per lane)
  const int64_t gt = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t row = gt / LPR;
  const int sub = int(gt % LPR);
  const bool ok = row < int64_t(T) * H;
  float acc = 0.f;
  if (ok) {
    const uint4 a = *reinterpret_cast<const uint4*>(o + row * HD + sub * 8);
    const uint4 b = *reinterpret_cast<const uint4*>(dout + row * HD + sub * 8);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __bfloat1622float2(pa[i]), y = __bfloat1622float2(pb[i]);
      acc += x.x * y.x + x.y * y.y;
    }
  }
#pragma unroll
  for (int off = LPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (ok && sub == 0) {
    const int t = int(row / H), h = int(row % H);
    dsum[int64_t(h) * Tp + t] = acc;
    lse2[int64_t(h) * Tp + t] = lse[int64_t(h) * T + t] * kLog2e;
    if (h == 0) {
      const RowSpan r = row_span(cu, prefix, nseq, mask, t, T);
      const RowSpan c = key_span(cu, prefix, nseq, mask, t, T);
      rows_span[t] = make_int2(r.lo, r.hi);
      cols_span[t] = make_int2(c.lo, c.hi);
    }
  }
}

// dQ = bf16(scale · dQacc), written to row row_map[t] (fused scatter) or t.
template <int HD>
__global__ void k_bwd_post(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                           const int32_t* __restrict__ row_map, int64_t rows, int H, float scale) {
  constexpr int LPR = HD / 8;
  const int64_t gt = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t row = gt / LPR;  // (t, h) row
  const int sub = int(gt % LPR);
  if (row >= rows) return;
  const int64_t t = row / H, h = row % H;
  const int64_t dst_t = row_map ? int64_t(__ldg(row_map + t)) : t;
  const float4 a = __ldcs(reinterpret_cast<const float4*>(acc + row * HD + sub * 8));
  const float4 b = __ldcs(reinterpret_cast<const float4*>(acc + row * HD + sub * 8 + 4));
  uint4 r;
  r.x = pack_bf16x2(a.x * scale, a.y * scale);
  r.y = pack_bf16x2(a.z * scale, a.w * scale);
  r.z = pack_bf16x2(b.x * scale, b.y * scale);
  r.w = pack_bf16x2(b.z * scale, b.w * scale);
  *reinterpret_cast<uint4*>(dq + (dst_t * H + h) * HD + sub * 8) = r;
}

// ------------------------------------------------------------------ main kernel
struct BwdParams {
  float* dq_acc;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  const int32_t* row_map;  // packed row → output row for dK/dV (NULL: identity)
  const float* lse2;       // [H, Tp] log2-domain LSE
  const float* dsum;       // [H, Tp] rowsum(dO ∘ O)
  const int2* rows_span;   // [T] visible keys of query t
  const int2* cols_span;   // [T] queries that see key t
  int T, Tp, H, Hkv, num_items;
  float scale_log2, scale;
};

template <int HD>
struct BwdCfg {
  static constexpr int BK = 128, BQ = 128;
  static constexpr int TILE = 128 * HD * 2;  // one 128-row bf16 tile (K, V, Q or dO)
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;                 // Q ring: stage s at OFF_Q + s*TILE
  static constexpr int OFF_DO = OFF_Q + 2 * TILE;        // dO: single buffer
  static constexpr int OFF_DS = OFF_DO + TILE;           // dSᵀ [128 keys × 128 q] bf16
  static constexpr int VEC = 544;                        // 132 floats (16-B aligned window) + pad
  static constexpr int OFF_LSE = OFF_DS + 128 * 128 * 2;  // lse2 [2][VEC]
  static constexpr int OFF_DSUM = OFF_LSE + 2 * VEC;      // D [VEC]
  static constexpr int OFF_BAR = OFF_DSUM + VEC;
  static constexpr int NUM_BARS = 16;
  static constexpr int SMEM_USED = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int SMEM = SMEM_USED + 1024;  // + alignment slack for the 1 KB swizzle atoms
  static constexpr uint32_t S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 256 + HD;
  static constexpr int THREADS = 448;
  static_assert(DK_COL + HD <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
};

// Work item i → (key tile, kv head); the q range comes from the precomputed key spans.
struct BwdItem {
  int k0, kh, q_lo, nq, iters;
};
__device__ __forceinline__ BwdItem bwd_item(const BwdParams& p, int i) {
  BwdItem it;
  it.kh = i % p.Hkv;
  it.k0 = (i / p.Hkv) * 128;
  const int2 first = __ldg(p.cols_span + it.k0);
  const int2 last = __ldg(p.cols_span + min(it.k0 + 127, p.T - 1));
  it.q_lo = first.x;
  it.nq = max(0, (last.y - first.x + 127) / 128);
  it.iters = it.nq * (p.H / p.Hkv);
  return it;
}

template <int HD>
__global__ void __launch_bounds__(448, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const BwdParams p) {
  using Cfg = BwdCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* bar_kv_full = bars + 0;
  uint64_t* bar_kv_empty = bars + 1;
  uint64_t* bar_q_full = bars + 2;   // [2]
  uint64_t* bar_q_empty = bars + 4;  // [2]
  uint64_t* bar_do_full = bars + 6;
  uint64_t* bar_do_empty = bars + 7;
  uint64_t* bar_s_full = bars + 8;
  uint64_t* bar_dp_full = bars + 9;
  uint64_t* bar_p_full = bars + 10;    // 256 arrivals
  uint64_t* bar_dq_full = bars + 11;
  uint64_t* bar_dq_empty = bars + 12;  // 128 arrivals
  uint64_t* bar_dkv_full = bars + 13;
  uint64_t* bar_dkv_empty = bars + 14;  // 256 arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int group = p.H / p.Hkv;

  if (tid == 0) {
    mbar_init(bar_kv_full, 1);
    mbar_init(bar_kv_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_q_full[s], 1);
      mbar_init(&bar_q_empty[s], 1);
    }
    mbar_init(bar_do_full, 1);
    mbar_init(bar_do_empty, 1);
    mbar_init(bar_s_full, 1);
    mbar_init(bar_dp_full, 1);
    mbar_init(bar_p_full, 256);
    mbar_init(bar_dq_full, 1);
    mbar_init(bar_dq_empty, 128);
    mbar_init(bar_dkv_full, 1);
    mbar_init(bar_dkv_empty, 256);
    fence_barrier_init();
  }
  if (warp == 13) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 12) {
    // ================================================ TMA producer
    if (lane == 0) {
      int G = 0, k = 0;
      for (int i = blockIdx.x; i < p.num_items; i += gridDim.x) {
        const BwdItem itm = bwd_item(p, i);
        if (itm.iters == 0) continue;
        for (int it = 0; it < itm.iters; ++it, ++G) {
          const int h = itm.kh * group + it / itm.nq;
          const int qb = itm.q_lo + (it % itm.nq) * Cfg::BQ;
          const int qs = G & 1;
          if (G >= 2) mbar_wait(&bar_q_empty[qs], ((G >> 1) - 1) & 1);
          uint8_t* sq = smem + Cfg::OFF_Q + qs * Cfg::TILE;
          mbar_expect_tx(&bar_q_full[qs], Cfg::TILE + 528);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c) tma_load_2d(sq + c * 16384, &tmQ, h * HD + c * 64, qb, &bar_q_full[qs]);
          bulk_load(smem + Cfg::OFF_LSE + qs * Cfg::VEC, p.lse2 + int64_t(h) * p.Tp + (qb & ~3), 528, &bar_q_full[qs]);
          if (it == 0) {
            if (k > 0) mbar_wait(bar_kv_empty, (k - 1) & 1);
            mbar_expect_tx(bar_kv_full, 2 * Cfg::TILE);
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
              tma_load_2d(smem + Cfg::OFF_K + c * 16384, &tmK, itm.kh * HD + c * 64, itm.k0, bar_kv_full);
              tma_load_2d(smem + Cfg::OFF_V + c * 16384, &tmV, itm.kh * HD + c * 64, itm.k0, bar_kv_full);
            }
          }
          if (G >= 1) mbar_wait(bar_do_empty, (G - 1) & 1);
          mbar_expect_tx(bar_do_full, Cfg::TILE + 528);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_2d(smem + Cfg::OFF_DO + c * 16384, &tmdO, h * HD + c * 64, qb, bar_do_full);
          bulk_load(smem + Cfg::OFF_DSUM, p.dsum + int64_t(h) * p.Tp + (qb & ~3), 528, bar_do_full);
        }
        ++k;
      }
    }
  } else if (warp == 13) {
    // ================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_kk = make_idesc_bf16(128, 128, false, false);  // S, dP
      constexpr uint32_t id_kmn = make_idesc_bf16(128, HD, false, true);   // dV, dK
      constexpr uint32_t id_mnmn = make_idesc_bf16(128, HD, true, true);   // dQ
      const uint32_t sK = smem_u32(smem + Cfg::OFF_K), sV = smem_u32(smem + Cfg::OFF_V);
      const uint32_t sdS = smem_u32(smem + Cfg::OFF_DS), sdO = smem_u32(smem + Cfg::OFF_DO);
      auto mma_S = [&](int G) {
        const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + (G & 1) * Cfg::TILE);
        mbar_wait(&bar_q_full[G & 1], (G >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < HD / 16; ++s)
          umma_f16_ss(tmem + Cfg::S_COL, make_sdesc_sw128(sK + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                      make_sdesc_sw128(sQ + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
        umma_commit(bar_s_full);
      };
      auto mma_dP = [&](int G) {
        mbar_wait(bar_do_full, G & 1);
        if (G > 0) mbar_wait(bar_dq_empty, (G - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < HD / 16; ++s)
          umma_f16_ss(tmem + Cfg::DP_COL, make_sdesc_sw128(sV + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                      make_sdesc_sw128(sdO + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
        umma_commit(bar_dp_full);
      };
      int G = 0, k = 0;
      for (int i = blockIdx.x; i < p.num_items; i += gridDim.x) {
        const BwdItem itm = bwd_item(p, i);
        if (itm.iters == 0) continue;
        mbar_wait(bar_kv_full, k & 1);
        tc_fence_after();
        mma_S(G);
        mma_dP(G);
        for (int it = 0; it < itm.iters; ++it, ++G) {
          const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + (G & 1) * Cfg::TILE);
          mbar_wait(bar_p_full, G & 1);
          if (it == 0 && k > 0) mbar_wait(bar_dkv_empty, (k - 1) & 1);
          tc_fence_after();
          // dV += Pᵀ·dO  (A = Pᵀ in TMEM: queries 0-63 at S cols 0-31, 64-127 at cols 64-95)
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ts(tmem + Cfg::DV_COL, tmem + Cfg::S_COL + (s < 4 ? s * 8 : 64 + (s - 4) * 8),
                        make_sdesc_sw128(sdO + s * 2048, 16384, 1024), id_kmn, (it > 0 || s > 0) ? 1u : 0u);
          umma_commit(bar_do_empty);
          // dK += dSᵀ·Q  (A = dSᵀ smem K-major, B = Q MN-major)
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ss(tmem + Cfg::DK_COL, make_sdesc_sw128(sdS + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                        make_sdesc_sw128(sQ + s * 2048, 16384, 1024), id_kmn, (it > 0 || s > 0) ? 1u : 0u);
          const bool more = it + 1 < itm.iters;
          if (more) mma_S(G + 1);  // next S into the S/P columns (after dV read P: issue order)
          // dQ = dS·K  (A = dS MN-major view of the same smem, B = K MN-major) → dP columns
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ss(tmem + Cfg::DP_COL, make_sdesc_sw128(sdS + s * 2048, 16384, 1024),
                        make_sdesc_sw128(sK + s * 2048, 16384, 1024), id_mnmn, s > 0);
          umma_commit(&bar_q_empty[G & 1]);
          umma_commit(bar_dq_full);
          if (!more) {
            umma_commit(bar_kv_empty);
            umma_commit(bar_dkv_full);
          } else {
            mma_dP(G + 1);
          }
        }
        ++k;
      }
    }
  } else if (warp < 8) {
    // ================================================ softmax warps
    const int quad = warp & 3, half = warp >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int krow = quad * 32 + lane;
    uint8_t* sds = smem + Cfg::OFF_DS + half * 16384 + krow * 128;  // this thread's 128-B dSᵀ row chunk
    int G = 0, k = 0;
    for (int i = blockIdx.x; i < p.num_items; i += gridDim.x) {
      const BwdItem itm = bwd_item(p, i);
      if (itm.iters == 0) continue;
      const int key = itm.k0 + krow;
      const int2 ks = key < p.T ? __ldg(p.cols_span + key) : make_int2(0, 0);
      for (int it = 0; it < itm.iters; ++it, ++G) {
        const int qb = itm.q_lo + (it % itm.nq) * Cfg::BQ;
        const int c0 = half * 64;
        const int c_lo = ks.x - qb - c0, c_hi = ks.y - qb - c0;  // visible columns of this half
        const float* lse2 = reinterpret_cast<const float*>(smem + Cfg::OFF_LSE + (G & 1) * Cfg::VEC) + (qb & 3) + c0;
        const float* dsum = reinterpret_cast<const float*>(smem + Cfg::OFF_DSUM) + (qb & 3) + c0;
        // ---- phase A: S → P (kept in fp32 registers, written to TMEM as bf16)
        mbar_wait(bar_s_full, G & 1);
        tc_fence_after();
        float pr[64];
#pragma unroll
        for (int cc = 0; cc < 64; cc += 32) {
          uint32_t sr[32];
          tmem_ld32(tmem + lane_off + Cfg::S_COL + c0 + cc, sr);
          tmem_wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int c = cc + j;
            pr[c] = (c >= c_lo && c < c_hi) ? ex2_approx(__uint_as_float(sr[j]) * p.scale_log2 - lse2[c]) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = pack_bf16x2(pr[cc + 2 * j], pr[cc + 2 * j + 1]);
          tmem_st16(tmem + lane_off + Cfg::S_COL + c0 + cc / 2, pk);
        }
        // ---- phase B: dP → dS = P ∘ (dP − D) → smem (dSᵀ row, swizzled)
        mbar_wait(bar_dp_full, G & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < 64; cc += 32) {
          uint32_t dr[32];
          tmem_ld32(tmem + lane_off + Cfg::DP_COL + c0 + cc, dr);
          tmem_wait_ld();
          uint32_t dk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int c = cc + 2 * j;
            dk[j] = pack_bf16x2(pr[c] * (__uint_as_float(dr[2 * j]) - dsum[c]),
                                pr[c + 1] * (__uint_as_float(dr[2 * j + 1]) - dsum[c + 1]));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int chunk = (cc / 8 + j) ^ (krow & 7);
            *reinterpret_cast<uint4*>(sds + chunk * 16) = make_uint4(dk[4 * j], dk[4 * j + 1], dk[4 * j + 2], dk[4 * j + 3]);
          }
        }
        tmem_wait_st();
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(bar_p_full);
      }
      // ---- item end: dK / dV epilogue (this thread: key row krow, head-dim half `half`)
      mbar_wait(bar_dkv_full, k & 1);
      tc_fence_after();
      const bool valid = key < p.T;
      const int64_t dst = valid ? (p.row_map ? int64_t(__ldg(p.row_map + key)) : int64_t(key)) : 0;
      __nv_bfloat16* dvrow = p.dv + (dst * p.Hkv + itm.kh) * HD + half * (HD / 2);
      __nv_bfloat16* dkrow = p.dk + (dst * p.Hkv + itm.kh) * HD + half * (HD / 2);
#pragma unroll 1
      for (int c = 0; c < HD / 2; c += 32) {
        uint32_t v[32], kk[32];
        tmem_ld32(tmem + lane_off + Cfg::DV_COL + half * (HD / 2) + c, v);
        tmem_ld32(tmem + lane_off + Cfg::DK_COL + half * (HD / 2) + c, kk);
        tmem_wait_ld();
        if (valid) {
          uint32_t pv[16], pk2[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            pv[j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
            pk2[j] = pack_bf16x2(__uint_as_float(kk[2 * j]) * p.scale, __uint_as_float(kk[2 * j + 1]) * p.scale);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            reinterpret_cast<uint4*>(dvrow + c)[j] = make_uint4(pv[4 * j], pv[4 * j + 1], pv[4 * j + 2], pv[4 * j + 3]);
            reinterpret_cast<uint4*>(dkrow + c)[j] = make_uint4(pk2[4 * j], pk2[4 * j + 1], pk2[4 * j + 2], pk2[4 * j + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(bar_dkv_empty);
      ++k;
    }
  } else if (warp < 12) {
    // ================================================ dQ drain: query row (warp-8)*32 + lane
    const int quad = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int r = quad * 32 + lane;
    int G = 0;
    for (int i = blockIdx.x; i < p.num_items; i += gridDim.x) {
      const BwdItem itm = bwd_item(p, i);
      for (int it = 0; it < itm.iters; ++it, ++G) {
        const int h = itm.kh * group + it / itm.nq;
        const int q = itm.q_lo + (it % itm.nq) * Cfg::BQ + r;
        bool live = false;
        if (q < p.T) {
          const int2 rs = __ldg(p.rows_span + q);
          live = rs.x < itm.k0 + Cfg::BK && rs.y > itm.k0;
        }
        float* dst = p.dq_acc + (static_cast<int64_t>(q) * p.H + h) * HD;
        mbar_wait(bar_dq_full, G & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + lane_off + Cfg::DP_COL + c, v);
          tmem_wait_ld();
          if (live) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              red_add_v4_f32(dst + c + 4 * j, __uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                             __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          }
        }
        tc_fence_before();
        mbar_arrive(bar_dq_empty);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) tmem_dealloc<512>(tmem);
}

struct BwdWs {
  float* dq_acc;
  float* lse2;
  float* dsum;
  int2* rows_span;
  int2* cols_span;
};

size_t bwd_ws(BwdWs* w, void* base, const vlasim_attn_args* a) {
  const size_t T = size_t(a->total_tokens), H = size_t(a->num_heads), d = size_t(a->head_dim);
  const size_t Tp = (T + 3) & ~size_t(3);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  uint8_t* b = static_cast<uint8_t*>(base);
  auto take = [&](size_t bytes) {
    uint8_t* r = b ? b + off : nullptr;
    off += up(bytes);
    return r;
  };
  w->dq_acc = reinterpret_cast<float*>(take(T * H * d * 4));
  w->lse2 = reinterpret_cast<float*>(take(Tp * H * 4 + 512 * 4));
  w->dsum = reinterpret_cast<float*>(take(Tp * H * 4 + 512 * 4));
  w->rows_span = reinterpret_cast<int2*>(take(T * 8));
  w->cols_span = reinterpret_cast<int2*>(take(T * 8));
  return off;
}

template <int HD>
int launch_bwd(const vlasim_attn_args* a, const vlasim_attn_grads* g, const BwdWs& w, cudaStream_t st) {
  using namespace vlasim_host;
  using Cfg = BwdCfg<HD>;
  const int T = int(a->total_tokens), H = a->num_heads, Hkv = a->num_kv_heads;
  const int Tp = (T + 3) & ~3;
  const int64_t rows = int64_t(T) * H;
  VLASIM_CUDA_TRY(cudaMemsetAsync(w.dq_acc, 0, size_t(rows) * HD * 4, st));
  k_bwd_pre<HD><<<(rows * (HD / 8) + 255) / 256, 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(a->o), static_cast<const __nv_bfloat16*>(g->dout), a->lse, w.lse2, w.dsum,
      w.rows_span, w.cols_span, a->cu_seqlens, a->prefix_len, a->num_seqs, a->mask_mode, T, Tp, H);
  VLASIM_LAUNCH_CHECK();
  CUtensorMap tq, tk, tv, tdo;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (int rc = encode_tmap_2d(&tq, a->q, BF, T, uint64_t(H) * HD, uint64_t(H) * HD * 2, 128, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&tdo, g->dout, BF, T, uint64_t(H) * HD, uint64_t(H) * HD * 2, 128, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&tk, a->k, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, 128, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&tv, a->v, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, 128, 64, true)) return rc;
  BwdParams p;
  p.dq_acc = w.dq_acc;
  p.dk = static_cast<__nv_bfloat16*>(g->dk);
  p.dv = static_cast<__nv_bfloat16*>(g->dv);
  p.row_map = g->row_map;
  p.lse2 = w.lse2;
  p.dsum = w.dsum;
  p.rows_span = w.rows_span;
  p.cols_span = w.cols_span;
  p.T = T;
  p.Tp = Tp;
  p.H = H;
  p.Hkv = Hkv;
  p.num_items = int((int64_t(T) + 127) / 128) * Hkv;
  p.scale = a->softmax_scale;
  p.scale_log2 = a->softmax_scale * kLog2e;
  auto kern = attn_bwd_kernel<HD>;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int grid = std::min(p.num_items, num_sms());
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(tq, tk, tv, tdo, p);
  VLASIM_LAUNCH_CHECK();
  k_bwd_post<HD><<<(rows * (HD / 8) + 255) / 256, 256, 0, st>>>(w.dq_acc, static_cast<__nv_bfloat16*>(g->dq),
                                                             g->row_map, rows, H, a->softmax_scale);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

}  // namespace

extern "C" size_t vlasim_varlen_attn_workspace_size(const vlasim_attn_args* a, int backward) {
  if (!a) return 0;
  if (!backward) return size_t(a->total_tokens) * 8 + 256;  // forward: per-token visible spans
  BwdWs w;
  return bwd_ws(&w, nullptr, a);
}

extern "C" int vlasim_varlen_attn_bwd_cuda(const vlasim_attn_args* a, const vlasim_attn_grads* g, void* ws,
                                           size_t ws_bytes, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = validate_attn_args(a, false)) return rc;
  if (!g || !g->dout || !g->dq || !g->dk || !g->dv) return set_error(VLASIM_ECONFIG, "attention bwd: grads required");
  if (a->head_dim == 256) return set_error(VLASIM_ECONFIG, "attention bwd: head_dim 256 not supported yet");
  BwdWs w;
  const size_t need = bwd_ws(&w, nullptr, a);
  if (!ws || ws_bytes < need) return set_error(VLASIM_ECONFIG, "attention bwd: workspace %zu < %zu", ws_bytes, need);
  bwd_ws(&w, ws, a);
  cudaStream_t st = as_stream(stream);
  return a->head_dim == 64 ? launch_bwd<64>(a, g, w, st) : launch_bwd<128>(a, g, w, st);
}
