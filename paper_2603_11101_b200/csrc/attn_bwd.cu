// attn_bwd.cu — block-diagonal varlen attention backward for sm_100a.
//
// Gradients of vlasim::packed_attention — the reference has no
// backward; the closed form is SURVEY.md §8(c):
//   P = exp(S·scale − LSE), dV = Pᵀ dO, dP = dO Vᵀ, dS = P ∘ (dP − D), D = rowsum(dO ∘ O),
//   dQ = scale · dS K, dK = scale · dSᵀ Q.
//
// Launches (no atomics, no fp32 dQ accumulator in HBM — dQ is deterministic):
//   k_bwd_pre   D = rowsum(dO∘O), LSE → log2 domain, per-token visible spans    [HBM-bound]
//   k_bwd_dkdv  persistent, KV-stationary: items = (128-key tile, kv head); loops over the q
//               heads of the group × the 128-row Q tiles of the tile's visible query range
//               (tile skipping: queries outside [q_lo, q_hi) are never loaded or multiplied).
//               4 GEMMs per (key tile, Q tile): Sᵀ, dPᵀ, dV, dK.
//   k_bwd_dq    persistent, Q-stationary: items = (128-row Q tile, head); loops over the key
//               tiles of the visible key range.  3 GEMMs per tile: S, dP, dQ (recomputing S and
//               dP costs 2 GEMMs but removes the dQ reduction across key tiles).
// Both kernels: warps 0-7 softmax (warp w: TMEM lane quadrant w%4, column half w/4), warp 8 TMA
// producer, warp 9 TMEM allocator + tcgen05.mma issuer.  P / dS are written as bf16 over the
// TMEM columns they were computed from and fed back as the A operand (A-from-TMEM MMAs); the
// column aliasing relies on tcgen05.mma executing in issue order.  dQ/dK/dV rows are written
// through the optional row_map (scatter back to sample order fused into the epilogues).
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
    // 4 copies shifted by s = 0..3 elements: any 128-wide window [qb, qb+128) starts 16-B aligned
    // in copy (−qb) & 3, so the dK/dV kernel reads it with 128-bit shared loads.
    const int64_t cp = int64_t(H) * Tp + 512;
    const float l2 = lse[int64_t(h) * T + t] * kLog2e;
#pragma unroll
    for (int sh = 0; sh < 4; ++sh) {
      dsum[sh * cp + int64_t(h) * Tp + t + sh] = acc;
      lse2[sh * cp + int64_t(h) * Tp + t + sh] = l2;
    }
    if (h == 0) {
      const RowSpan r = row_span(cu, prefix, nseq, mask, t, T);
      const RowSpan c = key_span(cu, prefix, nseq, mask, t, T);
      rows_span[t] = make_int2(r.lo, r.hi);
      cols_span[t] = make_int2(c.lo, c.hi);
    }
  }
}

// ------------------------------------------------------------------ main kernels
struct BwdParams {
  __nv_bfloat16* dq;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  const int32_t* row_map;  // packed row → output row for dQ/dK/dV (NULL: identity)
  const float* lse2;       // [H, Tp] log2-domain LSE
  const float* dsum;       // [H, Tp] rowsum(dO ∘ O)
  const int2* rows_span;   // [T] visible keys of query t
  const int2* cols_span;   // [T] queries that see key t
  int T, Tp, H, Hkv, kv_items, q_items;
  int64_t vec_copy;  // element stride between the 4 shifted copies of lse2 / dsum
  float scale_log2, scale;
  unsigned long long* prof;  // [3 roles][8] wait cycles (PROF instantiation only)
};

// ================================================================== dK / dV (KV-stationary)
// One CTA loops over items = (128-key tile, kv head).  Per iteration G (q head of the group,
// 128-row Q tile of the visible query range):
//   Sᵀ = K·Qᵀ, dPᵀ = V·dOᵀ                                  (SS, K-major operands)
//   softmax warps: phase A  Pᵀ = exp2(Sᵀ·scale·log2e − lse2) → bf16 → smem (K-major SW128)
//                  phase B  dSᵀ = Pᵀ ∘ (dPᵀ − D) → bf16 over the dP TMEM columns
//   dV += Pᵀ·dO (A = Pᵀ smem), dK += dSᵀ·Q (A = dSᵀ TMEM)     (B = dO / Q, MN-major)
// Because Pᵀ lives in smem, the S columns are free as soon as phase A has read them, so S(G+1)
// is issued before dV(G)/dK(G) and phase A(G+1) overlaps them.  The Pᵀ buffer doubles as the
// epilogue staging buffer (dK/dV rows leave through per-thread async bulk stores).
// TMEM: S [0,128) · dP/dS [128,256) · dV [256,256+HD) · dK after.  Q and dO double-buffered.
template <int HD>
struct DkvCfg {
  static constexpr int TILE = 128 * HD * 2;
  static constexpr int OFF_K = 0, OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;        // [2]
  static constexpr int OFF_DO = 4 * TILE;       // [2]
  static constexpr int OFF_PT = 6 * TILE;       // Pᵀ [128 keys × 128 q] bf16 (SW128) / epilogue staging
  static constexpr int PT_BYTES = 128 * 128 * 2 > TILE ? 128 * 128 * 2 : TILE;
  static constexpr int VEC = 544;               // 132 floats (16-B aligned window of 128) + pad
  static constexpr int OFF_LSE = OFF_PT + PT_BYTES;   // [2][VEC]
  static constexpr int OFF_DSUM = OFF_LSE + 2 * VEC;  // [2][VEC]
  static constexpr int OFF_BAR = OFF_DSUM + 2 * VEC;
  static constexpr int NUM_BARS = 18;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + 512;  // + rows[128]; base is 1 KB aligned
  static constexpr uint32_t S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 256 + HD;
  static_assert(DK_COL + HD <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
};

struct KvItem {
  int k0, kh, q_lo, nq, iters;
};
__device__ __forceinline__ KvItem kv_item(const BwdParams& p, int i) {
  KvItem it;
  it.kh = i % p.Hkv;
  it.k0 = (i / p.Hkv) * 128;
  const int2 first = __ldg(p.cols_span + it.k0);
  const int2 last = __ldg(p.cols_span + min(it.k0 + 127, p.T - 1));
  it.q_lo = first.x;
  it.nq = max(0, (last.y - first.x + 127) / 128);
  it.iters = it.nq * (p.H / p.Hkv);
  return it;
}

// Coalesced epilogue store of a [128 rows × HD] bf16 tile held by NT softmax threads as packed
// registers (thread = (row, 1/NP of the head dim)): registers → swizzled smem staging → 16-B
// global stores, consecutive threads covering consecutive 16-B chunks of a 256-B row.
// rows[r] < 0 skips row r.  NT = 128·NP threads participate (named barrier bar_id).
template <int HD, int NP>
__device__ __forceinline__ void store_tile_coalesced(uint8_t* stg, const int* rows, const uint32_t* pk, int krow,
                                                     int part, int tid, __nv_bfloat16* base, int64_t row_stride,
                                                     int bar_id) {
  constexpr int CH = HD / 8;        // 16-B chunks per row
  constexpr int CPT = CH / NP;      // chunks per thread
  constexpr int NT = 128 * NP;
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int ch = (part * CPT + j) ^ (krow & (CH - 1));
    *reinterpret_cast<uint4*>(stg + krow * (HD * 2) + ch * 16) =
        make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
  }
  named_bar_sync(bar_id, NT);
#pragma unroll
  for (int idx = tid; idx < 128 * CH; idx += NT) {
    const int r = idx / CH, ch = idx % CH;
    const int dst = rows[r];
    if (dst >= 0) {
      const uint4 v = *reinterpret_cast<const uint4*>(stg + r * (HD * 2) + ((ch ^ (r & (CH - 1))) * 16));
      *reinterpret_cast<uint4*>(base + int64_t(dst) * row_stride + ch * 8) = v;
    }
  }
  named_bar_sync(bar_id, NT);
}

// Warp roles (576 threads): warps 0-15 softmax — warp w owns key rows 32·(w%4).. (TMEM lane
// quadrant w%4) and query columns [32·(w/4), +32); warp 16 TMA producer; warp 17 MMA issuer.
constexpr int kDkvThreads = 576;

template <int HD, bool PROF>
__global__ void __launch_bounds__(kDkvThreads, 1)
    k_bwd_dkdv(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO, const BwdParams p) {
  using Cfg = DkvCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* bar_kv_full = bars + 0;
  uint64_t* bar_kv_empty = bars + 1;
  uint64_t* bar_q_full = bars + 2;    // [2]
  uint64_t* bar_q_empty = bars + 4;   // [2]
  uint64_t* bar_do_full = bars + 6;   // [2]
  uint64_t* bar_do_empty = bars + 8;  // [2]
  uint64_t* bar_s_full = bars + 10;
  uint64_t* bar_dp_full = bars + 11;
  uint64_t* bar_p_full = bars + 12;     // 512 arrivals: Pᵀ in smem, dSᵀ in TMEM
  uint64_t* bar_dkv_full = bars + 13;
  uint64_t* bar_dkv_empty = bars + 14;  // 512 arrivals
  uint64_t* bar_s_free = bars + 15;     // 512 arrivals: S columns read by phase A
  uint64_t* bar_pv_done = bars + 16;    // dV(G) has read Pᵀ from smem
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);
  int* rows = reinterpret_cast<int*>(tmem_slot + 4);  // [128] epilogue destination rows

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int group = p.H / p.Hkv;
  if (tid == 0) {
    if (smem_u32(smem) & 1023) __trap();
    mbar_init(bar_kv_full, 1);
    mbar_init(bar_kv_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_q_full[s], 1);
      mbar_init(&bar_q_empty[s], 1);
      mbar_init(&bar_do_full[s], 1);
      mbar_init(&bar_do_empty[s], 1);
    }
    mbar_init(bar_s_full, 1);
    mbar_init(bar_dp_full, 1);
    mbar_init(bar_p_full, 512);
    mbar_init(bar_dkv_full, 1);
    mbar_init(bar_dkv_empty, 512);
    mbar_init(bar_s_free, 512);
    mbar_init(bar_pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 17) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 16) {
    // ================================================ TMA producer
    if (lane == 0) {
      WaitProf<PROF> wp;
      int G = 0, k = 0;
      KvItem nxt = kv_item(p, blockIdx.x < p.kv_items ? blockIdx.x : 0);
      for (int i = blockIdx.x; i < p.kv_items; i += gridDim.x) {
        const KvItem itm = nxt;
        if (i + int(gridDim.x) < p.kv_items) nxt = kv_item(p, i + gridDim.x);  // prefetch
        if (itm.iters == 0) continue;
        for (int it = 0; it < itm.iters; ++it, ++G) {
          const int h = itm.kh * group + it / itm.nq;
          const int qb = itm.q_lo + (it % itm.nq) * 128;
          const int b = G & 1;
          if (G >= 2) wp.template wait<0>(&bar_q_empty[b], ((G >> 1) - 1) & 1);
          mbar_expect_tx(&bar_q_full[b], Cfg::TILE + 512);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_2d(smem + Cfg::OFF_Q + b * Cfg::TILE + c * 16384, &tmQ, h * HD + c * 64, qb, &bar_q_full[b]);
          bulk_load(smem + Cfg::OFF_LSE + b * Cfg::VEC, p.lse2 + ((-qb) & 3) * p.vec_copy + int64_t(h) * p.Tp + qb + ((-qb) & 3), 512, &bar_q_full[b]);
          if (it == 0) {
            if (k > 0) wp.template wait<1>(bar_kv_empty, (k - 1) & 1);
            mbar_expect_tx(bar_kv_full, 2 * Cfg::TILE);
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
              tma_load_2d(smem + Cfg::OFF_K + c * 16384, &tmK, itm.kh * HD + c * 64, itm.k0, bar_kv_full);
              tma_load_2d(smem + Cfg::OFF_V + c * 16384, &tmV, itm.kh * HD + c * 64, itm.k0, bar_kv_full);
            }
          }
          if (G >= 2) wp.template wait<2>(&bar_do_empty[b], ((G >> 1) - 1) & 1);
          mbar_expect_tx(&bar_do_full[b], Cfg::TILE + 512);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_2d(smem + Cfg::OFF_DO + b * Cfg::TILE + c * 16384, &tmdO, h * HD + c * 64, qb, &bar_do_full[b]);
          bulk_load(smem + Cfg::OFF_DSUM + b * Cfg::VEC, p.dsum + ((-qb) & 3) * p.vec_copy + int64_t(h) * p.Tp + qb + ((-qb) & 3), 512, &bar_do_full[b]);
        }
        ++k;
      }
      wp.flush(p.prof);
    }
  } else if (warp == 17) {
    // ================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_kk = make_idesc_bf16(128, 128, false, false);  // Sᵀ, dPᵀ
      constexpr uint32_t id_kmn = make_idesc_bf16(128, HD, false, true);   // dV, dK
      const uint32_t sK = smem_u32(smem + Cfg::OFF_K), sV = smem_u32(smem + Cfg::OFF_V);
      const uint32_t sPT = smem_u32(smem + Cfg::OFF_PT);
      WaitProf<PROF> wp;
      auto mma_S = [&](int G) {
        const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + (G & 1) * Cfg::TILE);
        wp.template wait<1>(&bar_q_full[G & 1], (G >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < HD / 16; ++s)
          umma_f16_ss(tmem + Cfg::S_COL, make_sdesc_sw128(sK + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                      make_sdesc_sw128(sQ + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
        umma_commit(bar_s_full);
      };
      auto mma_dP = [&](int G) {
        const uint32_t sdO = smem_u32(smem + Cfg::OFF_DO + (G & 1) * Cfg::TILE);
        wp.template wait<2>(&bar_do_full[G & 1], (G >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < HD / 16; ++s)
          umma_f16_ss(tmem + Cfg::DP_COL, make_sdesc_sw128(sV + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                      make_sdesc_sw128(sdO + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
        umma_commit(bar_dp_full);
      };
      int G = 0, k = 0;
      KvItem nxt = kv_item(p, blockIdx.x < p.kv_items ? blockIdx.x : 0);
      for (int i = blockIdx.x; i < p.kv_items; i += gridDim.x) {
        const KvItem itm = nxt;
        if (i + int(gridDim.x) < p.kv_items) nxt = kv_item(p, i + gridDim.x);  // prefetch
        if (itm.iters == 0) continue;
        wp.template wait<0>(bar_kv_full, k & 1);
        tc_fence_after();
        if (G > 0) wp.template wait<5>(bar_s_free, (G - 1) & 1);  // previous item's last S was read
        mma_S(G);
        mma_dP(G);
        if (itm.iters == 1) umma_commit(bar_kv_empty);  // K, V are read only by S and dP
        for (int it = 0; it < itm.iters; ++it, ++G) {
          const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + (G & 1) * Cfg::TILE);
          const uint32_t sdO = smem_u32(smem + Cfg::OFF_DO + (G & 1) * Cfg::TILE);
          const bool more = it + 1 < itm.iters;
          if (more) {  // S(G+1) as soon as phase A(G) has read S(G)
            wp.template wait<5>(bar_s_free, G & 1);
            mma_S(G + 1);
          }
          wp.template wait<3>(bar_p_full, G & 1);
          if (it == 0 && k > 0) wp.template wait<4>(bar_dkv_empty, (k - 1) & 1);
          tc_fence_after();
          // dV += Pᵀ·dO  (A = Pᵀ smem K-major, B = dO MN-major)
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ss(tmem + Cfg::DV_COL, make_sdesc_sw128(sPT + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                        make_sdesc_sw128(sdO + s * 2048, 16384, 1024), id_kmn, (it > 0 || s > 0) ? 1u : 0u);
          umma_commit(bar_pv_done);
          umma_commit(&bar_do_empty[G & 1]);
          // dK += dSᵀ·Q  (A = dSᵀ in TMEM: queries 32j..32j+31 packed at dP cols 32j .. 32j+15)
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ts(tmem + Cfg::DK_COL, tmem + Cfg::DP_COL + (s >> 1) * 32 + (s & 1) * 8,
                        make_sdesc_sw128(sQ + s * 2048, 16384, 1024), id_kmn, (it > 0 || s > 0) ? 1u : 0u);
          umma_commit(&bar_q_empty[G & 1]);
          if (more) {
            mma_dP(G + 1);  // over the dS columns after dK read them (issue order)
            if (it + 2 == itm.iters) umma_commit(bar_kv_empty);  // last readers of K and V issued
          } else {
            umma_commit(bar_dkv_full);
          }
        }
        ++k;
      }
      wp.flush(p.prof + 8);
    }
  } else {
    // ================================================ softmax warps 0-15 (key row, 32-query quarter)
    const int quad = warp & 3, part = warp >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int krow = quad * 32 + lane;
    const int c0 = part * 32;
    // Pᵀ row chunk: box part/2 (queries 64·(part/2)..), 16-B chunks (part%2)*4 .. +3, swizzled
    uint8_t* spt_row = smem + Cfg::OFF_PT + (part >> 1) * 16384 + krow * 128;
    WaitProf<PROF> wp;
    int G = 0, k = 0;
    KvItem nxt = kv_item(p, blockIdx.x < p.kv_items ? blockIdx.x : 0);
    int2 ks_nxt = nxt.k0 + krow < p.T ? __ldg(p.cols_span + nxt.k0 + krow) : make_int2(0, 0);
    for (int i = blockIdx.x; i < p.kv_items; i += gridDim.x) {
      const KvItem itm = nxt;
      const int2 ks = ks_nxt;
      if (i + int(gridDim.x) < p.kv_items) {  // prefetch the next item's parameters
        nxt = kv_item(p, i + gridDim.x);
        ks_nxt = nxt.k0 + krow < p.T ? __ldg(p.cols_span + nxt.k0 + krow) : make_int2(0, 0);
      }
      if (itm.iters == 0) continue;
      const int key = itm.k0 + krow;
      for (int it = 0; it < itm.iters; ++it, ++G) {
        const int qb = itm.q_lo + (it % itm.nq) * 128;
        const int c_lo = ks.x - qb - c0, c_hi = ks.y - qb - c0;  // visible columns of this quarter
        const bool full = c_lo <= 0 && c_hi >= 32;
        const float4* lse4 = reinterpret_cast<const float4*>(smem + Cfg::OFF_LSE + (G & 1) * Cfg::VEC) + c0 / 4;
        const float4* dsum4 = reinterpret_cast<const float4*>(smem + Cfg::OFF_DSUM + (G & 1) * Cfg::VEC) + c0 / 4;
        // ---- phase A: Sᵀ → Pᵀ (fp32 registers; bf16 to smem)
        wp.template wait<0>(bar_s_full, G & 1);
        const long long ta = wp.now();
        tc_fence_after();
        float pr[32];
        {
          uint32_t sa[32];
          tmem_ld32(tmem + lane_off + Cfg::S_COL + c0, sa);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(bar_s_free);  // the MMA warp may overwrite S now
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 l = lse4[j4];  // 128-bit broadcast load
            const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = 4 * j4 + u;
              const float e = ex2_approx(fmaf(__uint_as_float(sa[j]), p.scale_log2, -lv[u]));
              pr[j] = (full || (j >= c_lo && j < c_hi)) ? e : 0.f;
            }
          }
        }
        if (G > 0) wp.template wait<2>(bar_pv_done, (G - 1) & 1);  // dV(G-1) has read the Pᵀ buffer
        if (it == 0 && k > 0) named_bar_sync(6, 512);              // epilogue staging reads finished
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) w[u] = pack_bf16x2(pr[8 * j + 2 * u], pr[8 * j + 2 * u + 1]);
          *reinterpret_cast<uint4*>(spt_row + ((((part & 1) * 4 + j) ^ (krow & 7)) * 16)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        wp.template add_since<4>(ta);
        // ---- phase B: dPᵀ → dSᵀ = Pᵀ ∘ (dPᵀ − D) → bf16 over the dP columns
        wp.template wait<1>(bar_dp_full, G & 1);
        const long long tb = wp.now();
        tc_fence_after();
        {
          uint32_t dr[32];
          tmem_ld32(tmem + lane_off + Cfg::DP_COL + c0, dr);
          tmem_wait_ld();
          uint32_t dk[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 dd = dsum4[j4];  // 128-bit broadcast load
            const int c = 4 * j4;
            dk[2 * j4] = pack_bf16x2(pr[c] * (__uint_as_float(dr[c]) - dd.x), pr[c + 1] * (__uint_as_float(dr[c + 1]) - dd.y));
            dk[2 * j4 + 1] =
                pack_bf16x2(pr[c + 2] * (__uint_as_float(dr[c + 2]) - dd.z), pr[c + 3] * (__uint_as_float(dr[c + 3]) - dd.w));
          }
          tmem_st16(tmem + lane_off + Cfg::DP_COL + c0, dk);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bar_p_full);
        wp.template add_since<5>(tb);
      }
      // ---- item end: dK / dV epilogue — TMEM → registers → release TMEM → coalesced stores
      //      through the (now idle) Pᵀ buffer
      const long long te = wp.now();
      wp.template wait<3>(bar_dkv_full, k & 1);
      tc_fence_after();
      uint32_t pv[HD / 8], pkk[HD / 8];
#pragma unroll
      for (int c = 0; c < HD / 4; c += 32 > HD / 4 ? HD / 4 : 32) {
        uint32_t v[32], kk[32];
        tmem_ld32(tmem + lane_off + Cfg::DV_COL + part * (HD / 4) + c, v);
        tmem_ld32(tmem + lane_off + Cfg::DK_COL + part * (HD / 4) + c, kk);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < (HD / 4 < 32 ? HD / 8 : 16); ++j) {
          pv[c / 2 + j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
          pkk[c / 2 + j] = pack_bf16x2(__uint_as_float(kk[2 * j]) * p.scale, __uint_as_float(kk[2 * j + 1]) * p.scale);
        }
      }
      tc_fence_before();
      mbar_arrive(bar_dkv_empty);  // TMEM drained: the next item's dV/dK may start
      if (part == 0) rows[krow] = key < p.T ? (p.row_map ? __ldg(p.row_map + key) : key) : -1;
      named_bar_sync(5, 512);
      uint8_t* stg = smem + Cfg::OFF_PT;
      store_tile_coalesced<HD, 4>(stg, rows, pv, krow, part, tid, p.dv + itm.kh * HD, int64_t(p.Hkv) * HD, 5);
      store_tile_coalesced<HD, 4>(stg, rows, pkk, krow, part, tid, p.dk + itm.kh * HD, int64_t(p.Hkv) * HD, 5);
      wp.template add_since<6>(te);
      ++k;
    }
    if (warp == 0 && lane == 0) wp.flush(p.prof + 16);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 17) tmem_dealloc<512>(tmem);
}

// ================================================================== dQ (Q-stationary)
// One CTA loops over items = (128-row Q tile, head).  Per key tile of the visible key range:
//   S = Q·Kᵀ (→ S buffer g%2), dP = dO·Vᵀ                    (SS, K-major operands)
//   softmax warps: P = exp2(S·scale·log2e − lse2_row) (registers), dS = P ∘ (dP − D_row) → bf16
//                  over the S columns
//   dQ += dS·K                                                (A from TMEM, B = K MN-major)
// and writes dQ = scale · dQacc once per item in bf16 (through row_map).  Deterministic: no atomics.
// TMEM: S0 [0,128) · dP [128,256) · dQ [256,256+HD) · S1 [384,512).
template <int HD, int STAGES>
struct DqCfg {
  static constexpr int TILE = 128 * HD * 2;
  static constexpr int OFF_Q = 0, OFF_DO = TILE;
  static constexpr int OFF_KV = 2 * TILE;  // stage s: K at +s*2*TILE, V right after
  static constexpr int OFF_STG = OFF_KV + STAGES * 2 * TILE;  // epilogue staging (128 × HD bf16)
  static constexpr int OFF_ROWS = OFF_STG + TILE;             // int [128]
  static constexpr int OFF_BAR = OFF_ROWS + 512;
  static constexpr int NUM_BARS = 2 + 2 * STAGES + 2 + 2 + 2 + 2;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16;  // dynamic smem base is 1 KB aligned
  static constexpr uint32_t DP_COL = 128, DQ_COL = 256;
  __host__ __device__ static constexpr uint32_t s_col(int g) { return (g & 1) ? 384u : 0u; }
  static_assert(DQ_COL + HD <= 384, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
};

struct QItem {
  int q0, h, kh, kv_lo, nkv;
};
__device__ __forceinline__ QItem q_item(const BwdParams& p, int i) {
  QItem it;
  it.h = i % p.H;
  it.q0 = (i / p.H) * 128;
  it.kh = it.h / (p.H / p.Hkv);
  const int2 a = __ldg(p.rows_span + it.q0);
  const int2 b = __ldg(p.rows_span + min(it.q0 + 127, p.T - 1));
  it.kv_lo = a.x;
  it.nkv = max(0, (b.y - a.x + 127) / 128);
  return it;
}

template <int HD, int STAGES>
__global__ void __launch_bounds__(320, 1)
    k_bwd_dq(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO, const BwdParams p) {
  using Cfg = DqCfg<HD, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* bar_qdo_full = bars + 0;
  uint64_t* bar_qdo_empty = bars + 1;
  uint64_t* bar_kv_full = bars + 2;                // [STAGES]
  uint64_t* bar_kv_empty = bars + 2 + STAGES;      // [STAGES]
  uint64_t* bar_s_full = bars + 2 + 2 * STAGES;    // [2]
  uint64_t* bar_dp_full = bar_s_full + 2;          // one per tile
  uint64_t* bar_p_full = bar_s_full + 3;           // [2] 256 arrivals (dS written over S buffer g%2)
  uint64_t* bar_dq_full = bar_s_full + 5;          // one per item
  uint64_t* bar_dq_empty = bar_s_full + 6;         // 256 arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(bar_qdo_full, 1);
    mbar_init(bar_qdo_empty, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bar_kv_full[s], 1);
      mbar_init(&bar_kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_s_full[s], 1);
      mbar_init(&bar_p_full[s], 256);
    }
    mbar_init(bar_dp_full, 1);
    mbar_init(bar_dq_full, 1);
    mbar_init(bar_dq_empty, 256);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ================================================ TMA producer
    if (lane == 0) {
      int g = 0, k = 0;
      QItem nxt = q_item(p, blockIdx.x < p.q_items ? blockIdx.x : 0);
      for (int i = blockIdx.x; i < p.q_items; i += gridDim.x) {
        const QItem itm = nxt;
        if (i + int(gridDim.x) < p.q_items) nxt = q_item(p, i + gridDim.x);
        if (itm.nkv == 0) continue;
        if (k > 0) mbar_wait(bar_qdo_empty, (k - 1) & 1);
        mbar_expect_tx(bar_qdo_full, 2 * Cfg::TILE);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          tma_load_2d(smem + Cfg::OFF_Q + c * 16384, &tmQ, itm.h * HD + c * 64, itm.q0, bar_qdo_full);
          tma_load_2d(smem + Cfg::OFF_DO + c * 16384, &tmdO, itm.h * HD + c * 64, itm.q0, bar_qdo_full);
        }
        for (int j = 0; j < itm.nkv; ++j, ++g) {
          const int st = g % STAGES;
          if (g >= STAGES) mbar_wait(&bar_kv_empty[st], ((g / STAGES) - 1) & 1);
          uint8_t* sk = smem + Cfg::OFF_KV + st * 2 * Cfg::TILE;
          const int kv0 = itm.kv_lo + j * 128;
          mbar_expect_tx(&bar_kv_full[st], 2 * Cfg::TILE);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c) {
            tma_load_2d(sk + c * 16384, &tmK, itm.kh * HD + c * 64, kv0, &bar_kv_full[st]);
            tma_load_2d(sk + Cfg::TILE + c * 16384, &tmV, itm.kh * HD + c * 64, kv0, &bar_kv_full[st]);
          }
        }
        ++k;
      }
    }
  } else if (warp == 9) {
    // ================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_kk = make_idesc_bf16(128, 128, false, false);  // S, dP
      constexpr uint32_t id_dq = make_idesc_bf16(128, HD, false, true);    // dQ (A from TMEM, B MN-major)
      const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q), sdO = smem_u32(smem + Cfg::OFF_DO);
      int g = 0, k = 0;
      int pj = -1, pg = 0;  // pending dQ MMA of tile pg (local index pj)
      bool plast = false;
      auto do_dq = [&]() {
        mbar_wait(&bar_p_full[pg & 1], (pg >> 1) & 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + Cfg::OFF_KV + (pg % STAGES) * 2 * Cfg::TILE);
        const uint32_t a = tmem + Cfg::s_col(pg);
#pragma unroll
        for (int s = 0; s < 8; ++s)  // dS: keys 0-63 at +0..31, 64-127 at +64..95
          umma_f16_ts(tmem + Cfg::DQ_COL, a + (s < 4 ? s * 8 : 64 + (s - 4) * 8),
                      make_sdesc_sw128(sK + s * 2048, 16384, 1024), id_dq, (pj > 0 || s > 0) ? 1u : 0u);
        umma_commit(&bar_kv_empty[pg % STAGES]);
        if (plast) umma_commit(bar_dq_full);
      };
      QItem nxt = q_item(p, blockIdx.x < p.q_items ? blockIdx.x : 0);
      for (int i = blockIdx.x; i < p.q_items; i += gridDim.x) {
        const QItem itm = nxt;
        if (i + int(gridDim.x) < p.q_items) nxt = q_item(p, i + gridDim.x);
        if (itm.nkv == 0) continue;
        mbar_wait(bar_qdo_full, k & 1);
        for (int j = 0; j < itm.nkv; ++j, ++g) {
          const int st = g % STAGES;
          mbar_wait(&bar_kv_full[st], (g / STAGES) & 1);
          tc_fence_after();
          const uint32_t sK = smem_u32(smem + Cfg::OFF_KV + st * 2 * Cfg::TILE);
          const uint32_t sV = sK + Cfg::TILE;
          // S_g = Q·K_gᵀ into S buffer g%2 (its previous dS was consumed by dQ_{g-2}: issue order)
#pragma unroll
          for (int s = 0; s < HD / 16; ++s)
            umma_f16_ss(tmem + Cfg::s_col(g), make_sdesc_sw128(sQ + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                        make_sdesc_sw128(sK + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
          umma_commit(&bar_s_full[g & 1]);
          // dQ of the previous tile (needs its dS), then dP_g over the dP columns it freed
          if (pj >= 0) do_dq();
          if (j == 0 && k > 0) mbar_wait(bar_dq_empty, (k - 1) & 1);  // previous item's dQ drained
#pragma unroll
          for (int s = 0; s < HD / 16; ++s)
            umma_f16_ss(tmem + Cfg::DP_COL, make_sdesc_sw128(sdO + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                        make_sdesc_sw128(sV + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
          umma_commit(bar_dp_full);
          if (j == itm.nkv - 1) umma_commit(bar_qdo_empty);
          pj = j;
          pg = g;
          plast = (j == itm.nkv - 1);
        }
        ++k;
      }
      if (pj >= 0) do_dq();
    }
  } else {
    // ================================================ softmax + epilogue warps 0-7 (query row, key-column half)
    const int quad = warp & 3, half = warp >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int r = quad * 32 + lane;
    const int c0 = half * 64;
    int g = 0, k = 0;
    // row parameters of the next item are prefetched one item ahead
    auto load_row = [&](const QItem& it, int2& rs_, float& l_, float& d_) {
      const int rw = it.q0 + r;
      const bool v = rw < p.T;
      rs_ = v ? __ldg(p.rows_span + rw) : make_int2(0, 0);
      l_ = v ? __ldg(p.lse2 + int64_t(it.h) * p.Tp + rw) : 0.f;  // copy 0 (unshifted)
      d_ = v ? __ldg(p.dsum + int64_t(it.h) * p.Tp + rw) : 0.f;
    };
    QItem nxt = q_item(p, blockIdx.x < p.q_items ? blockIdx.x : 0);
    int2 rs_n;
    float lse_n, dsum_n;
    load_row(nxt, rs_n, lse_n, dsum_n);
    for (int i = blockIdx.x; i < p.q_items; i += gridDim.x) {
      const QItem itm = nxt;
      const int2 rs = rs_n;
      const float lse2 = lse_n, dsum = dsum_n;
      if (i + int(gridDim.x) < p.q_items) {
        nxt = q_item(p, i + gridDim.x);
        load_row(nxt, rs_n, lse_n, dsum_n);
      }
      if (itm.nkv == 0) continue;
      const int row = itm.q0 + r;
      const bool valid = row < p.T;
      for (int j = 0; j < itm.nkv; ++j, ++g) {
        const uint32_t s_tm = tmem + lane_off + Cfg::s_col(g) + c0;
        const int kv0 = itm.kv_lo + j * 128 + c0;
        const int c_lo = rs.x - kv0, c_hi = rs.y - kv0;
        const bool full = c_lo <= 0 && c_hi >= 64;
        mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        float pr[64];
#pragma unroll
        for (int cc = 0; cc < 64; cc += 32) {
          uint32_t sr[32];
          tmem_ld32(s_tm + cc, sr);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int c = cc + t;
            const float e = ex2_approx(fmaf(__uint_as_float(sr[t]), p.scale_log2, -lse2));
            pr[c] = (full || (c >= c_lo && c < c_hi)) ? e : 0.f;
          }
        }
        mbar_wait(bar_dp_full, g & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < 64; cc += 32) {
          uint32_t dr[32];
          tmem_ld32(tmem + lane_off + Cfg::DP_COL + c0 + cc, dr);
          tmem_wait_ld();
          uint32_t dk[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int c = cc + 2 * t;
            dk[t] = pack_bf16x2(pr[c] * (__uint_as_float(dr[2 * t]) - dsum),
                                pr[c + 1] * (__uint_as_float(dr[2 * t + 1]) - dsum));
          }
          tmem_st16(s_tm + cc / 2, dk);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bar_p_full[g & 1]);
      }
      // ---- item end: dQ = scale · acc → bf16 (half of the head dim per warp), coalesced store
      mbar_wait(bar_dq_full, k & 1);
      tc_fence_after();
      uint32_t pq[HD / 4];
#pragma unroll
      for (int c = 0; c < HD / 2; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + Cfg::DQ_COL + half * (HD / 2) + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 16; ++t)
          pq[c / 2 + t] = pack_bf16x2(__uint_as_float(v[2 * t]) * p.scale, __uint_as_float(v[2 * t + 1]) * p.scale);
      }
      tc_fence_before();
      mbar_arrive(bar_dq_empty);  // TMEM drained: the next item's first dQ MMA may start
      if (valid) {  // this thread's half row → staging → async bulk store
        uint8_t* stg_row = smem + Cfg::OFF_STG + r * (HD * 2) + half * HD;
        const int64_t dst = p.row_map ? int64_t(__ldg(p.row_map + row)) : int64_t(row);
        bulk_wait_read0();  // previous item's store has finished reading the staging row
#pragma unroll
        for (int j = 0; j < HD / 16; ++j)
          *reinterpret_cast<uint4*>(stg_row + j * 16) = make_uint4(pq[4 * j], pq[4 * j + 1], pq[4 * j + 2], pq[4 * j + 3]);
        fence_proxy_async_smem();
        bulk_store(p.dq + (dst * p.H + itm.h) * HD + half * (HD / 2), stg_row, HD);
        bulk_commit();
      }
      ++k;
    }
    bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

struct BwdWs {
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
  (void)d;
  w->lse2 = reinterpret_cast<float*>(take(4 * (Tp * H + 512) * 4));  // 4 shifted copies
  w->dsum = reinterpret_cast<float*>(take(4 * (Tp * H + 512) * 4));
  w->rows_span = reinterpret_cast<int2*>(take(T * 8));
  w->cols_span = reinterpret_cast<int2*>(take(T * 8));
  return off;
}

template <int HD>
int launch_bwd(const vlasim_attn_args* a, const vlasim_attn_grads* g, const BwdWs& w, cudaStream_t st) {
  using namespace vlasim_host;
  const int T = int(a->total_tokens), H = a->num_heads, Hkv = a->num_kv_heads;
  const int Tp = (T + 3) & ~3;
  const int64_t rows = int64_t(T) * H;
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
  p.dq = static_cast<__nv_bfloat16*>(g->dq);
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
  p.kv_items = int((int64_t(T) + 127) / 128) * Hkv;
  p.vec_copy = int64_t(H) * Tp + 512;
  p.q_items = int((int64_t(T) + 127) / 128) * H;
  p.scale = a->softmax_scale;
  p.scale_log2 = a->softmax_scale * kLog2e;
  {
    using Cfg = DkvCfg<HD>;
    const int grid = std::min(p.kv_items, num_sms());
    p.prof = prof_enabled() ? prof_buffer() : nullptr;
    auto kern = p.prof ? k_bwd_dkdv<HD, true> : k_bwd_dkdv<HD, false>;
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    kern<<<grid, kDkvThreads, Cfg::SMEM, st>>>(tq, tk, tv, tdo, p);
    VLASIM_LAUNCH_CHECK();
    if (p.prof)
      prof_report("k_bwd_dkdv", grid, st,
                  {"prod:q_empty", "prod:kv_empty", "prod:do_empty", "", "", "", "", "prod:total", "mma:kv_full",
                   "mma:q_full", "mma:do_full", "mma:p_full", "mma:dkv_empty", "mma:s_free", "", "mma:total",
                   "smx:s_full", "smx:dp_full", "smx:pv_done", "smx:dkv_full", "smx:phaseA", "smx:phaseB",
                   "smx:epilogue", "smx:total"});
  }
  {
    constexpr int ST = HD == 64 ? 4 : 2;
    using Cfg = DqCfg<HD, ST>;
    auto kern = k_bwd_dq<HD, ST>;
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    kern<<<std::min(p.q_items, num_sms()), 320, Cfg::SMEM, st>>>(tq, tk, tv, tdo, p);
    VLASIM_LAUNCH_CHECK();
  }
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
