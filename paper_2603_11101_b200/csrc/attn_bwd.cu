// attn_bwd.cu — block-diagonal varlen attention backward for sm_100a.
//
// Gradients of vlasim::packed_attention — the reference has no
// backward; the closed form is SURVEY.md §8(c):
//   P = exp(S·scale − LSE), dV = Pᵀ dO, dP = dO Vᵀ, dS = P ∘ (dP − D), D = rowsum(dO ∘ O),
//   dQ = scale · dS K, dK = scale · dSᵀ Q.
//
// Three launches:
//   k_bwd_pre   D = rowsum(dO∘O), LSE → log2 domain, zero the fp32 dQ accumulator   [HBM-bound]
//   k_bwd_main  one CTA = one 128-key tile (global grid) × one KV head; loops over the q heads
//               of its group and over the 128-row Q tiles of the tile's visible query range
//               (tile skipping: queries outside [q_lo, q_hi) are never loaded).  K and V stay
//               resident in smem; Q/dO/LSE/D stream through a 2-stage TMA ring.
//   k_bwd_post  dQ = bf16(scale · dQacc)
//
// k_bwd_main warp roles (320 threads):
//   warps 0-3  "softmax": thread i owns key row i (TMEM lane i): Pᵀ → TMEM (aliasing S),
//              dSᵀ → smem (SWIZZLE_128B, read back as K-major A for dK and MN-major A for dQ);
//              final dK/dV epilogue.
//   warps 4-7  dQ drain: TMEM dQ rows → red.global.add.v4.f32 into the fp32 accumulator.
//   warp 8     TMA producer.  warp 9  TMEM allocator + tcgen05.mma issuer.
// TMEM (512 cols): S/P [0,128) · dP/dQ [128,256) · dV [256,256+HD) · dK after dV.
// The P→S and dP→dQ aliasing relies on tcgen05.mma executing in issue order (the same
// property CUTLASS/FA4 SM100 backward kernels use).
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
template <int HD>
__global__ void k_bwd_pre(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                          const float* __restrict__ lse, float* __restrict__ lse2, float* __restrict__ dsum,
                          int T, int Tp, int H) {
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
  const int32_t* cu;
  const int32_t* prefix;
  int nseq, T, H, Hkv, mask;
  float scale_log2, scale;
  const int32_t* row_map;  // packed row → output row for dK/dV (NULL: identity)
  const float* lse2;  // [H, Tp] log2-domain LSE
  const float* dsum;  // [H, Tp] rowsum(dO ∘ O)
  int Tp;
  int dbg;  // debug bisection mask (VLASIM_BWD_DEBUG), 0 in production
};

template <int HD>
struct BwdCfg {
  static constexpr int BK = 128, BQ = 128, QSTAGES = 2;
  static constexpr int TILE = 128 * HD * 2;     // one 128-row bf16 tile (K, V, Q or dO)
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;        // Q ring: stage s at OFF_Q + s*TILE
  static constexpr int OFF_DO = OFF_Q + QSTAGES * TILE;  // dO: single buffer
  static constexpr int OFF_DS = OFF_DO + TILE;
  static constexpr int VEC = 544;                        // 132 floats (16-B aligned window of 128) + pad
  static constexpr int OFF_LSE = OFF_DS + 128 * 128 * 2;  // lse2 [QSTAGES][VEC]
  static constexpr int OFF_DSUM = OFF_LSE + QSTAGES * VEC;  // D [VEC]
  static constexpr int OFF_BAR = OFF_DSUM + VEC;
  static constexpr int NUM_BARS = 2 * QSTAGES + 9;
  static constexpr int SMEM_USED = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int SMEM = SMEM_USED + 1024;  // + alignment slack (dynamic smem base is not 1 KB aligned)
  static constexpr uint32_t S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 256 + HD;
  static_assert(DK_COL + HD <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
};

template <int HD>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const BwdParams p) {
  using Cfg = BwdCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* bar_kv = bars + 0;                          // K,V landed
  uint64_t* bar_q_full = bars + 1;                      // [QSTAGES] Q + lse2 landed
  uint64_t* bar_q_empty = bars + 1 + Cfg::QSTAGES;      // [QSTAGES]
  uint64_t* bar_do_full = bars + 1 + 2 * Cfg::QSTAGES;  // dO + D landed
  uint64_t* bar_do_empty = bar_do_full + 1;             // dV MMA done with dO
  uint64_t* bar_s_full = bar_do_full + 2;               // S, dP computed
  uint64_t* bar_p_full = bar_do_full + 3;               // P in TMEM + dS in smem (128 arrivals)
  uint64_t* bar_dq_full = bar_do_full + 4;              // dQ computed
  uint64_t* bar_dq_empty = bar_do_full + 5;             // dQ drained (128 arrivals)
  uint64_t* bar_done = bar_do_full + 6;                 // all MMAs done (dK, dV final)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + Cfg::NUM_BARS * 8);
  int* s_range = reinterpret_cast<int*>(tmem_slot + 1);  // q_lo, q_hi

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kh = blockIdx.x % p.Hkv;
  const int kt = blockIdx.x / p.Hkv;
  const int k0 = kt * Cfg::BK;
  const int group = p.H / p.Hkv;

  if (tid == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < Cfg::QSTAGES; ++s) {
      mbar_init(&bar_q_full[s], 1);
      mbar_init(&bar_q_empty[s], 1);
    }
    mbar_init(bar_do_full, 1);
    mbar_init(bar_do_empty, 1);
    mbar_init(bar_s_full, 1);
    mbar_init(bar_p_full, 128);
    mbar_init(bar_dq_full, 1);
    mbar_init(bar_dq_empty, 128);
    mbar_init(bar_done, 1);
    s_range[0] = INT_MAX;
    s_range[1] = INT_MIN;
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  __syncthreads();

  RowSpan ks{0, 0, -1};
  if (tid < 128) {
    ks = key_span(p.cu, p.prefix, p.nseq, p.mask, k0 + tid, p.T);
    if (ks.lo < ks.hi) {
      atomicMin(&s_range[0], ks.lo);
      atomicMax(&s_range[1], ks.hi);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int q_lo = s_range[0];
  const int nq = (s_range[1] - q_lo + Cfg::BQ - 1) / Cfg::BQ;  // q tiles per head
  const int iters = nq * group;                               // (head, q tile) pairs

  if (warp == 8) {
    // ------------------------------------------------ TMA producer
    if (lane == 0 && iters > 0) {
      mbar_expect_tx(bar_kv, 2 * Cfg::TILE);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        tma_load_2d(smem + Cfg::OFF_K + c * 128 * 128, &tmK, kh * HD + c * 64, k0, bar_kv);
        tma_load_2d(smem + Cfg::OFF_V + c * 128 * 128, &tmV, kh * HD + c * 64, k0, bar_kv);
      }
      for (int it = 0; it < iters; ++it) {
        const int st = it % Cfg::QSTAGES;
        const int h = kh * group + it / nq;
        const int qb = q_lo + (it % nq) * Cfg::BQ;
        if (it >= Cfg::QSTAGES) mbar_wait(&bar_q_empty[st], ((it / Cfg::QSTAGES) - 1) & 1);
        uint8_t* sq = smem + Cfg::OFF_Q + st * Cfg::TILE;
        mbar_expect_tx(&bar_q_full[st], Cfg::TILE + 528);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) tma_load_2d(sq + c * 128 * 128, &tmQ, h * HD + c * 64, qb, &bar_q_full[st]);
        bulk_load(smem + Cfg::OFF_LSE + st * Cfg::VEC, p.lse2 + int64_t(h) * p.Tp + (qb & ~3), 528, &bar_q_full[st]);
        if (it >= 1) mbar_wait(bar_do_empty, (it - 1) & 1);
        uint8_t* sdo = smem + Cfg::OFF_DO;
        mbar_expect_tx(bar_do_full, Cfg::TILE + 528);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) tma_load_2d(sdo + c * 128 * 128, &tmdO, h * HD + c * 64, qb, bar_do_full);
        bulk_load(smem + Cfg::OFF_DSUM, p.dsum + int64_t(h) * p.Tp + (qb & ~3), 528, bar_do_full);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0 && iters > 0) {
      constexpr uint32_t id_kk = make_idesc_bf16(128, 128, false, false);  // S, dP
      constexpr uint32_t id_kmn = make_idesc_bf16(128, HD, false, true);   // dV, dK
      constexpr uint32_t id_mnmn = make_idesc_bf16(128, HD, true, true);   // dQ
      const uint32_t sK = smem_u32(smem + Cfg::OFF_K), sV = smem_u32(smem + Cfg::OFF_V);
      const uint32_t sdS = smem_u32(smem + Cfg::OFF_DS);
      mbar_wait(bar_kv, 0);
      const uint32_t sdO = smem_u32(smem + Cfg::OFF_DO);
      for (int it = 0; it < iters; ++it) {
        const int st = it % Cfg::QSTAGES;
        const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + st * Cfg::TILE);
        mbar_wait(&bar_q_full[st], (it / Cfg::QSTAGES) & 1);
        tc_fence_after();
        // S^T = K · Q^T
#pragma unroll
        for (int s = 0; s < HD / 16; ++s)
          umma_f16_ss(tmem + Cfg::S_COL, make_sdesc_sw128(sK + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                      make_sdesc_sw128(sQ + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
        // dP^T = V · dO^T   (dP region must be drained of the previous dQ)
        mbar_wait(bar_do_full, it & 1);
        if (it > 0) mbar_wait(bar_dq_empty, (it - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < HD / 16; ++s)
          umma_f16_ss(tmem + Cfg::DP_COL, make_sdesc_sw128(sV + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                      make_sdesc_sw128(sdO + (s / 4) * 16384 + (s % 4) * 32, 16, 1024), id_kk, s > 0);
        umma_commit(bar_s_full);
        mbar_wait(bar_p_full, it & 1);
        tc_fence_after();
        // dV += P^T · dO        (A = P^T in TMEM, B = dO MN-major)
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (!(p.dbg & 8))
          umma_f16_ts(tmem + Cfg::DV_COL, tmem + Cfg::S_COL + s * 8, make_sdesc_sw128(sdO + s * 2048, 16384, 1024),
                      id_kmn, (it > 0 || s > 0) ? 1u : 0u);
        umma_commit(bar_do_empty);
        // dK += dS^T · Q        (A = dS^T smem K-major, B = Q MN-major)
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (!(p.dbg & 4))
          umma_f16_ss(tmem + Cfg::DK_COL, make_sdesc_sw128(sdS + (s / 4) * 16384 + (s % 4) * 32, 16, 1024),
                      make_sdesc_sw128(sQ + s * 2048, 16384, 1024), id_kmn, (it > 0 || s > 0) ? 1u : 0u);
        // dQ = dS · K           (A = dS MN-major view of the same smem, B = K MN-major)
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (!(p.dbg & 2))
          umma_f16_ss(tmem + Cfg::DP_COL, make_sdesc_sw128(sdS + s * 2048, 16384, 1024),
                      make_sdesc_sw128(sK + s * 2048, 16384, 1024), id_mnmn, s > 0);
        umma_commit(&bar_q_empty[st]);
        umma_commit(bar_dq_full);
      }
      umma_commit(bar_done);
    }
  } else if (warp < 4) {
    // ------------------------------------------------ softmax warps: key row = tid
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const int krow = tid;
    uint8_t* sds = smem + Cfg::OFF_DS;
    for (int it = 0; it < iters; ++it) {
      const int st = it % Cfg::QSTAGES;
      const int qb = q_lo + (it % nq) * Cfg::BQ;
      const float* lse2 = reinterpret_cast<const float*>(smem + Cfg::OFF_LSE + st * Cfg::VEC) + (qb & 3);
      const float* dsum = reinterpret_cast<const float*>(smem + Cfg::OFF_DSUM) + (qb & 3);
      mbar_wait(bar_s_full, it & 1);
      tc_fence_after();
      const int c_lo = ks.lo - qb, c_hi = ks.hi - qb;  // visible query columns of this key row
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t sr[32], dr[32];
        tmem_ld32(tmem + lane_off + Cfg::S_COL + c0, sr);
        tmem_ld32(tmem + lane_off + Cfg::DP_COL + c0, dr);
        tmem_wait_ld();
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float pp[2], dd[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int c = c0 + 2 * i + u;
            const bool vis = c >= c_lo && c < c_hi;
            const float pv = vis ? ex2_approx(__uint_as_float(sr[2 * i + u]) * p.scale_log2 - lse2[c]) : 0.f;
            pp[u] = pv;
            dd[u] = pv * (__uint_as_float(dr[2 * i + u]) - dsum[c]);
          }
          pk[i] = pack_bf16x2(pp[0], pp[1]);
          dk[i] = pack_bf16x2(dd[0], dd[1]);
        }
        if (!(p.dbg & 32)) tmem_st16(tmem + lane_off + Cfg::S_COL + c0 / 2, pk);
        // dS^T row krow, queries c0..c0+31 → box c0/64, 16-B chunks (c0%64)/8 .. +3, swizzled
        uint8_t* rowp = sds + (c0 / 64) * 16384 + krow * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int chunk = ((c0 % 64) / 8 + j) ^ (krow & 7);
          *reinterpret_cast<uint4*>(rowp + chunk * 16) = make_uint4(dk[4 * j], dk[4 * j + 1], dk[4 * j + 2], dk[4 * j + 3]);
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(bar_p_full);
    }
    // ------------------------------------------------ dK / dV epilogue
    if (iters > 0) {
      mbar_wait(bar_done, 0);
      tc_fence_after();
    }
    const int key = k0 + krow;
    const bool valid = key < p.T;
    const int64_t dst = valid ? (p.row_map ? int64_t(__ldg(p.row_map + key)) : int64_t(key)) : 0;
    __nv_bfloat16* dvrow = p.dv + (dst * p.Hkv + kh) * HD;
    __nv_bfloat16* dkrow = p.dk + (dst * p.Hkv + kh) * HD;
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t v[32], k[32];
      tmem_ld32(tmem + lane_off + Cfg::DV_COL + c, v);
      tmem_ld32(tmem + lane_off + Cfg::DK_COL + c, k);
      tmem_wait_ld();
      if (valid) {
        uint32_t pv[16], pk2[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float a0 = iters > 0 ? __uint_as_float(v[2 * i]) : 0.f, a1 = iters > 0 ? __uint_as_float(v[2 * i + 1]) : 0.f;
          const float b0 = iters > 0 ? __uint_as_float(k[2 * i]) * p.scale : 0.f;
          const float b1 = iters > 0 ? __uint_as_float(k[2 * i + 1]) * p.scale : 0.f;
          pv[i] = pack_bf16x2(a0, a1);
          pk2[i] = pack_bf16x2(b0, b1);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          reinterpret_cast<uint4*>(dvrow + c)[i] = make_uint4(pv[4 * i], pv[4 * i + 1], pv[4 * i + 2], pv[4 * i + 3]);
          reinterpret_cast<uint4*>(dkrow + c)[i] = make_uint4(pk2[4 * i], pk2[4 * i + 1], pk2[4 * i + 2], pk2[4 * i + 3]);
        }
      }
    }
  } else {
    // ------------------------------------------------ dQ drain warps 4-7: query row = (warp-4)*32 + lane
    const int wq = warp - 4;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const int r = wq * 32 + lane;
    for (int it = 0; it < iters; ++it) {
      const int h = kh * group + it / nq;
      const int q = q_lo + (it % nq) * Cfg::BQ + r;
      // does query q see any key of this tile?
      bool live = false;
      if (q < p.T) {
        const RowSpan rs = row_span(p.cu, p.prefix, p.nseq, p.mask, q, p.T);
        live = rs.lo < min(rs.hi, k0 + Cfg::BK) && max(rs.lo, k0) < rs.hi;
      }
      mbar_wait(bar_dq_full, it & 1);
      tc_fence_after();
      float* dst = p.dq_acc + (static_cast<int64_t>(q) * p.H + h) * HD;
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + Cfg::DP_COL + c, v);
        tmem_wait_ld();
        if (live && !(p.dbg & 16)) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            red_add_v4_f32(dst + c + 4 * i, __uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                           __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        }
      }
      tc_fence_before();
      mbar_arrive(bar_dq_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

struct BwdWs {
  float* dq_acc;
  float* lse2;
  float* dsum;
};

size_t bwd_ws(BwdWs* w, void* base, const vlasim_attn_args* a) {
  const size_t T = size_t(a->total_tokens), H = size_t(a->num_heads), d = size_t(a->head_dim);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  uint8_t* b = static_cast<uint8_t*>(base);
  w->dq_acc = reinterpret_cast<float*>(b ? b + off : nullptr);
  off += up(T * H * d * 4);
  w->lse2 = reinterpret_cast<float*>(b ? b + off : nullptr);
  off += up(((T + 3) & ~size_t(3)) * H * 4 + 512 * 4);
  w->dsum = reinterpret_cast<float*>(b ? b + off : nullptr);
  off += up(((T + 3) & ~size_t(3)) * H * 4 + 512 * 4);
  return off;
}

template <int HD>
int launch_bwd(const vlasim_attn_args* a, const vlasim_attn_grads* g, const BwdWs& w, cudaStream_t st) {
  using namespace vlasim_host;
  using Cfg = BwdCfg<HD>;
  const int T = int(a->total_tokens), H = a->num_heads, Hkv = a->num_kv_heads;
  const int64_t rows = int64_t(T) * H;
  VLASIM_CUDA_TRY(cudaMemsetAsync(w.dq_acc, 0, size_t(rows) * HD * 4, st));
  k_bwd_pre<HD><<<(rows * (HD / 8) + 255) / 256, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a->o),
                                                            static_cast<const __nv_bfloat16*>(g->dout), a->lse,
                                                            w.lse2, w.dsum, T, (T + 3) & ~3, H);
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
  p.cu = a->cu_seqlens;
  p.prefix = a->prefix_len;
  p.nseq = a->num_seqs;
  p.T = T;
  p.H = H;
  p.Hkv = Hkv;
  p.mask = a->mask_mode;
  p.scale = a->softmax_scale;
  p.scale_log2 = a->softmax_scale * kLog2e;
  p.row_map = g->row_map;
  p.lse2 = w.lse2;
  p.dsum = w.dsum;
  p.Tp = (T + 3) & ~3;
  p.dbg = getenv("VLASIM_BWD_DEBUG") ? atoi(getenv("VLASIM_BWD_DEBUG")) : 0;
  auto kern = attn_bwd_kernel<HD>;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int64_t ktiles = (int64_t(T) + 127) / 128;
  kern<<<ktiles * Hkv, 320, Cfg::SMEM, st>>>(tq, tk, tv, tdo, p);
  VLASIM_LAUNCH_CHECK();
  k_bwd_post<HD><<<(rows * (HD / 8) + 255) / 256, 256, 0, st>>>(w.dq_acc, static_cast<__nv_bfloat16*>(g->dq),
                                                             g->row_map, rows, H, a->softmax_scale);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

}  // namespace

extern "C" size_t vlasim_varlen_attn_workspace_size(const vlasim_attn_args* a, int backward) {
  if (!a || !backward) return 0;
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
