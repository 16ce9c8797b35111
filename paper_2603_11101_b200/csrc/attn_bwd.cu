// attn_bwd.cu — block-diagonal varlen attention backward for sm_100a.
//
// Gradients of vlasim::packed_attention — the reference has no
// backward; the closed form is SURVEY.md §8(c):
//   P = exp(S·scale − LSE), dV = Pᵀ dO, dP = dO Vᵀ, dS = P ∘ (dP − D), D = rowsum(dO ∘ O),
//   dQ = scale · dS K, dK = scale · dSᵀ Q.
//
// Launches (no atomics, no fp32 dQ accumulator in HBM — dQ is deterministic):
//   k_bwd_pre   D = rowsum(dO∘O), LSE → log2 domain, per-token visible spans    [HBM-bound]
//   k_bwd_dkdv  persistent, KV-stationary: items = (segment-aligned key tile of ≤ 128 rows
//               (attn_tiles.cu), kv head); loops over the q
//               heads of the group × the 128-row Q tiles of the tile's visible query range
//               (tile skipping: queries outside [q_lo, q_hi) are never loaded or multiplied).
//               4 GEMMs per (key tile, Q tile): Sᵀ, dPᵀ, dV, dK.
//   k_bwd_dq    persistent, Q-stationary: items = (segment-aligned Q tile, head); loops over the key
//               tiles of the visible key range.  3 GEMMs per tile: S, dP, dQ (recomputing S and
//               dP costs 2 GEMMs but removes the dQ reduction across key tiles).
// Both kernels: warps 0-7 softmax (warp w: TMEM lane quadrant w%4, column half w/4), warp 8 TMA
// producer, warp 9 TMEM allocator + tcgen05.mma issuer.  P / dS are written as bf16 over the
// TMEM columns they were computed from and fed back as the A operand (A-from-TMEM MMAs); the
// column aliasing relies on tcgen05.mma executing in issue order.  dQ/dK/dV rows are written
// through the optional row_map (scatter back to sample order fused into the epilogues).
#include <cfloat>
#include <climits>
#include <cstring>

#include "attn_common.cuh"
#include "common.hpp"
#include "sm100.cuh"

using namespace vlasim_dev;

namespace vlasim_host {
int validate_attn_args(const vlasim_attn_args* a, bool fp8);
int launch_fp8_dequant_bf16(const uint8_t* codes, const float* scales, int64_t T, int heads, int d, void* out,
                            cudaStream_t st);
}

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// ------------------------------------------------------------------ pre / post
// D[h][t] = Σ_c dO·O (fp32) and LSE → log2 domain.  A block owns 32 consecutive tokens × all heads,
// a contiguous [32·H, HD] slab of O and dO read with 16-byte loads (HD/8 lanes per (t, h) row,
// reduced by shuffles); D goes through smem so that the 4 shifted copies of D and lse2 (and the
// per-token visible spans, attn_common.cuh) are written coalesced along the token axis:
// rows[t] = visible keys of query t, cols[t] = queries that see key t.
constexpr int kPreTokens = 32;

template <int HD>
__global__ void __launch_bounds__(256) k_bwd_pre(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                                 const float* __restrict__ lse, float* __restrict__ lse2,
                                                 float* __restrict__ dsum, int2* __restrict__ rows_span,
                                                 int2* __restrict__ cols_span, const int32_t* __restrict__ cu,
                                                 const int32_t* __restrict__ prefix, int nseq, int mask, int T, int Tp,
                                                 int H) {
  constexpr int LPR = HD / 8;  // lanes per row (8 bf16 per lane)
  extern __shared__ float sh_d[];  // [H][kPreTokens]
  const int t0 = blockIdx.x * kPreTokens;
  const int nt = min(kPreTokens, T - t0);
  const int tasks = nt * H * LPR;
  const int64_t base = int64_t(t0) * H * HD;
  // r / H by multiply-high (r < 32·H ≤ 2^16: exact), one division per thread instead of per row
  const unsigned long long mH = (1ull << 32) / unsigned(H) + 1ull;  // H = 1 needs the 33rd bit
  auto slot = [&](int r) {
    const int q = int((static_cast<unsigned long long>(r) * mH) >> 32);
    return (r - q * H) * kPreTokens + q;
  };
#pragma unroll 4
  // Loop exits are warp-uniform (a warp's 32 tasks are consecutive) so that the shuffle reduction
  // always runs with the full warp; tasks past the end contribute zeros and are not written.
  for (int task = threadIdx.x; task < kPreTokens * 16 * LPR; task += 256) {  // uniform trip count (H ≤ 16 fast path)
    if (task - (threadIdx.x & 31) >= tasks) break;
    const bool act = task < tasks;
    const int r = act ? task / LPR : 0, sub = task % LPR;
    const uint4 x = act ? *reinterpret_cast<const uint4*>(o + base + int64_t(r) * HD + sub * 8) : make_uint4(0, 0, 0, 0);
    const uint4 y = act ? *reinterpret_cast<const uint4*>(dout + base + int64_t(r) * HD + sub * 8) : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* px = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* py = reinterpret_cast<const __nv_bfloat162*>(&y);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 a = __bfloat1622float2(px[i]), b = __bfloat1622float2(py[i]);
      acc += a.x * b.x + a.y * b.y;
    }
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (act && sub == 0) sh_d[slot(r)] = acc;
  }
  for (int task = kPreTokens * 16 * LPR + threadIdx.x; task - int(threadIdx.x & 31) < tasks; task += 256) {  // H > 16
    const bool act = task < tasks;
    const int r = act ? task / LPR : 0, sub = task % LPR;
    const uint4 x = act ? *reinterpret_cast<const uint4*>(o + base + int64_t(r) * HD + sub * 8) : make_uint4(0, 0, 0, 0);
    const uint4 y = act ? *reinterpret_cast<const uint4*>(dout + base + int64_t(r) * HD + sub * 8) : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* px = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* py = reinterpret_cast<const __nv_bfloat162*>(&y);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 a = __bfloat1622float2(px[i]), b = __bfloat1622float2(py[i]);
      acc += a.x * b.x + a.y * b.y;
    }
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (act && sub == 0) sh_d[slot(r)] = acc;
  }
  __syncthreads();
  // 4 copies shifted by s = 0..3 elements: any 64/128-wide window [qb, qb+w) starts 16-B aligned
  // in copy (−qb) & 3, so the dK/dV kernel reads it with 128-bit shared loads.
  const int64_t cp = int64_t(H) * Tp + 512;
  for (int idx = threadIdx.x; idx < H * kPreTokens; idx += 256) {
    const int h = idx / kPreTokens, tl = idx % kPreTokens;
    if (tl >= nt) continue;
    const int t = t0 + tl;
    const float d = sh_d[h * kPreTokens + tl];
    const float l2 = lse[int64_t(h) * T + t] * kLog2e;
#pragma unroll
    for (int sh = 0; sh < 4; ++sh) {
      dsum[sh * cp + int64_t(h) * Tp + t + sh] = d;
      lse2[sh * cp + int64_t(h) * Tp + t + sh] = l2;
    }
  }
  if (blockIdx.x == gridDim.x - 1) {
    // Cells no token writes — [h·Tp + sh + T, (h+1)·Tp + sh) after every head (the next head's
    // first sh slots included), [0, sh) and the +512 tail of each copy — are read by the dK/dV
    // kernel's UQ-wide windows past the last token: give them finite neutral values (lse2 = 0,
    // D = 0) so that a masked column computes exp2(−inf) = 0 and 0 · (dP − 0) = 0, never NaN.
    const int gap = Tp - T;  // 0..3
    for (int sh = 0; sh < 4; ++sh) {
      float* l = lse2 + sh * cp;
      float* dd = dsum + sh * cp;
      for (int i = threadIdx.x; i < sh; i += 256) l[i] = dd[i] = 0.f;
      for (int h = 0; h + 1 < H; ++h)
        for (int i = threadIdx.x; i < gap; i += 256) {
          const int64_t c = int64_t(h) * Tp + sh + T + i;
          l[c] = dd[c] = 0.f;
        }
      for (int64_t c = int64_t(H - 1) * Tp + sh + T + threadIdx.x; c < cp; c += 256) l[c] = dd[c] = 0.f;
    }
  }
  if (threadIdx.x < nt) {
    const int t = t0 + threadIdx.x;
    const RowSpan rr = row_span(cu, prefix, nseq, mask, t, T);
    const RowSpan c = key_span(cu, prefix, nseq, mask, t, T);
    rows_span[t] = make_int2(rr.lo, rr.hi);
    cols_span[t] = make_int2(c.lo, c.hi);
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
  const int4* tiles;       // segment-aligned 128-row tiles {t0, te, delta}, sorted by cost (attn_tiles.cu)
  const int* ntiles;       // device-side tile count
  int T, Tp, H, Hkv;
  int64_t vec_copy;  // element stride between the 4 shifted copies of lse2 / dsum
  float scale_log2, scale;
  unsigned long long* prof;  // [3 roles][8] wait cycles (PROF instantiation only)
  int dbg;                   // VLASIM_DBG ablations, honoured by the PROF instantiation only (timing experiments)
  int ohalf;                 // dK/dV head-dim half of this launch (head_dim 256: two launches; else 0)
};

// ================================================================== dK / dV (KV-stationary)
// One CTA loops over items = (128-key tile, kv head).  An item is a run of units u = (q head of
// the group, 64-row Q tile of the key tile's visible query range); per unit:
//   Sᵀ = K·Qᵀ → S[u&1], dPᵀ = V·dOᵀ → dP[u&1]                  (SS, K-major operands, N = 64)
//   softmax group u&1: phase A  Pᵀ = exp2(Sᵀ·scale·log2e − lse2) → bf16 over the S columns
//                      phase B  dSᵀ = Pᵀ ∘ (dPᵀ − D)        → bf16 over the dP columns
//   dV += Pᵀ·dO, dK += dSᵀ·Q                                 (A from TMEM, B = dO / Q MN-major)
// Two softmax groups of 8 warps take alternate units, so while one group exponentiates unit u
// the tensor cores run the GEMMs of its neighbours.  The MMA warp issues one block per unit,
// dV(u) · S(u+2) · dK(u) · dP(u+2), once dSᵀ(u) is written (S/dP run two units ahead; the
// column aliasing — S(u+2) over Pᵀ(u), dP(u+2) over dSᵀ(u) — relies on tcgen05.mma executing in
// issue order).  One wait and one issue block per unit keep the MMA warp's serial overhead
// (≈ 6 cycles per instruction) from draining the shallow MMA queue between blocks.  Q/dO stream through
// NS = 5 stages (the look-ahead of 2 units plus ~2 units of HBM latency; per ring, see DkvCfg); every role prefetches
// the next item's descriptor so item boundaries do not expose a global-load round trip.  The
// item epilogue writes dK/dV from TMEM-loaded registers through row_map after a 4-lane chunk
// transpose (store_rows_xpose: 8 rows × 64 B per warp store; no smem staging, barrier or TMA).
// TMEM: S0 [0,UQ) · S1 [UQ,2UQ) · dP0 [128,128+UQ) · dP1 [128+UQ,..) · dV · dK.
// head_dim 256: dV and dK of the full head dim (2 × 256 fp32 columns) do not fit next to S / dP,
// so two launches each accumulate one 128-column half (p.ohalf; S / dP recomputed), and the
// unit is 32 queries (UQ) so that 3 Q/dO stages fit beside the 64 KB K and V tiles.
// MODE (head_dim 256): 0 = dV and dK together (head_dim ≤ 128: HO = HD); 1 = dV only, 2 = dK only,
// each over the full head dim (HO = 256) in its own launch.  The dV pass needs neither dP nor dS
// (Sᵀ → Pᵀ → dV) and loads no V; the dK pass skips the dV GEMM — 5 GEMMs per (key, query) pair over
// the two launches against the 6 of two head-dim halves that each recompute S and dP.
template <int HD, int UQ = 64, int MODE = 0>
struct DkvCfg {
  static constexpr int HO = MODE ? HD : (HD < 128 ? HD : 128);  // dK / dV head-dim columns per launch
  // MODE 3 (head_dim ≤ 128, one pass): K and V resident in TMEM (A operands of Sᵀ and dPᵀ: no
  // smem-bound SS MMAs), single Sᵀ / dPᵀ buffers, all 16 softmax warps on every unit (16 queries each)
  static constexpr bool kTm = MODE == 3;
  static constexpr int CW = kTm ? 16 : UQ / 2;    // query columns per softmax warp
  static constexpr int QBOX = UQ * 128;           // one 64-column TMA box of a Q / dO stage
  static constexpr int KT = 128 * HD * 2;  // K or V tile (128 keys)
  static constexpr int QT = UQ * HD * 2;   // Q or dO tile (UQ queries)
  // Q / dO stages: 5, except head_dim 256 with K and V resident (3); the dV pass loads no V, and its
  // 64 KB hold two more stages — with S look-ahead of 2 units, 3 stages leave no load in flight
  // head_dim 128 (one pass): 4, so that the dK / dV staging tile of the TMA-store epilogue fits
  static constexpr int NS = HD == 256 && MODE != 1 ? 3 : (HD == 128 && (MODE == 0 || MODE == 3) ? 4 : 5);
  // Q (+ lse2 / D windows) and dO have separate rings: NQ / ND stages.  Where dO is read only by
  // dP (the dK pass) its stage is released right after dP — 4 Q + 2 dO stages in the smem of 3 pairs,
  // so one more unit's loads are in flight; elsewhere dV reads dO at the end of the unit (NQ = ND).
  static constexpr int NQ = MODE == 2 && HD == 256 ? 4 : NS, ND = MODE == 2 && HD == 256 ? 2 : NS;
  static constexpr bool kEarlyDO = MODE == 2;  // dO stage released after dP
  static constexpr int OFF_K = 0, OFF_V = KT;
  static constexpr int OFF_Q = (MODE == 1 ? 1 : 2) * KT;  // [NQ]
  static constexpr int OFF_DO = OFF_Q + NQ * QT;    // [ND]
  static constexpr int VEC = UQ * 4;                // UQ floats of lse2 / D (16-B aligned window)
  static constexpr int OFF_LSE = OFF_DO + ND * QT;  // [NQ][VEC]
  static constexpr int OFF_DSUM = OFF_LSE + NQ * VEC;
  // single-pass launches (head_dim ≤ 128) write dK / dV through an SW128 staging tile and TMA stores
  // (128 rows × HO bf16, 64-column boxes of 16 KB); the head-dim-256 passes store rows directly
  static constexpr bool kTmaEpi = (MODE == 0 || MODE == 3) && HD <= 128;
  // single-pass launches (d ≤ 128): four dedicated epilogue warps (20-23, one per TMEM lane
  // quadrant) drain dK / dV, so the softmax groups never stall on an item boundary; registers are
  // rebalanced with setmaxnreg (softmax 96, the rest 48: 768 threads × 80 at launch)
  static constexpr bool kEpiWarps = kTmaEpi;
  static constexpr int THREADS = kEpiWarps ? 768 : 576;
  static constexpr int OFF_STG = kTmaEpi ? (OFF_DSUM + NQ * VEC + 1023) & ~1023 : OFF_DSUM + NQ * VEC;
  static constexpr int STG = kTmaEpi ? 128 * HO * 2 : 0;
  static constexpr int OFF_BAR = OFF_STG + STG;
  static constexpr int NUM_BARS = 12 + 2 * NQ + 2 * ND + 1;  // + epi_done
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16;  // dynamic smem base is 1 KB aligned
  static constexpr uint32_t DV_COL = 256, DK_COL = (MODE == 1 || MODE == 2) ? 256 : 256 + HO;
  // head_dim-256 passes: the item's K tile lives in TMEM (tcgen05.cp from the TMA-loaded smem tile at
  // the item's first unit), so Sᵀ = K·Qᵀ takes A from TMEM instead of re-reading 64 KB of smem per
  // 32-query unit: 16 K-steps × 8 columns in the columns S / dP leave free
  static constexpr bool kKTmem = HD == 256 && (MODE == 1 || MODE == 2);
  __host__ __device__ static constexpr uint32_t k_col(int s) {
    return kTm ? 128u + 8u * s : MODE == 1 ? 128u + 8u * s : (s < 8 ? 64u + 8u * s : 192u + 8u * (s - 8));
  }
  __host__ __device__ static constexpr uint32_t v_col(int s) { return 128u + uint32_t(HD / 2) + 8u * s; }  // MODE 3
  __host__ __device__ static constexpr uint32_t s_col(int b) { return kTm ? 0u : (b ? uint32_t(UQ) : 0u); }
  __host__ __device__ static constexpr uint32_t dp_col(int b) { return kTm ? 64u : 128u + (b ? uint32_t(UQ) : 0u); }
  // TMEM column of K-step j (16 queries) of Pᵀ / dSᵀ: warp chunks of CW queries sit at column
  // offsets part·CW, each packed into CW/2 columns as bf16 pairs
  __host__ __device__ static constexpr uint32_t a_col(int j) { return (j / (CW / 16)) * CW + (j % (CW / 16)) * 8; }
  static_assert(UQ == 64 || UQ == 32, "unit width");
  static_assert(DK_COL + HO <= 512 && DV_COL + HO <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
  static_assert(4 * 2001 * 8 <= (NQ + ND) * QT, "PROF trace fits the Q/dO stages");
};

// Item descriptors are loaded one item ahead; only the raw span loads are issued then and the
// derived counts are computed when the item becomes current (kv_item_finish), so the loads'
// latency never stalls a role at an item boundary.
// k0, ke, q_lo, q_hi: packed-stream rows (spans, masks); data rows are those + dl (seg_src).
struct KvItem {
  int k0, ke, dl, kh, q_lo, q_hi, nq, iters;
};
__device__ __forceinline__ KvItem kv_item_t(const BwdParams& p, int i, int4 t) {
  KvItem it;
  it.kh = i % p.Hkv;
  it.k0 = t.x;
  it.ke = t.y;
  it.dl = t.z;
  it.q_lo = __ldg(&p.cols_span[t.x].x);      // key spans are monotone inside a segment
  it.q_hi = __ldg(&p.cols_span[t.y - 1].y);
  return it;
}
__device__ __forceinline__ int4 kv_tile(const BwdParams& p, int i) { return __ldg(&p.tiles[i / p.Hkv]); }
__device__ __forceinline__ KvItem kv_item(const BwdParams& p, int i) { return kv_item_t(p, i, kv_tile(p, i)); }
template <int UQ>
__device__ __forceinline__ void kv_item_finish(const BwdParams& p, KvItem& it) {
  it.nq = max(0, (it.q_hi - it.q_lo + UQ - 1) / UQ);
  it.iters = it.nq * (p.H / p.Hkv);
}

// Walks this CTA's units in order: item i = sched_item(k) (attn_common.cuh), unit it within the
// item, k = ordinal of the item, u = ordinal of the unit.  The next item's descriptor is loaded
// one item ahead (its global loads overlap the current item).  Every key sees itself, so every
// item has iters ≥ 1.
template <int UQ>
struct UnitCursor {
  int i, it, k, u, n;
  int iq, hq;  // unit = (q head hq of the group, query tile iq): it = hq·nq + iq, kept without division
  KvItem itm, nxt;
  // The tile record of item k+2 is loaded one boundary before its spans (which index by it): no
  // role stalls on the dependent tiles → cols_span load chain at an item boundary.
  int4 tnn;
  __device__ __forceinline__ bool has_next() const { return sched_item(k + 1) < n; }
  __device__ __forceinline__ bool start(const BwdParams& p) {
    n = __ldg(p.ntiles) * p.Hkv;
    it = k = u = iq = hq = 0;
    i = sched_item(0);
    if (i >= n) return false;
    itm = kv_item(p, i);
    kv_item_finish<UQ>(p, itm);
    if (has_next()) nxt = kv_item(p, sched_item(1));
    if (sched_item(2) < n) tnn = kv_tile(p, sched_item(2));
    return true;
  }
  __device__ __forceinline__ bool next(const BwdParams& p) {
    ++u;
    if (++iq == itm.nq) {
      iq = 0;
      ++hq;
    }
    if (++it < itm.iters) return true;
    it = iq = hq = 0;
    i = sched_item(++k);
    if (i >= n) return false;
    itm = nxt;
    kv_item_finish<UQ>(p, itm);
    if (has_next()) {
      nxt = kv_item_t(p, sched_item(k + 1), tnn);
      if (sched_item(k + 2) < n) tnn = kv_tile(p, sched_item(k + 2));
    }
    return true;
  }
  __device__ __forceinline__ bool last() const { return it + 1 == itm.iters; }
  __device__ __forceinline__ int head(int group) const { return itm.kh * group + hq; }
  __device__ __forceinline__ int qb() const { return itm.q_lo + iq * UQ; }
};

// Warp roles (576 threads): warps 0-15 softmax — group g = w/8 takes the units with u%2 == g;
// warp w owns key rows 32·(w%4).. (TMEM lane quadrant w%4) and query columns [32·((w/4)%2), +32)
// of the 64-wide unit; in the epilogue all 16 warps split the head dim in quarters (w/4) and
// store their 2·HD/4 bytes of every dK / dV row directly.
// Warp 16 TMA producer, warp 17 TMEM allocator + MMA issuer.
constexpr int kDkvThreads = 576;

// dK / dV output tensor maps of the TMA-store epilogue: boxes of 128 / 64 / 32 / 16 / 8 rows × 64
// columns (a partial tile's rows [0, n & ~7) go out as the binary digits of n; its last n & 7 rows
// are stored directly)
struct DkvOutMaps {
  CUtensorMap dv[5], dk[5];
};

template <int HD, int UQ, bool PROF, int MODE = 0>
__global__ void __launch_bounds__(DkvCfg<HD, UQ, MODE>::THREADS, 1)
    k_bwd_dkdv(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
               const __grid_constant__ DkvOutMaps om, const BwdParams p) {
  using Cfg = DkvCfg<HD, UQ, MODE>;
  constexpr bool kDV = MODE != 2, kDK = MODE != 1;  // accumulators of this launch (dK needs dP / dS)
  constexpr int NQ = Cfg::NQ, ND = Cfg::ND, HO = Cfg::HO, CW = Cfg::CW;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* bar_kv_full = bars + 0;
  uint64_t* bar_kv_empty = bars + 1;   // committed after the item's last S / dP
  uint64_t* bar_dkv_full = bars + 2;
  uint64_t* bar_dkv_empty = bars + 3;  // 8 warp arrivals (the epilogue group): TMEM dV / dK drained
  uint64_t* bar_s_full = bars + 4;     // [2]
  uint64_t* bar_dp_full = bars + 6;    // [2]
  // bars + 8, + 9: spare (Pᵀ completion rides on the dSᵀ barrier: one MMA wait per unit)
  uint64_t* bar_ds_full = bars + 10;   // [2] 8 warp arrivals: dSᵀ written over dP
  uint64_t* bar_qd_full = bars + 12;        // [NQ] Q (+ lse2 / D windows) of a unit
  uint64_t* bar_qd_empty = bars + 12 + NQ;  // [NQ] committed after the unit's dK (dV pass: dV)
  uint64_t* bar_do_full = bars + 12 + 2 * NQ;       // [ND] dO of a unit
  uint64_t* bar_do_empty = bars + 12 + 2 * NQ + ND;  // [ND] after its last reader (dV, or dP)
  uint64_t* bar_epi_done = bars + 12 + 2 * NQ + 2 * ND;  // the item's dK store has read the staging tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // event trace (PROF builds with VLASIM_DBG & 2: the idle Q/dO stages hold 4 × 2001 words)
  unsigned long long* const trb =
      PROF && (p.dbg & 2) && blockIdx.x == 0 ? reinterpret_cast<unsigned long long*>(smem + Cfg::OFF_Q) : nullptr;
  const int group = p.H / p.Hkv;
  if (tid == 0) {
    if (smem_u32(smem) & 1023) __trap();
    mbar_init(bar_kv_full, 1);
    mbar_init(bar_kv_empty, 1);
    mbar_init(bar_dkv_full, 1);
    mbar_init(bar_dkv_empty, Cfg::kEpiWarps ? 4 : 8);
    mbar_init(bar_epi_done, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_s_full[b], 1);
      mbar_init(&bar_dp_full[b], 1);
      mbar_init(&bar_ds_full[b], Cfg::kTm ? 16 : 8);
    }
    mbar_init(bars + 8, 16);  // MODE 3: Pᵀ written (16 softmax warps)
    mbar_init(bars + 9, 4);   // MODE 3: dK drained (bar_dkv_empty then tracks dV alone)
    for (int s = 0; s < NQ; ++s) {
      mbar_init(&bar_qd_full[s], 1);
      mbar_init(&bar_qd_empty[s], 1);
    }
    for (int s = 0; s < ND; ++s) {
      mbar_init(&bar_do_full[s], 1);
      mbar_init(&bar_do_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 17) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 16) {
  // warpgroups 4-5 (producer, MMA, epilogue): registers handed to the softmax warpgroups
  if constexpr (Cfg::kEpiWarps) asm volatile("setmaxnreg.dec.sync.aligned.u32 48;\n" ::: "memory");
  if (Cfg::kEpiWarps && warp >= 18) {
    // ================================================ dK / dV epilogue warps (20-23; 18, 19 idle)
    // Per item: wait dkv_full; dV rows (this warp's lane quadrant, all HO columns) → SW128 staging
    // tile → TMA stores by one elected thread; once their smem reads are done, dK the same way;
    // TMEM released (dkv_empty, 4 arrivals) after the last dK load.  Partial tiles: 64/32/16/8-row
    // boxes + direct stores of the last n & 7 rows; the row_map layout stores every row directly.
    if constexpr (Cfg::kEpiWarps) {
      if (warp >= 20) {
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const bool elected = warp == 20 && lane == 0;
        uint8_t* stg = smem + Cfg::OFF_STG;
        const int64_t stride = int64_t(p.Hkv) * HD;
        const int n_items = __ldg(p.ntiles) * p.Hkv;
        int4 tn = kv_tile(p, sched_item(0) < n_items ? sched_item(0) : 0);
        for (int k = 0, i = sched_item(0); i < n_items; i = sched_item(++k)) {
          const int4 t = tn;
          if (sched_item(k + 1) < n_items) tn = kv_tile(p, sched_item(k + 1));
          const int kh = i % p.Hkv, k0 = t.x, n = t.y - t.x, row0 = t.x + t.z;
          const bool tail = r >= (n & ~7) && r < n;
          const int dst_row = r < n ? (p.row_map ? __ldg(p.row_map + k0 + r) : row0 + r) : -1;
          mbar_wait(bar_dkv_full, k & 1);
          tc_fence_after();
          auto pass = [&](uint32_t col0, float sc, __nv_bfloat16* out, const CUtensorMap* maps, bool last) {
            // TMEM → bf16 → staging (or direct rows), 32 columns at a time
#pragma unroll
            for (int cc = 0; cc < HO; cc += 32) {
              uint32_t v[32];
              tmem_ld32(tmem + lane_off + col0 + cc, v);
              tmem_wait_ld();
              uint32_t w[16];
#pragma unroll
              for (int j = 0; j < 16; ++j)
                w[j] = pack_bf16x2(__uint_as_float(v[2 * j]) * sc, __uint_as_float(v[2 * j + 1]) * sc);
              if (p.row_map) {
                if (dst_row >= 0) {
                  uint4* dst = reinterpret_cast<uint4*>(out + int64_t(dst_row) * stride + kh * HD + cc);
#pragma unroll
                  for (int t4 = 0; t4 < 4; ++t4) dst[t4] = make_uint4(w[4 * t4], w[4 * t4 + 1], w[4 * t4 + 2], w[4 * t4 + 3]);
                }
              } else {
#pragma unroll
                for (int t4 = 0; t4 < 4; ++t4) {
                  const int col = cc + 8 * t4;
                  *reinterpret_cast<uint4*>(stg + (col >> 6) * 16384 + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4)) =
                      make_uint4(w[4 * t4], w[4 * t4 + 1], w[4 * t4 + 2], w[4 * t4 + 3]);
                }
                if (tail) {
                  uint4* dst = reinterpret_cast<uint4*>(out + int64_t(row0 + r) * stride + kh * HD + cc);
#pragma unroll
                  for (int t4 = 0; t4 < 4; ++t4) dst[t4] = make_uint4(w[4 * t4], w[4 * t4 + 1], w[4 * t4 + 2], w[4 * t4 + 3]);
                }
              }
            }
            if (last || Cfg::kTm) {  // MODE 3: dV and dK accumulators released separately
              tc_fence_before();
              warp_arrive(Cfg::kTm && last ? bars + 9 : bar_dkv_empty);  // the next item's dV / dK may start
            }
            if (p.row_map) return;
            fence_proxy_async_smem();
            named_bar_sync(3, 128);  // staged
            if (elected) {
              if (n == 128) {
#pragma unroll
                for (int b = 0; b < HO / 64; ++b) tma_store_2d(&maps[0], kh * HD + b * 64, row0, stg + b * 16384);
              } else {
                int r0 = 0;
#pragma unroll
                for (int bi = 1; bi <= 4; ++bi) {
                  const int bh = 128 >> bi;
                  if (!(n & bh)) continue;
#pragma unroll
                  for (int b = 0; b < HO / 64; ++b)
                    tma_store_2d(&maps[bi], kh * HD + b * 64, row0 + r0, stg + b * 16384 + r0 * 128);
                  r0 += bh;
                }
              }
              bulk_commit();
              bulk_wait_read0();  // the staging tile may take the next pass
            }
            named_bar_sync(3, 128);
          };
          pass(Cfg::DV_COL, 1.f, p.dv, om.dv, false);
          pass(Cfg::DK_COL, p.scale, p.dk, om.dk, true);
        }
        if (elected) bulk_wait_all();
      }
    }
  } else if (warp == 16) {
    // ================================================ TMA producer
    if (lane == 0) {
      WaitProf<PROF> wp;
      TraceCtr trace(trb);
      UnitCursor<UQ> c;
      int s = 0, sd = 0;        // Q / dO stages of unit c.u
      uint32_t ph = 0, phd = 0;  // parities of those stages' current use
      for (bool v = c.start(p); v; v = c.next(p)) {
        if (c.it == 0) {
          if (c.k > 0) wp.template wait<1>(bar_kv_empty, (c.k - 1) & 1);
          trace(2, c.u);  // P: K/V load issued
          mbar_expect_tx(bar_kv_full, (kDK ? 2 : 1) * Cfg::KT);
#pragma unroll
          for (int j = 0; j < HD / 64; ++j) {
            tma_load_2d(smem + Cfg::OFF_K + j * 16384, &tmK, c.itm.kh * HD + j * 64, c.itm.k0 + c.itm.dl, bar_kv_full);
            if (kDK)  // V only for dP (the dV pass has no dP)
              tma_load_2d(smem + Cfg::OFF_V + j * 16384, &tmV, c.itm.kh * HD + j * 64, c.itm.k0 + c.itm.dl, bar_kv_full);
          }
          // the next item's K/V into L2 now: its load (single K/V buffer, issued only once this
          // item's last dP has run) then hits L2 at the item boundary
          if (c.has_next()) {
#pragma unroll
            for (int j = 0; j < HD / 64; ++j) {
              tma_prefetch_2d(&tmK, c.nxt.kh * HD + j * 64, c.nxt.k0 + c.nxt.dl);
              if (kDK) tma_prefetch_2d(&tmV, c.nxt.kh * HD + j * 64, c.nxt.k0 + c.nxt.dl);
            }
          }
        }
        const int h = c.head(group), qb = c.qb() + c.itm.dl;  // data row of the unit's first query
        const int sh = (-qb) & 3;  // 16-B aligned window in shifted copy sh (k_bwd_pre)
        const int64_t vo = sh * p.vec_copy + int64_t(h) * p.Tp + qb + sh;
        if (c.u >= NQ) wp.template wait<0>(&bar_qd_empty[s], ph ^ 1);
        trace(1, c.u);  // P: Q/dO load issued
        if (PROF && (p.dbg & 2)) {  // timing experiment: no Q/dO traffic (the trace lives in the Q stages)
          mbar_arrive(&bar_qd_full[s]);
          if (c.u >= ND) wp.template wait<0>(&bar_do_empty[sd], phd ^ 1);
          mbar_arrive(&bar_do_full[sd]);
        } else {
          mbar_expect_tx(&bar_qd_full[s], Cfg::QT + (kDK ? 2 : 1) * Cfg::VEC);
#pragma unroll
          for (int j = 0; j < HD / 64; ++j)
            tma_load_2d(smem + Cfg::OFF_Q + s * Cfg::QT + j * Cfg::QBOX, &tmQ, h * HD + j * 64, qb, &bar_qd_full[s]);
          bulk_load(smem + Cfg::OFF_LSE + s * Cfg::VEC, p.lse2 + vo, Cfg::VEC, &bar_qd_full[s]);
          if (kDK) bulk_load(smem + Cfg::OFF_DSUM + s * Cfg::VEC, p.dsum + vo, Cfg::VEC, &bar_qd_full[s]);
          if (c.u >= ND) wp.template wait<0>(&bar_do_empty[sd], phd ^ 1);
          mbar_expect_tx(&bar_do_full[sd], Cfg::QT);
#pragma unroll
          for (int j = 0; j < HD / 64; ++j)
            tma_load_2d(smem + Cfg::OFF_DO + sd * Cfg::QT + j * Cfg::QBOX, &tmdO, h * HD + j * 64, qb,
                        &bar_do_full[sd]);
        }
        if (++s == NQ) {
          s = 0;
          ph ^= 1;
        }
        if (++sd == ND) {
          sd = 0;
          phd ^= 1;
        }
      }
      wp.flush(p.prof);
    }
  } else if (warp == 17) {
    // ================================================ MMA issuer (whole warp, so descriptors and
    // counters stay in uniform registers; one elected lane issues).  Per unit u, in issue order:
    //   dV(u) · S(u+2) · dK(u) · dP(u+2)   — one issue block after one barrier wait.
    // Look-ahead S/dP stay inside the current item: the next item's first units are issued only
    // after the current item's last dK and its dkv_full commit, so the epilogue never waits
    // behind the next item's K/V load (single K/V buffer).  The warp's serial instruction
    // latency is the budget here, so stages and parities are counters, never u % NS.
    {
      constexpr uint32_t id_s = make_idesc_bf16(128, UQ, false, false);   // Sᵀ, dPᵀ
      constexpr uint32_t id_acc = make_idesc_bf16(128, HO, false, true);  // dV, dK (this launch's half)
      constexpr uint32_t QT16 = Cfg::QT >> 4;                             // stage stride, desc units
      WaitProf<PROF> wp;
      TraceCtr trace(lane == 0 && trb ? trb + 2001 : nullptr);
      const uint64_t dK0 = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_K), 16, 1024);
      const uint64_t dV0 = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_V), 16, 1024);
      const uint64_t dQk = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_Q), 16, 1024);     // K-major view
      const uint64_t dOk = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_DO), 16, 1024);
      // MN-major views of this launch's head-dim half (boxes of 64 columns, QBOX bytes apart)
      const uint32_t hoff = uint32_t(p.ohalf) * (HO / 64) * Cfg::QBOX;
      const uint64_t dQm = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_Q) + hoff, Cfg::QBOX, 1024);
      const uint64_t dOm = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_DO) + hoff, Cfg::QBOX, 1024);
      // Descriptor bases are made opaque where they are used (empty asm), so the per-MMA operand
      // descriptors are formed by uniform adds interleaved with the MMAs (hidden behind MMA-queue
      // back-pressure) instead of being hoisted into ~20 registers re-converted every unit.
      auto opaque = [](uint64_t v) {
        asm volatile("" : "+l"(v));
        return v;
      };
      auto mma_S = [&](uint32_t col, uint32_t soff) {
        const uint64_t a0 = opaque(dK0), b0 = opaque(dQk) + soff;
#pragma unroll
        for (int j = 0; j < HD / 16; ++j) {
          if constexpr (Cfg::kKTmem)
            umma_f16_ts(tmem + col, tmem + Cfg::k_col(j), sdesc_add(b0, (j / 4) * Cfg::QBOX + (j % 4) * 32), id_s,
                        j > 0 ? 1u : 0u);
          else
            umma_f16_ss(tmem + col, sdesc_add(a0, (j / 4) * 16384 + (j % 4) * 32),
                        sdesc_add(b0, (j / 4) * Cfg::QBOX + (j % 4) * 32), id_s, j > 0);
        }
      };
      auto mma_dP = [&](uint32_t col, uint32_t soff) {
        const uint64_t a0 = opaque(dV0), b0 = opaque(dOk) + soff;
#pragma unroll
        for (int j = 0; j < HD / 16; ++j)
          umma_f16_ss(tmem + col, sdesc_add(a0, (j / 4) * 16384 + (j % 4) * 32),
                      sdesc_add(b0, (j / 4) * Cfg::QBOX + (j % 4) * 32), id_s, j > 0);
      };
      if constexpr (MODE == 3) {
        // K / V resident in TMEM; single Sᵀ / dPᵀ buffers.  Per unit u of an item:
        //   wait Pᵀ(u) → dV(u) · Sᵀ(u+1)   (Sᵀ(u+1) over Pᵀ(u), after its reader in issue order)
        //   wait dSᵀ(u) → dK(u) · dPᵀ(u+1)
        // At an item's start: wait K/V, copy both tiles to TMEM (after the previous item's last
        // Sᵀ / dPᵀ in issue order; the smem tiles are released at once), then Sᵀ / dPᵀ of its first unit.
        uint64_t* bar_p_full = bars + 8;
        auto mma_St = [&](uint32_t soff) {  // Sᵀ = K·Qᵀ, A = K in TMEM, B = Q (K-major)
          const uint64_t b0 = opaque(dQk) + soff;
#pragma unroll
          for (int j = 0; j < HD / 16; ++j)
            umma_f16_ts(tmem + Cfg::s_col(0), tmem + Cfg::k_col(j), sdesc_add(b0, (j / 4) * Cfg::QBOX + (j % 4) * 32),
                        id_s, j > 0 ? 1u : 0u);
        };
        auto mma_dPt = [&](uint32_t soff) {  // dPᵀ = V·dOᵀ, A = V in TMEM
          const uint64_t b0 = opaque(dOk) + soff;
#pragma unroll
          for (int j = 0; j < HD / 16; ++j)
            umma_f16_ts(tmem + Cfg::dp_col(0), tmem + Cfg::v_col(j), sdesc_add(b0, (j / 4) * Cfg::QBOX + (j % 4) * 32),
                        id_s, j > 0 ? 1u : 0u);
        };
        UnitCursor<UQ> c;
        int u = 0;
        for (bool v = c.start(p); v;) {
          const int k = c.k;
          {  // item start
            const uint32_t st = uint32_t(u % NQ), sph = uint32_t((u / NQ) & 1);
            wp.template wait<0>(bar_kv_full, k & 1);
            wp.template wait<1>(&bar_qd_full[st], sph);
            wp.template wait<1>(&bar_do_full[st], sph);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t ka = opaque(dK0), va = opaque(dV0);
#pragma unroll
              for (int j = 0; j < HD / 16; ++j)
                tmem_cp_128x256b(tmem + Cfg::k_col(j), sdesc_add(ka, (j / 4) * 16384 + (j % 4) * 32));
#pragma unroll
              for (int j = 0; j < HD / 16; ++j)
                tmem_cp_128x256b(tmem + Cfg::v_col(j), sdesc_add(va, (j / 4) * 16384 + (j % 4) * 32));
              umma_commit(bar_kv_empty);  // K / V smem tiles free once copied
              mma_St(st * QT16);
              umma_commit(&bar_s_full[0]);
              mma_dPt(st * QT16);
              umma_commit(&bar_dp_full[0]);
            }
            __syncwarp();
          }
          for (;;) {
            const int it = c.it, iters = c.itm.iters;
            const bool nx = it + 1 < iters;
            const uint32_t cs = uint32_t(u % NQ), ns = uint32_t((u + 1) % NQ), nph = uint32_t(((u + 1) / NQ) & 1);
            const uint32_t par = uint32_t(u & 1);
            wp.template wait<5>(bar_p_full, par);
            trace(10, u);  // M: Pᵀ seen
            if (it == 0 && k > 0) wp.template wait<4>(bar_dkv_empty, (k - 1) & 1);  // previous item's dV drained
            if (nx) wp.template wait<1>(&bar_qd_full[ns], nph);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t acc0 = it > 0 ? 1u : 0u;
              const uint64_t om = opaque(dOm) + cs * QT16;
#pragma unroll
              for (int j = 0; j < UQ / 16; ++j)  // dV += Pᵀ·dO
                umma_f16_ts(tmem + Cfg::DV_COL, tmem + Cfg::s_col(0) + Cfg::a_col(j), sdesc_add(om, j * 2048), id_acc,
                            j > 0 ? 1u : acc0);
              umma_commit(&bar_do_empty[cs]);  // dPᵀ(u) and dV(u) have read dO(u)
              if (nx) {
                mma_St(ns * QT16);
                umma_commit(&bar_s_full[0]);
              }
            }
            __syncwarp();
            trace(11, u);  // M: dV + S issued
            wp.template wait<5>(&bar_ds_full[0], par);
            trace(12, u);  // M: dSᵀ seen
            if (it == 0 && k > 0) wp.template wait<4>(bars + 9, (k - 1) & 1);  // previous item's dK drained
            if (nx) wp.template wait<1>(&bar_do_full[ns], nph);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t acc0 = it > 0 ? 1u : 0u;
              const uint64_t qm = opaque(dQm) + cs * QT16;
#pragma unroll
              for (int j = 0; j < UQ / 16; ++j)  // dK += dSᵀ·Q
                umma_f16_ts(tmem + Cfg::DK_COL, tmem + Cfg::dp_col(0) + Cfg::a_col(j), sdesc_add(qm, j * 2048), id_acc,
                            j > 0 ? 1u : acc0);
              umma_commit(&bar_qd_empty[cs]);  // Sᵀ(u) and dK(u) have read Q(u)
              if (!nx) umma_commit(bar_dkv_full);
              if (nx) {
                mma_dPt(ns * QT16);
                umma_commit(&bar_dp_full[0]);
              }
            }
            __syncwarp();
            trace(13, u);  // M: dK + dP issued
            ++u;
            v = c.next(p);
            if (!v || !nx) break;
          }
        }
        if (lane == 0) wp.flush(p.prof + 8);
      } else if constexpr (MODE == 0) {
        // Single-pass launches: one cursor, stages / parities / TMEM buffers derived from the
        // unit ordinal (NQ = ND, compile-time).  S/dP of unit x are issued in the block of x − 2
        // when both lie in the same item; an item's first min(2, units) S/dP are issued after the
        // previous item's last block (item 0: before the loop) — no second cursor, no search.
        static_assert(NQ == ND, "single-pass stage rings");
        auto sdp = [&](int x, bool item_first, int k, bool item_last) {  // S and dP of unit x
          const uint32_t st = uint32_t(x % NQ), sph = uint32_t((x / NQ) & 1), bb = uint32_t(x & 1);
          if (item_first) wp.template wait<0>(bar_kv_full, k & 1);
          wp.template wait<1>(&bar_qd_full[st], sph);
          wp.template wait<1>(&bar_do_full[st], sph);
          tc_fence_after();
          if (elect_one()) {
            mma_S(Cfg::s_col(bb), st * QT16);
            umma_commit(&bar_s_full[bb]);
            mma_dP(Cfg::dp_col(bb), st * QT16);
            umma_commit(&bar_dp_full[bb]);
            if (item_last) umma_commit(bar_kv_empty);  // the item's last readers of K and V
          }
          __syncwarp();
        };
        UnitCursor<UQ> cc;
        bool vc = cc.start(p);
        if (vc) {
          sdp(0, true, 0, cc.itm.iters == 1);
          if (cc.itm.iters >= 2) sdp(1, false, 0, cc.itm.iters == 2);
        }
        for (int u = 0; vc; vc = cc.next(p), ++u) {
          const int it = cc.it, iters = cc.itm.iters;
          const bool la = it + 2 < iters;  // S/dP(u+2) in this block
          const uint32_t b = uint32_t(u & 1), cs = uint32_t(u % NQ);
          const uint32_t ls = uint32_t((u + 2) % NQ), lph = uint32_t(((u + 2) / NQ) & 1);
          if (la) {
            wp.template wait<1>(&bar_qd_full[ls], lph);
            wp.template wait<1>(&bar_do_full[ls], lph);
          }
          wp.template wait<5>(&bar_ds_full[b], uint32_t((u >> 1) & 1));
          if (it == 0 && cc.k > 0) wp.template wait<4>(bar_dkv_empty, (cc.k - 1) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t acc0 = it > 0 ? 1u : 0u;
            const uint64_t om = opaque(dOm) + cs * QT16, qm = opaque(dQm) + cs * QT16;
#pragma unroll
            for (int j = 0; j < UQ / 16; ++j)  // dV += Pᵀ·dO (A = Pᵀ in TMEM over the S columns)
              umma_f16_ts(tmem + Cfg::DV_COL, tmem + Cfg::s_col(b) + Cfg::a_col(j), sdesc_add(om, j * 2048), id_acc,
                          j > 0 ? 1u : acc0);
            if (la) {  // S(u+2) over Pᵀ(u): after dV(u) in issue order
              mma_S(Cfg::s_col(b), ls * QT16);
              umma_commit(&bar_s_full[b]);
            }
#pragma unroll
            for (int j = 0; j < UQ / 16; ++j)  // dK += dSᵀ·Q (A = dSᵀ in TMEM over the dP columns)
              umma_f16_ts(tmem + Cfg::DK_COL, tmem + Cfg::dp_col(b) + Cfg::a_col(j), sdesc_add(qm, j * 2048), id_acc,
                          j > 0 ? 1u : acc0);
            umma_commit(&bar_qd_empty[cs]);
            umma_commit(&bar_do_empty[cs]);  // dV(u) was dO's last reader
            if (it + 1 == iters) umma_commit(bar_dkv_full);
            if (la) {  // dP(u+2) over dSᵀ(u): after dK(u) in issue order
              mma_dP(Cfg::dp_col(b), ls * QT16);
              umma_commit(&bar_dp_full[b]);
              if (it + 3 == iters) umma_commit(bar_kv_empty);
            }
          }
          __syncwarp();
          if (it + 1 == iters && cc.has_next()) {  // the next item's first units (after its dkv_full)
            KvItem nx = cc.nxt;
            kv_item_finish<UQ>(p, nx);
            sdp(u + 1, true, cc.k + 1, nx.iters == 1);
            if (nx.iters >= 2) sdp(u + 2, false, cc.k + 1, nx.iters == 2);
          }
        }
        if (lane == 0) wp.flush(p.prof + 8);
      } else {
      UnitCursor<UQ> ca, cc;
      uint32_t as = 0, aph = 0;    // Q stage / parity of the look-ahead unit ca.u
      uint32_t ads = 0, adph = 0;  // its dO stage / parity
      bool va = false;
      auto adv_a = [&] {
        va = ca.next(p);
        if (++as == NQ) { as = 0; aph ^= 1; }
        if (++ads == ND) { ads = 0; adph ^= 1; }
      };
      auto issue_SdP = [&] {  // S and dP of unit ca.u (both buffers of its parity are free)
        trace(14, ca.u);  // M: boundary S/dP issue entered
        if (ca.it == 0) wp.template wait<0>(bar_kv_full, ca.k & 1);
        wp.template wait<1>(&bar_qd_full[as], aph);
        wp.template wait<1>(&bar_do_full[ads], adph);  // (dV pass: for dV(u), issued later)
        trace(15, ca.u);  // M: K/V + Q/dO ready
        tc_fence_after();
        const uint32_t bb = ca.u & 1;
        if (elect_one()) {
          if (Cfg::kKTmem && ca.it == 0) {  // the item's K tile → TMEM (in order after the previous
            const uint64_t a0 = opaque(dK0);  // item's last Sᵀ, before this item's first)
#pragma unroll
            for (int j = 0; j < HD / 16; ++j)
              tmem_cp_128x256b(tmem + Cfg::k_col(j), sdesc_add(a0, (j / 4) * 16384 + (j % 4) * 32));
            if (!kDK) umma_commit(bar_kv_empty);  // dV pass: K's smem tile is free once copied
          }
          mma_S(Cfg::s_col(bb), as * QT16);
          umma_commit(&bar_s_full[bb]);
          if (kDK) {
            mma_dP(Cfg::dp_col(bb), ads * QT16);
            umma_commit(&bar_dp_full[bb]);
            if (Cfg::kEarlyDO) umma_commit(&bar_do_empty[ads]);  // dP is dO's only reader here
          }
          if (ca.last() && !(Cfg::kKTmem && !kDK)) umma_commit(bar_kv_empty);  // the item's last readers of K and V
        }
        __syncwarp();
        adv_a();
      };
      va = ca.start(p);
      while (va && ca.k == 0 && ca.u < 2) issue_SdP();  // prologue: first item only
      uint32_t cs = 0, cds = 0, b = 0, ph = 0;  // Q / dO stages of cc.u; TMEM buffer cc.u & 1; its use parity
      for (bool vc = cc.start(p); vc; vc = cc.next(p)) {
        const uint32_t coff = cs * QT16, aoff = as * QT16, cdoff = cds * QT16, adoff = ads * QT16;
        const bool early = va && ca.u == cc.u + 2 && ca.k == cc.k;  // S/dP(u+2) in this unit's block
        const bool a_last = ca.last(), c_last = cc.last();
        const uint32_t acc0 = cc.it > 0 ? 1u : 0u;
        if (early) {
          wp.template wait<1>(&bar_qd_full[as], aph);
          wp.template wait<1>(&bar_do_full[ads], adph);
        }
        // dSᵀ(u) written ⇒ Pᵀ(u) written (each softmax warp stores P before dS): one wait per unit
        wp.template wait<5>(&bar_ds_full[b], ph);
        trace(12, cc.u);  // M: ds_full seen
        if (cc.it == 0 && cc.k > 0) wp.template wait<4>(bar_dkv_empty, (cc.k - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          // dV += Pᵀ·dO: A = Pᵀ in TMEM (queries 32j'..32j'+31 packed at S cols 32j'.. 32j'+15)
          const uint64_t om = opaque(dOm) + cdoff, qm = opaque(dQm) + coff;
          if (kDV) {
#pragma unroll
            for (int j = 0; j < UQ / 16; ++j)
              umma_f16_ts(tmem + Cfg::DV_COL, tmem + Cfg::s_col(b) + Cfg::a_col(j),
                          sdesc_add(om, j * 2048), id_acc, j > 0 ? 1u : acc0);
          }
          if (early) {  // S(u+2) over Pᵀ(u): after dV(u) in issue order
            mma_S(Cfg::s_col(b), aoff);
            umma_commit(&bar_s_full[b]);
            if (!kDK && a_last && !Cfg::kKTmem) umma_commit(bar_kv_empty);
          }
          if (kDK) {
            // dK += dSᵀ·Q: A = dSᵀ in TMEM over the dP columns
#pragma unroll
            for (int j = 0; j < UQ / 16; ++j)
              umma_f16_ts(tmem + Cfg::DK_COL, tmem + Cfg::dp_col(b) + Cfg::a_col(j),
                          sdesc_add(qm, j * 2048), id_acc, j > 0 ? 1u : acc0);
          }
          umma_commit(&bar_qd_empty[cs]);
          if (!Cfg::kEarlyDO) umma_commit(&bar_do_empty[cds]);  // dV(u) was dO's last reader
          if (c_last) umma_commit(bar_dkv_full);
          if (early && kDK) {  // dP(u+2) over dSᵀ(u): after dK(u) in issue order
            mma_dP(Cfg::dp_col(b), adoff);
            umma_commit(&bar_dp_full[b]);
            if (Cfg::kEarlyDO) umma_commit(&bar_do_empty[ads]);
            if (a_last) umma_commit(bar_kv_empty);
          }
        }
        __syncwarp();
        trace(13, cc.u);  // M: unit issued
        if (early) adv_a();
        // item boundary: the next item's first units (their buffers' previous readers, the dV /
        // dK of units ≤ u, are issued)
        while (va && ca.u <= cc.u + 2 && (ca.k == cc.k || (c_last && ca.k == cc.k + 1))) issue_SdP();
        if (++cs == NQ) cs = 0;
        if (++cds == ND) cds = 0;
        b ^= 1;
        ph ^= b ^ 1;  // flips after each pair of units (when b returns to 0)
      }
      if (lane == 0) wp.flush(p.prof + 8);
      }  // MODE != 0
    }
  }
  } else {
    if constexpr (Cfg::kEpiWarps) asm volatile("setmaxnreg.inc.sync.aligned.u32 96;\n" ::: "memory");
    if constexpr (MODE == 3) {
    // ================================================ softmax warps 0-15, MODE 3: every warp on every
    // unit — TMEM lane quadrant w%4 (32 keys) × query slice w/4 (16 of the unit's 64 queries)
    const int quad = warp & 3, part = warp >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int krow = quad * 32 + lane;
    const int c0 = part * CW;
    uint64_t* bar_p_full = bars + 8;
    WaitProf<PROF, 12> wp;
    TraceCtr trace(lane == 0 && warp == 0 && trb ? trb + 2001 * 2 : nullptr);
    UnitCursor<UQ> c;
    auto span_of = [&](int key) { return key < p.T ? __ldg(p.cols_span + key) : make_int2(0, 0); };
    int ss = 0;  // stage of unit c.u
    int2 ks = make_int2(0, 0), ks_nxt = ks;
    int u = 0;
    for (bool v = c.start(p); v; v = c.next(p), ++u) {
      if (c.it == 0) {  // this item's key spans were prefetched one item ahead (first item: now)
        ks = c.k == 0 ? span_of(c.itm.k0 + krow) : ks_nxt;
        if (c.has_next()) ks_nxt = span_of(c.nxt.k0 + krow);
      }
      const int s = ss;
      if (++ss == NQ) ss = 0;
      const uint32_t par = uint32_t(u & 1);
      const int qb = c.qb();
      const int c_lo = ks.x - qb - c0, c_hi = ks.y - qb - c0;  // visible query columns of this slice
      const bool all_full = __all_sync(0xffffffffu, c_lo <= 0 && c_hi >= CW);
      const bool none = __all_sync(0xffffffffu, c_hi <= 0 || c_lo >= CW);
      const int lo = max(c_lo, 0), hi = min(c_hi, CW);
      const uint32_t vis = hi <= lo ? 0u : ((hi >= 32 ? 0xffffffffu : (1u << hi) - 1u) & ~((1u << lo) - 1u));
      const float4* lse4 = reinterpret_cast<const float4*>(smem + Cfg::OFF_LSE + s * Cfg::VEC) + c0 / 4;
      const float4* dsum4 = reinterpret_cast<const float4*>(smem + Cfg::OFF_DSUM + s * Cfg::VEC) + c0 / 4;
      uint32_t pp[CW / 2];
      // ---- phase A: Sᵀ → Pᵀ (bf16 over this slice's first CW/2 S columns)
      wp.template wait<0>(&bar_s_full[0], par);
      trace(20, u);  // S: s_full seen
      const long long ta = wp.now();
      tc_fence_after();
      if (!none) {
        uint32_t sa[CW];
        tmem_ld16(tmem + lane_off + Cfg::s_col(0) + c0, sa);
        tmem_wait_ld();
        if (!all_full) {
#pragma unroll
          for (int q = 0; q < CW; ++q) sa[q] = ((vis >> q) & 1u) ? sa[q] : __float_as_uint(-INFINITY);
        }
        const float2 sl2v = make_float2(p.scale_log2, p.scale_log2);
#pragma unroll
        for (int j4 = 0; j4 < CW / 4; ++j4) {
          const float4 l = lse4[j4];
          const float2 a0 = f2_fma(make_float2(__uint_as_float(sa[4 * j4 + 0]), __uint_as_float(sa[4 * j4 + 1])), sl2v,
                                   make_float2(-l.x, -l.y));
          const float2 a1 = f2_fma(make_float2(__uint_as_float(sa[4 * j4 + 2]), __uint_as_float(sa[4 * j4 + 3])), sl2v,
                                   make_float2(-l.z, -l.w));
          pp[2 * j4] = pack_bf16x2(ex2_approx(a0.x), ex2_approx(a0.y));
          pp[2 * j4 + 1] = pack_bf16x2(ex2_approx(a1.x), ex2_approx(a1.y));
        }
      } else {
#pragma unroll
        for (int j = 0; j < CW / 2; ++j) pp[j] = 0u;
      }
      tmem_st8(tmem + lane_off + Cfg::s_col(0) + c0, pp);
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(bar_p_full);
      trace(22, u);  // S: Pᵀ arrived
      wp.template add_since<4>(ta);
      // ---- phase B: dPᵀ → dSᵀ = Pᵀ ∘ (dPᵀ − D) → bf16 over this slice's first CW/2 dP columns
      wp.template wait<1>(&bar_dp_full[0], par);
      trace(24, u);  // S: dp_full seen
      const long long tb = wp.now();
      tc_fence_after();
      uint32_t pk[CW / 2];
      if (!none) {
        uint32_t dr[CW];
        tmem_ld16(tmem + lane_off + Cfg::dp_col(0) + c0, dr);
        tmem_wait_ld();
#pragma unroll
        for (int j4 = 0; j4 < CW / 4; ++j4) {
          const float4 dd = dsum4[j4];
          const int q = 4 * j4;
          const float p0 = __uint_as_float(pp[2 * j4] << 16), p1 = __uint_as_float(pp[2 * j4] & 0xFFFF0000u);
          const float p2 = __uint_as_float(pp[2 * j4 + 1] << 16), p3 = __uint_as_float(pp[2 * j4 + 1] & 0xFFFF0000u);
          const float2 d0 = f2_mul(make_float2(p0, p1), f2_add(make_float2(__uint_as_float(dr[q]), __uint_as_float(dr[q + 1])),
                                                               make_float2(-dd.x, -dd.y)));
          const float2 d1 = f2_mul(make_float2(p2, p3), f2_add(make_float2(__uint_as_float(dr[q + 2]), __uint_as_float(dr[q + 3])),
                                                               make_float2(-dd.z, -dd.w)));
          pk[2 * j4] = pack_bf16x2(d0.x, d0.y);
          pk[2 * j4 + 1] = pack_bf16x2(d1.x, d1.y);
        }
      } else {
#pragma unroll
        for (int j = 0; j < CW / 2; ++j) pk[j] = 0u;
      }
      tmem_st8(tmem + lane_off + Cfg::dp_col(0) + c0, pk);
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(&bar_ds_full[0]);
      trace(26, u);  // S: dSᵀ arrived
      wp.template add_since<5>(tb);
    }
    if (warp == 0 && lane == 0) wp.flush(p.prof + 16);
    } else {
    // ================================================ softmax warps 0-15
    const int g = warp >> 3, quad = warp & 3, part = warp >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int krow = quad * 32 + lane;
    const int c0 = (part & 1) * CW;
    WaitProf<PROF, 12> wp;
    TraceCtr trace(lane == 0 && (warp & 7) == 0 && trb ? trb + 2001 * (2 + (warp >> 3)) : nullptr);
    UnitCursor<UQ> c;
    auto span_of = [&](int key) { return key < p.T ? __ldg(p.cols_span + key) : make_int2(0, 0); };
    // keys past the tile's end belong to the next segment: never stored
    auto dst_of = [&](int key, int ke, int dl) {
      return key < ke ? (p.row_map ? __ldg(p.row_map + key) : key + dl) : -1;
    };
    int ss = 0;  // stage of unit c.u
    int2 ks = make_int2(0, 0), ks_nxt = ks;
    int dst_key = -1, dst_nxt = -1;
    for (bool v = c.start(p); v; v = c.next(p)) {
      if (c.it == 0) trace(36 + g, c.u);  // S: item start (after the cursor advance)
      if (c.it == 0) {  // this item's spans were prefetched one item ahead (first item: now)
        const int key = c.itm.k0 + krow;
        ks = c.k == 0 ? span_of(key) : ks_nxt;
        dst_key = c.k == 0 ? dst_of(key, c.itm.ke, c.itm.dl) : dst_nxt;
        if (c.has_next()) {
          const int nkey = c.nxt.k0 + krow;
          ks_nxt = span_of(nkey);
          dst_nxt = dst_of(nkey, c.nxt.ke, c.nxt.dl);
        }
      }
      const int s = ss;
      if (++ss == NQ) ss = 0;
      if ((c.u & 1) == g) {
        const uint32_t ph = (c.u >> 1) & 1;
        const int qb = c.qb();
        const int c_lo = ks.x - qb - c0, c_hi = ks.y - qb - c0;  // visible columns of this half
        const bool all_full = __all_sync(0xffffffffu, c_lo <= 0 && c_hi >= CW);
        const bool none = __all_sync(0xffffffffu, c_hi <= 0 || c_lo >= CW) || (PROF && (p.dbg & 1));  // ablation
        // visible-column bitmask (used only when some row of the warp is partial)
        const int lo = max(c_lo, 0), hi = min(c_hi, CW);
        const uint32_t vis = hi <= lo ? 0u : ((hi >= 32 ? 0xffffffffu : (1u << hi) - 1u) & ~((1u << lo) - 1u));
        if (c.it == 0) trace(38 + g, c.u);  // S: unit set up (before the s_full wait)
        const float4* lse4 = reinterpret_cast<const float4*>(smem + Cfg::OFF_LSE + s * Cfg::VEC) + c0 / 4;
        const float4* dsum4 = reinterpret_cast<const float4*>(smem + Cfg::OFF_DSUM + s * Cfg::VEC) + c0 / 4;
        uint32_t pp[CW / 2];  // Pᵀ row chunk as bf16 pairs: written over S, kept for phase B
        // ---- phase A: Sᵀ → Pᵀ (bf16 over the S columns)
        wp.template wait<0>(&bar_s_full[g], ph);
        trace(20 + g, c.u);  // S: s_full seen
        const long long ta = wp.now();
        tc_fence_after();
        if (!none) {
          uint32_t sa[CW];
          if constexpr (CW == 32) tmem_ld32(tmem + lane_off + Cfg::s_col(g) + c0, sa);
          else tmem_ld16(tmem + lane_off + Cfg::s_col(g) + c0, sa);
          tmem_wait_ld();
          // invisible columns → −∞ before the exponent (exp2 → 0) in one warp-uniform branch, so the
          // exponent loop below has no branch between its iterations
          if (!all_full) {
#pragma unroll
            for (int q = 0; q < CW; ++q) sa[q] = ((vis >> q) & 1u) ? sa[q] : __float_as_uint(-INFINITY);
          }
          const float2 sl2v = make_float2(p.scale_log2, p.scale_log2);
#pragma unroll
          for (int j4 = 0; j4 < CW / 4; ++j4) {
            const float4 l = lse4[j4];  // 128-bit broadcast load
            // packed FFMA2: s·scale·log2e − lse2, two columns per instruction (same rounding as FFMA)
            const float2 a0 = f2_fma(make_float2(__uint_as_float(sa[4 * j4 + 0]), __uint_as_float(sa[4 * j4 + 1])), sl2v,
                                     make_float2(-l.x, -l.y));
            const float2 a1 = f2_fma(make_float2(__uint_as_float(sa[4 * j4 + 2]), __uint_as_float(sa[4 * j4 + 3])), sl2v,
                                     make_float2(-l.z, -l.w));
            float e[4];
            e[0] = ex2_approx(a0.x);
            e[1] = ex2_approx(a0.y);
            e[2] = ex2_approx(a1.x);
            e[3] = ex2_approx(a1.y);
            pp[2 * j4] = pack_bf16x2(e[0], e[1]);
            pp[2 * j4 + 1] = pack_bf16x2(e[2], e[3]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < CW / 2; ++j) pp[j] = 0u;
        }
        if constexpr (CW == 32) tmem_st16(tmem + lane_off + Cfg::s_col(g) + c0, pp);
        else tmem_st8(tmem + lane_off + Cfg::s_col(g) + c0, pp);  // completion awaited with dS's (phase B)
        trace(22 + g, c.u);  // S: P written
        wp.template add_since<4>(ta);
        if constexpr (!kDK) {  // dV pass: Pᵀ is all the MMA needs (released on the dS barrier)
          tmem_wait_st();
          tc_fence_before();
          warp_arrive(&bar_ds_full[g]);
        } else {
        // ---- phase B: dPᵀ → dSᵀ = Pᵀ ∘ (dPᵀ − D) → bf16 over the dP columns (P as the dV GEMM saw it)
        wp.template wait<1>(&bar_dp_full[g], ph);
        trace(24 + g, c.u);  // S: dp_full seen
        const long long tb = wp.now();
        tc_fence_after();
        uint32_t pk[CW / 2];
        if (!none) {
          uint32_t dr[CW];
          if constexpr (CW == 32) tmem_ld32(tmem + lane_off + Cfg::dp_col(g) + c0, dr);
          else tmem_ld16(tmem + lane_off + Cfg::dp_col(g) + c0, dr);
          tmem_wait_ld();
#pragma unroll
          for (int j4 = 0; j4 < CW / 4; ++j4) {
            const float4 dd = dsum4[j4];  // 128-bit broadcast load
            const int q = 4 * j4;
            const float p0 = __uint_as_float(pp[2 * j4] << 16), p1 = __uint_as_float(pp[2 * j4] & 0xFFFF0000u);
            const float p2 = __uint_as_float(pp[2 * j4 + 1] << 16), p3 = __uint_as_float(pp[2 * j4 + 1] & 0xFFFF0000u);
            // packed FADD2 / FMUL2 (same rounding as the scalar forms)
            const float2 d0 = f2_mul(make_float2(p0, p1), f2_add(make_float2(__uint_as_float(dr[q]), __uint_as_float(dr[q + 1])),
                                                                 make_float2(-dd.x, -dd.y)));
            const float2 d1 = f2_mul(make_float2(p2, p3), f2_add(make_float2(__uint_as_float(dr[q + 2]), __uint_as_float(dr[q + 3])),
                                                                 make_float2(-dd.z, -dd.w)));
            pk[2 * j4] = pack_bf16x2(d0.x, d0.y);
            pk[2 * j4 + 1] = pack_bf16x2(d1.x, d1.y);
          }
        } else {
#pragma unroll
          for (int j = 0; j < CW / 2; ++j) pk[j] = 0u;
        }
        if constexpr (CW == 32) tmem_st16(tmem + lane_off + Cfg::dp_col(g) + c0, pk);
        else tmem_st8(tmem + lane_off + Cfg::dp_col(g) + c0, pk);
        tmem_wait_st();
        tc_fence_before();
        warp_arrive(&bar_ds_full[g]);
        trace(26 + g, c.u);  // S: ds arrived
        wp.template add_since<5>(tb);
        }  // phase B (dK)
      }
      if (!Cfg::kEpiWarps && c.last() && (c.u & 1) == g) {
        // ---- item epilogue, by the group that ran the item's last unit (the other group goes
        //      straight on to the next item's first unit): TMEM → registers → release TMEM →
        //      8-lane chunk transpose → stores of 4 rows × 128 B per warp instruction.  Warp
        //      (quadrant, half hh) owns HD/2 columns of its 32 dV and dK rows; dV, then dK.
        const long long te = wp.now();
        trace(30 + (warp >> 3), c.u);  // E: epilogue entered
        wp.template wait<3>(bar_dkv_full, c.k & 1);
        trace(32 + (warp >> 3), c.u);  // E: dkv_full seen
        tc_fence_after();
        const int hh = (warp >> 2) & 1;
        const int64_t stride = int64_t(p.Hkv) * HD;
        bool done = false;
        if (PROF && (p.dbg & 8)) {  // ablation: no epilogue work (TMEM released at once)
          tc_fence_before();
          warp_arrive(bar_dkv_empty);
          if (Cfg::kTmaEpi && (warp & 7) == 0 && lane == 0) mbar_arrive(bar_epi_done);
          done = true;
        }
        if constexpr (Cfg::kTmaEpi) {
          if (!done && p.row_map == nullptr) {
            // Each thread's key row r (its TMEM lane) goes into the SW128 staging tile as 16-B chunks
            // (no transposes); the group's elected thread writes the tile with TMA stores.  dV first;
            // dK is loaded from TMEM (TMEM drained) while dV's stores read the tile, then staged over it.
            constexpr int HC = HO / 2;  // columns of this warp half
            uint8_t* stg = smem + Cfg::OFF_STG;
            const int n = c.itm.ke - c.itm.k0, r = krow;
            const int row0 = c.itm.k0 + c.itm.dl;  // data row of the tile's first key
            const bool tail = r >= (n & ~7) && r < n;
            const bool elected = (warp & 7) == 0 && lane == 0;
            auto ld_pack = [&](uint32_t col, float sc, uint32_t (&w)[HC / 2]) {
#pragma unroll
              for (int cc = 0; cc < HC; cc += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + lane_off + col + cc, v);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  w[cc / 2 + j] = pack_bf16x2(__uint_as_float(v[2 * j]) * sc, __uint_as_float(v[2 * j + 1]) * sc);
              }
            };
            auto stage = [&](const uint32_t (&w)[HC / 2]) {
#pragma unroll
              for (int t = 0; t < HC / 8; ++t) {
                const int col = hh * HC + 8 * t;
                *reinterpret_cast<uint4*>(stg + (col >> 6) * 16384 + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4)) =
                    make_uint4(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3]);
              }
            };
            auto direct = [&](const uint32_t (&w)[HC / 2], __nv_bfloat16* base) {
              uint4* dst = reinterpret_cast<uint4*>(base + int64_t(row0 + r) * stride + c.itm.kh * HD + hh * HC);
#pragma unroll
              for (int t = 0; t < HC / 8; ++t) dst[t] = make_uint4(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3]);
            };
            auto issue = [&](const CUtensorMap* maps) {  // the group's elected thread
              if (n == 128) {
#pragma unroll
                for (int b = 0; b < HO / 64; ++b) tma_store_2d(&maps[0], c.itm.kh * HD + b * 64, row0, stg + b * 16384);
              } else {
                int r0 = 0;
#pragma unroll
                for (int bi = 1; bi <= 4; ++bi) {
                  const int bh = 128 >> bi;
                  if (!(n & bh)) continue;
#pragma unroll
                  for (int b = 0; b < HO / 64; ++b)
                    tma_store_2d(&maps[bi], c.itm.kh * HD + b * 64, row0 + r0, stg + b * 16384 + r0 * 128);
                  r0 += bh;
                }
              }
              bulk_commit();
              bulk_wait_read0();
            };
            if (c.k > 0) wp.template wait<3>(bar_epi_done, (c.k - 1) & 1);  // previous item's dK store read the tile
            uint32_t w[HC / 2];
            ld_pack(Cfg::DV_COL + hh * HC, 1.f, w);
            stage(w);
            if (tail) direct(w, p.dv);
            ld_pack(Cfg::DK_COL + hh * HC, p.scale, w);
            tc_fence_before();
            warp_arrive(bar_dkv_empty);  // TMEM drained: the next item's dV/dK may start
            trace(50, c.u);  // E: TMEM drained
            fence_proxy_async_smem();
            named_bar_sync(1 + g, 256);  // dV staged
            if (elected) issue(om.dv);
            named_bar_sync(1 + g, 256);  // dV's stores have read the tile
            stage(w);
            if (tail) direct(w, p.dk);
            fence_proxy_async_smem();
            named_bar_sync(1 + g, 256);  // dK staged
            if (elected) {
              issue(om.dk);
              mbar_arrive(bar_epi_done);
            }
            done = true;
          }
        }
        if (!done) {
        constexpr int HW = HO / 2 < 64 ? HO / 2 : 64;  // columns per transposed store pass
        uint32_t pw[HW / 2];
#pragma unroll
        for (int t = kDV ? 0 : 1; t < (kDK ? 2 : 1); ++t) {  // t = 0: dV, 1: dK (· scale)
          const float sc = t ? p.scale : 1.f;
#pragma unroll
          for (int h0 = 0; h0 < HO / 2; h0 += HW) {  // this warp's HO/2 columns, HW at a time
            const uint32_t col = (t ? Cfg::DK_COL : Cfg::DV_COL) + hh * (HO / 2) + h0;
            const int col0 = c.itm.kh * HD + p.ohalf * HO + hh * (HO / 2) + h0;
#pragma unroll
            for (int cc = 0; cc < HW; cc += 32) {
              uint32_t v[32];
              tmem_ld32(tmem + lane_off + col + cc, v);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 16; ++j)
                pw[cc / 2 + j] = pack_bf16x2(__uint_as_float(v[2 * j]) * sc, __uint_as_float(v[2 * j + 1]) * sc);
            }
            if (t == (kDK ? 1 : 0) && h0 + HW == HO / 2) {
              tc_fence_before();
              warp_arrive(bar_dkv_empty);  // TMEM drained: the next item's dV/dK may start
              trace(50, c.u);  // E: TMEM drained
            }
            if (!(PROF && (p.dbg & 4)))  // ablation: no dK / dV stores
              store_rows_xpose<HW / 8>(pw, dst_key, t ? p.dk : p.dv, stride, col0);
          }
        }
        }  // direct-store epilogue
        trace(51, c.u);  // E: stored
        trace(34 + (warp >> 3), c.u);  // E: epilogue done
        wp.template add_since<6>(te);
      }
    }
    bulk_wait_all();  // dK / dV row stores of the last item
    if (warp == 0 && lane == 0) wp.flush(p.prof + 16);  // 12 slots: 16..27
    }  // MODE != 3
  }
  tc_fence_before();
  __syncthreads();
  if (trb)  // copy CTA 0's event trace out
    for (int i = tid; i < 4 * 2001; i += int(blockDim.x)) p.prof[64 + i] = trb[i];
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
template <int HD, int BN, int KS, int VS>
struct DqCfg {
  static constexpr int TILE = 128 * HD * 2;          // Q / dO tile (128 rows)
  static constexpr int KTILE = BN * HD * 2;          // K / V tile (BN keys)
  static constexpr int OFF_Q = 0, OFF_DO = TILE;
  static constexpr int OFF_K = 2 * TILE;             // K ring [KS]: released after dQ
  static constexpr int OFF_V = OFF_K + KS * KTILE;   // V ring [VS]: released after dP
  // VS = 0 (head_dim 256): ONE ring of 3 slots shared by K and V.  K(g) is held until dQ(g), V(g)
  // only until dP(g), so with K(g) in slot g % 3 and V(g) in slot (g+1) % 3, K(g+1) reuses the slot
  // V(g) frees at dP(g) and V(g+2) the slot K(g) frees at dQ(g): the S(g+1) load no longer waits
  // for dQ(g−1) (split 2 K + 1 V rings: the MMA waited for K 28 % of the kernel)
  static_assert(VS > 0 || KS == 3, "unified K/V ring: 3 slots");
  // decoded item descriptors, written by the producer one item ahead: the softmax warps hold no
  // next-item state in registers (at the 96-register cap it spilled and exposed the loads)
  static constexpr int NDESC = 4;
  static constexpr int OFF_DESC = OFF_V + VS * KTILE;    // int4 [NDESC][2]
  static constexpr int OFF_BAR = OFF_DESC + NDESC * 32;
  static constexpr int NUM_BARS = 2 + 2 * KS + 2 * VS + 8 + 2 * NDESC;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16;  // dynamic smem base is 1 KB aligned
  // TMEM: BN 128 → S0 [0,128) · dP [128,256) · dQ [256,256+HD) · S1 [384,512)
  //       BN  64 → S0 [0,64) · S1 [64,128) · dP [128,192) · dQ [256,256+HD)   (HD up to 256)
  static constexpr uint32_t DP_COL = 128, DQ_COL = 256;
  __host__ __device__ static constexpr uint32_t s_col(int g) {
    return BN == 128 ? ((g & 1) ? 384u : 0u) : ((g & 1) ? 64u : 0u);
  }
  static_assert(BN == 128 ? DQ_COL + HD <= 384 : DQ_COL + HD <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
};

struct QItem {
  int q0, qe, dl, h, kh, kv_lo, kv_hi, nkv;
};
__device__ __forceinline__ int4 q_tile(const BwdParams& p, int i) { return __ldg(&p.tiles[i / p.H]); }
__device__ __forceinline__ QItem q_item_t(const BwdParams& p, int i, int4 t) {  // raw loads (see KvItem)
  QItem it;
  it.h = i % p.H;
  it.q0 = t.x;
  it.qe = t.y;
  it.dl = t.z;
  it.kh = it.h / (p.H / p.Hkv);
  it.kv_lo = __ldg(&p.rows_span[t.x].x);
  it.kv_hi = __ldg(&p.rows_span[t.y - 1].y);
  it.nkv = -1;
  return it;
}
__device__ __forceinline__ QItem q_item(const BwdParams& p, int i) { return q_item_t(p, i, q_tile(p, i)); }
__device__ __forceinline__ QItem q_item_cur(QItem it, int BN) {  // derived count, when the item is current
  it.nkv = max(0, (it.kv_hi - it.kv_lo + BN - 1) / BN);
  return it;
}

// Warp roles (576 threads): warps 0-15 softmax — warp w owns Q rows 32·(w%4).. (TMEM lane quadrant
// w%4) and key columns [BN/4·(w/4), +BN/4) of each BN-key tile; warp 16 TMA producer; warp 17
// TMEM allocator + MMA issuer.  BN = 128 for head_dim ≤ 128, 64 for head_dim 256 (TMEM / smem).
constexpr int kDqThreads = 576;

template <int HD, int BN, int KS, int VS, bool PROF>
__global__ void __launch_bounds__(kDqThreads, 1)
    k_bwd_dq(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO, const BwdParams p) {
  using Cfg = DqCfg<HD, BN, KS, VS>;
  constexpr int W = BN / 4;  // key columns per softmax warp
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* bar_qdo_full = bars + 0;
  uint64_t* bar_qdo_empty = bars + 1;
  uint64_t* bar_k_full = bars + 2;                  // [KS]
  uint64_t* bar_k_empty = bars + 2 + KS;            // [KS]
  uint64_t* bar_v_full = bars + 2 + 2 * KS;         // [VS]
  uint64_t* bar_v_empty = bars + 2 + 2 * KS + VS;   // [VS]
  uint64_t* bar_s_full = bars + 2 + 2 * KS + 2 * VS;  // [2]
  uint64_t* bar_dp_full = bar_s_full + 2;          // one per tile
  uint64_t* bar_p_full = bar_s_full + 3;           // [2] 16 warp arrivals (dS written over S buffer g%2)
  uint64_t* bar_dq_full = bar_s_full + 5;          // one per item
  uint64_t* bar_dq_empty = bar_s_full + 6;         // 16 warp arrivals
  uint64_t* bar_dp_free = bar_s_full + 7;          // 16 warp arrivals: phase B has loaded dP(g)
  uint64_t* bar_desc_full = bar_s_full + 8;        // [NDESC] producer wrote item m's descriptor
  uint64_t* bar_desc_empty = bar_desc_full + Cfg::NDESC;  // [NDESC] 16 warp arrivals: read
  int4* descs = reinterpret_cast<int4*>(smem + Cfg::OFF_DESC);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = __ldg(p.ntiles) * p.H, i0 = sched_item(0);
  // event trace (PROF builds with VLASIM_DBG & 2: the idle K/V stages hold 4 × 2001 words)
  unsigned long long* const trb =
      PROF && (p.dbg & 2) && blockIdx.x == 0 ? reinterpret_cast<unsigned long long*>(smem + Cfg::OFF_K) : nullptr;
  if (tid == 0) {
    mbar_init(bar_qdo_full, 1);
    mbar_init(bar_qdo_empty, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(&bar_k_full[s], 1);
      mbar_init(&bar_k_empty[s], 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(&bar_v_full[s], 1);
      mbar_init(&bar_v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_s_full[s], 1);
      mbar_init(&bar_p_full[s], 16);
    }
    mbar_init(bar_dp_full, 1);
    mbar_init(bar_dq_full, 1);
    mbar_init(bar_dq_empty, 16);
    mbar_init(bar_dp_free, 16);
    for (int d = 0; d < Cfg::NDESC; ++d) {
      mbar_init(&bar_desc_full[d], 1);
      mbar_init(&bar_desc_empty[d], 16);
    }
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
      TraceCtr trace(trb);
      int g = 0, k = 0;
      QItem nxt = q_item(p, i0 < n_items ? i0 : 0);
      // descriptor of item ordinal mm (decoded) into the ring: {q0, qe, dl, h}, {kv_lo, kv_hi, nkv, kh}
      auto put_desc = [&](int mm, const QItem& it) {
        const int d = mm % Cfg::NDESC;
        if (mm >= Cfg::NDESC) mbar_wait(&bar_desc_empty[d], ((mm / Cfg::NDESC) - 1) & 1);
        descs[2 * d] = make_int4(it.q0, it.qe, it.dl, it.h);
        descs[2 * d + 1] = make_int4(it.kv_lo, it.kv_hi, it.nkv, it.kh);
        mbar_arrive(&bar_desc_full[d]);  // release semantics: the stores above are visible
      };
      if (i0 < n_items) put_desc(0, q_item_cur(nxt, BN));
      // descriptor m+1 published at the start of item m from span loads issued one item earlier,
      // whose tile record was fetched one item before that (no dependent-load stall)
      QItem n1 = q_item(p, sched_item(1) < n_items ? sched_item(1) : 0);
      int4 t2 = q_tile(p, sched_item(2) < n_items ? sched_item(2) : 0);
      for (int m = 0, i = i0; i < n_items; i = sched_item(++m)) {
        const QItem itm = q_item_cur(nxt, BN);
        if (sched_item(m + 1) < n_items) {
          put_desc(m + 1, q_item_cur(n1, BN));
          nxt = n1;
          if (sched_item(m + 2) < n_items) {
            n1 = q_item_t(p, sched_item(m + 2), t2);
            if (sched_item(m + 3) < n_items) t2 = q_tile(p, sched_item(m + 3));
          }
        }
        if (itm.nkv == 0) continue;
        if (k > 0) mbar_wait(bar_qdo_empty, (k - 1) & 1);
        trace(1, g);  // P: Q/dO load issued
        mbar_expect_tx(bar_qdo_full, 2 * Cfg::TILE);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          tma_load_2d(smem + Cfg::OFF_Q + c * 16384, &tmQ, itm.h * HD + c * 64, itm.q0 + itm.dl, bar_qdo_full);
          tma_load_2d(smem + Cfg::OFF_DO + c * 16384, &tmdO, itm.h * HD + c * 64, itm.q0 + itm.dl, bar_qdo_full);
        }
        for (int j = 0; j < itm.nkv; ++j, ++g) {
          const int kv0 = itm.kv_lo + j * BN + itm.dl;  // data row
          // ring slots and their use ordinals (unified ring: K(g) → g % 3, V(g) → (g+1) % 3)
          const int ks = VS ? g % KS : g % 3, vs = VS ? g % VS : (g + 1) % 3;
          const int ku = VS ? g / KS : g / 3 + (g + 2) / 3, vu = VS ? g / VS : (g + 1) / 3 + g / 3;
          uint64_t* const vfull = VS ? bar_v_full : bar_k_full;
          uint64_t* const vempty = VS ? bar_v_empty : bar_k_empty;
          uint8_t* const vbase = smem + (VS ? Cfg::OFF_V : Cfg::OFF_K);
          if (ku > 0) mbar_wait(&bar_k_empty[ks], (ku - 1) & 1);
          if (PROF && (p.dbg & 2)) {  // timing experiment: no K/V traffic (the trace lives in the K ring)
            mbar_arrive(&bar_k_full[ks]);
          } else {
            mbar_expect_tx(&bar_k_full[ks], Cfg::KTILE);
#pragma unroll
            for (int c = 0; c < HD / 64; ++c)
              tma_load_2d(smem + Cfg::OFF_K + ks * Cfg::KTILE + c * (BN * 128), &tmK, itm.kh * HD + c * 64, kv0,
                          &bar_k_full[ks]);
          }
          if (vu > 0) mbar_wait(&vempty[vs], (vu - 1) & 1);
          if (PROF && (p.dbg & 2)) {
            mbar_arrive(&vfull[vs]);
          } else {
            mbar_expect_tx(&vfull[vs], Cfg::KTILE);
#pragma unroll
            for (int c = 0; c < HD / 64; ++c)
              tma_load_2d(vbase + vs * Cfg::KTILE + c * (BN * 128), &tmV, itm.kh * HD + c * 64, kv0, &vfull[vs]);
          }
        }
        ++k;
      }
    }
  } else if (warp == 17) {
    // ================================================ MMA issuer (whole warp; one elected lane
    // issues).  Per key tile g: S(g) · [dQ(g−1) after its dS] · dP(g).  At an item boundary the
    // previous item's last dQ is issued before waiting for the next item's Q/dO, so dq_full —
    // and the epilogue — never wait behind that load.
    {
      constexpr uint32_t id_kk0 = make_idesc_bf16(128, 0, false, false);  // S, dP: | N/8 << 17
      constexpr uint32_t id_dq = make_idesc_bf16(128, HD, false, true);    // dQ (A from TMEM, B MN-major)
      constexpr uint32_t T16 = Cfg::KTILE >> 4;                            // ring stage stride, desc units
      const uint64_t dQk = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_Q), 16, 1024);
      const uint64_t dOk = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_DO), 16, 1024);
      const uint64_t dKk = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_K), 16, 1024);
      const uint64_t dVk = make_sdesc_sw128(smem_u32(smem + (VS ? Cfg::OFF_V : Cfg::OFF_K)), 16, 1024);
      uint64_t* const vfull = VS ? bar_v_full : bar_k_full;
      uint64_t* const vempty = VS ? bar_v_empty : bar_k_empty;
      const uint64_t dKm = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_K), BN * 128, 1024);  // MN-major view
      int g = 0, k = 0;
      int ks = 0, vs = 0;          // K / V ring stages of tile g
      uint32_t kph = 0, vph = 0;   // their use parities
      bool pend = false;    // dQ of the previous tile not issued yet
      bool plast = false, pfirst = false;
      int pks = 0, pg = 0, pna = 4;  // its K stage, tile ordinal and active W-key slices
      TraceCtr trace(lane == 0 && trb ? trb + 2001 : nullptr);
      int pk = 0;  // item ordinal of the pending dQ
      auto do_dq = [&]() {
        mbar_wait(&bar_p_full[pg & 1], (pg >> 1) & 1);
        trace(10, pg);  // M: p_full seen
        if (pfirst && pk > 0) mbar_wait(bar_dq_empty, (pk - 1) & 1);  // previous item's dQ drained
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = tmem + Cfg::s_col(pg);
#pragma unroll
          for (int s = 0; s < BN / 16; ++s)  // dS: keys Wp..Wp+W−1 packed at S cols Wp .. Wp+W/2−1
            if (s < pna * (W / 16))
              umma_f16_ts(tmem + Cfg::DQ_COL, a + (s / (W / 16)) * W + (s % (W / 16)) * 8,
                          sdesc_add(dKm, s * 2048) + pks * T16, id_dq, (!pfirst || s > 0) ? 1u : 0u);
          umma_commit(&bar_k_empty[pks]);
          if (plast) umma_commit(bar_dq_full);
        }
        __syncwarp();
        trace(11, pg);  // M: dQ issued
        pend = false;
      };
      QItem nxt = q_item(p, i0 < n_items ? i0 : 0);
      int4 tn = q_tile(p, sched_item(1) < n_items ? sched_item(1) : 0);  // tile record one item ahead
      for (int m = 0, i = i0; i < n_items; i = sched_item(++m)) {
        const QItem itm = q_item_cur(nxt, BN);
        if (sched_item(m + 1) < n_items) {
          nxt = q_item_t(p, sched_item(m + 1), tn);
          if (sched_item(m + 2) < n_items) tn = q_tile(p, sched_item(m + 2));
        }
        if (itm.nkv == 0) continue;
        if (pend) do_dq();  // previous item's last dQ before this item's Q/dO wait
        mbar_wait(bar_qdo_full, k & 1);
        for (int j = 0; j < itm.nkv; ++j, ++g) {
          // the item's last key tile: N = W · ⌈valid keys / W⌉ for S and dP, dQ over those keys
          const int na = j + 1 < itm.nkv ? 4 : (itm.kv_hi - itm.kv_lo - j * BN + W - 1) / W;
          const uint32_t id_kk = id_kk0 | (uint32_t(na * W / 8) << 17);
          if constexpr (VS == 0) {  // unified ring (producer comment): slots and use parities from g
            ks = g % 3;
            vs = (g + 1) % 3;
            kph = uint32_t(g / 3 + (g + 2) / 3) & 1u;
            vph = uint32_t((g + 1) / 3 + g / 3) & 1u;
          }
          mbar_wait(&bar_k_full[ks], kph);
          trace(12, g);  // M: K seen
          tc_fence_after();
          // S_g = Q·K_gᵀ into S buffer g%2 (its previous dS was consumed by dQ_{g-2}: issue order)
          if (elect_one()) {
#pragma unroll
            for (int s = 0; s < HD / 16; ++s)
              umma_f16_ss(tmem + Cfg::s_col(g), sdesc_add(dQk, (s / 4) * 16384 + (s % 4) * 32),
                          sdesc_add(dKk, (s / 4) * (BN * 128) + (s % 4) * 32) + ks * T16, id_kk, s > 0);
            umma_commit(&bar_s_full[g & 1]);
          }
          __syncwarp();
          // dP_g as soon as phase B(g−1) has loaded dP_{g−1} (dS goes over S, not dP), then dQ_{g−1}
          if (g > 0) mbar_wait(bar_dp_free, (g - 1) & 1);
          mbar_wait(&vfull[vs], vph);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int s = 0; s < HD / 16; ++s)
              umma_f16_ss(tmem + Cfg::DP_COL, sdesc_add(dOk, (s / 4) * 16384 + (s % 4) * 32),
                          sdesc_add(dVk, (s / 4) * (BN * 128) + (s % 4) * 32) + vs * T16, id_kk, s > 0);
            umma_commit(bar_dp_full);
            umma_commit(&vempty[vs]);
            if (j == itm.nkv - 1) umma_commit(bar_qdo_empty);
          }
          __syncwarp();
          trace(13, g);  // M: S + dP issued
          if (pend) do_dq();
          pend = true;
          pfirst = j == 0;
          plast = j == itm.nkv - 1;
          pks = ks;
          pg = g;
          pk = k;
          pna = na;
          if constexpr (VS > 0) {
            if (++ks == KS) { ks = 0; kph ^= 1; }
            if (++vs == VS) { vs = 0; vph ^= 1; }
          }
        }
        ++k;
      }
      if (pend) do_dq();
    }
  } else {
    // ================================================ softmax + epilogue warps 0-15 (query row, key-column quarter)
    const int quad = warp & 3, part = warp >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int r = quad * 32 + lane;
    const int c0 = part * W;
    TraceCtr trace(lane == 0 && (warp == 0 || warp == 4) && trb ? trb + 2001 * (2 + (part & 1)) : nullptr);
    int g = 0, k = 0;
    // row parameters of the next item are prefetched one item ahead
    auto load_row = [&](const QItem& it, int2& rs_, float& l_, float& d_) {
      const int rw = it.q0 + r;
      const bool v = rw < it.qe;  // rows past the tile's end belong to the next segment
      rs_ = rw < p.T ? __ldg(p.rows_span + rw) : make_int2(0, 0);
      l_ = v ? __ldg(p.lse2 + int64_t(it.h) * p.Tp + rw + it.dl) : 0.f;  // copy 0 (unshifted), data row
      d_ = v ? __ldg(p.dsum + int64_t(it.h) * p.Tp + rw + it.dl) : 0.f;
    };
    auto get_desc = [&](int mm, QItem& it, bool full) {  // item ordinal mm from the producer's ring
      const int d = mm % Cfg::NDESC;
      mbar_wait(&bar_desc_full[d], (mm / Cfg::NDESC) & 1);
      const int4 a = descs[2 * d];
      it.q0 = a.x;
      it.qe = a.y;
      it.dl = a.z;
      it.h = a.w;
      if (full) {
        const int4 b = descs[2 * d + 1];
        it.kv_lo = b.x;
        it.kv_hi = b.y;
        it.nkv = b.z;
        it.kh = b.w;
      }
    };
    int2 rs_n = make_int2(0, 0);
    float lse_n = 0.f, dsum_n = 0.f;
    if (i0 < n_items) {
      QItem f;
      get_desc(0, f, false);
      load_row(f, rs_n, lse_n, dsum_n);
    }
    for (int m = 0, i = i0; i < n_items; i = sched_item(++m)) {
      QItem itm;
      get_desc(m, itm, true);
      __syncwarp();
      warp_arrive(&bar_desc_empty[m % Cfg::NDESC]);  // (item m+1's row parameters read its slot below)
      const int2 rs = rs_n;
      const float lse2 = lse_n, dsum = dsum_n;
      if (sched_item(m + 1) < n_items) {
        QItem f;
        get_desc(m + 1, f, false);
        load_row(f, rs_n, lse_n, dsum_n);
      }
      if (itm.nkv == 0) continue;
      const int row = itm.q0 + r;
      const bool valid = row < itm.qe;  // rows past the tile's end belong to the next segment
      // the last key tile computes ⌈valid/W⌉ slices of W keys: this warp's slice is idle there
      const int j_skip = part >= (itm.kv_hi - itm.kv_lo - (itm.nkv - 1) * BN + W - 1) / W ? itm.nkv - 1 : -1;
      for (int j = 0; j < itm.nkv; ++j, ++g) {
        const uint32_t s_tm = tmem + lane_off + Cfg::s_col(g) + c0;
        const int kv0 = itm.kv_lo + j * BN + c0;
        const int c_lo = rs.x - kv0, c_hi = rs.y - kv0;
        // visible columns of this W-column slice as a bitmask (rows are intervals)
        const bool all_full = __all_sync(0xffffffffu, c_lo <= 0 && c_hi >= W);
        const int vlo = min(max(c_lo, 0), W), vhi = min(max(c_hi, 0), W);
        const uint32_t vm = vhi <= vlo ? 0u : ((vhi >= 32 ? 0xffffffffu : (1u << vhi) - 1u) & ~((1u << vlo) - 1u));
        if (j == j_skip) {
          // a slice past the last key tile's ⌈valid/W⌉ (S and dP ran with N = W · that): no loads,
          // exponentials or dS stores — only the barrier handshakes
          mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
          mbar_wait(bar_dp_full, g & 1);
          tc_fence_before();
          warp_arrive(bar_dp_free);
          warp_arrive(&bar_p_full[g & 1]);
          continue;
        }
        mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
        trace(20, g);  // S: s_full seen
        tc_fence_after();
        float2 pr[W / 2];  // P (fp32 pairs) kept for phase B
        const float2 sl2v = make_float2(p.scale_log2, p.scale_log2), nl2 = make_float2(-lse2, -lse2);
        {
          uint32_t sr[W];
          if constexpr (W == 32) tmem_ld32(s_tm, sr);
          else tmem_ld16(s_tm, sr);
          tmem_wait_ld();
          // masked columns → −∞ before the exponent (exp2 → 0) in a warp-uniform branch, so the
          // common all-visible tile runs no per-element select (it was if-converted before)
          if (!all_full) {
#pragma unroll
            for (int c = 0; c < W; ++c) sr[c] = ((vm >> c) & 1u) ? sr[c] : __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int t = 0; t < W / 2; ++t) {
            const float2 a = f2_fma(make_float2(__uint_as_float(sr[2 * t]), __uint_as_float(sr[2 * t + 1])), sl2v, nl2);
            pr[t] = make_float2(ex2_approx(a.x), ex2_approx(a.y));
          }
        }
        trace(21, g);  // S: phase A done
        mbar_wait(bar_dp_full, g & 1);
        trace(22, g);  // S: dp_full seen
        tc_fence_after();
        const float2 nd2 = make_float2(-dsum, -dsum);
        {
          uint32_t dr[W];
          if constexpr (W == 32) tmem_ld32(tmem + lane_off + Cfg::DP_COL + c0, dr);
          else tmem_ld16(tmem + lane_off + Cfg::DP_COL + c0, dr);
          tmem_wait_ld();
          tc_fence_before();
          warp_arrive(bar_dp_free);  // dP(g) is in registers: the MMA may issue dP(g+1)
          uint32_t dk[W / 2];
#pragma unroll
          for (int t = 0; t < W / 2; ++t) {  // dS = P ∘ (dP − D): FADD2 + FMUL2 per pair
            const float2 ds = f2_mul(pr[t], f2_add(make_float2(__uint_as_float(dr[2 * t]), __uint_as_float(dr[2 * t + 1])), nd2));
            dk[t] = pack_bf16x2(ds.x, ds.y);
          }
          if constexpr (W == 32) tmem_st16(s_tm, dk);  // dS over the first W/2 of this slice's S columns
          else tmem_st8(s_tm, dk);
        }
        tmem_wait_st();
        tc_fence_before();
        warp_arrive(&bar_p_full[g & 1]);
        trace(23, g);  // S: p_full arrived
      }
      // ---- item end: dQ = scale · acc → bf16 (half of the head dim per warp), coalesced store
      trace(30, g);  // E: epilogue entered
      mbar_wait(bar_dq_full, k & 1);
      trace(31, g);  // E: dq_full seen
      tc_fence_after();
      uint32_t pq[HD / 8];  // this quarter's HD/4 columns of dQ as bf16 pairs
#pragma unroll
      for (int c = 0; c < HD / 4; c += 32 > HD / 4 ? HD / 4 : 32) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + Cfg::DQ_COL + part * (HD / 4) + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < (HD / 4 < 32 ? HD / 8 : 16); ++t)
          pq[c / 2 + t] = pack_bf16x2(__uint_as_float(v[2 * t]) * p.scale, __uint_as_float(v[2 * t + 1]) * p.scale);
      }
      static_assert(HD / 4 <= 64, "dQ quarter held in registers");
      tc_fence_before();
      warp_arrive(bar_dq_empty);  // TMEM drained: the next item's first dQ MMA may start
      // registers → 4-lane chunk transpose → row-segment stores through row_map (8 rows × 64 B
      // per warp store; no smem staging, barrier or TMA op per row)
      {
        const int dst = valid ? (p.row_map ? __ldg(p.row_map + row) : row + itm.dl) : -1;
        store_rows_xpose<HD / 32>(pq, dst, p.dq, int64_t(p.H) * HD, itm.h * HD + part * (HD / 4));
      }
      trace(32, g);  // E: done
      ++k;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (trb)  // copy CTA 0's event trace out
    for (int i = tid; i < 4 * 2001; i += kDqThreads) p.prof[64 + i] = trb[i];
  if (warp == 17) tmem_dealloc<512>(tmem);
}

struct BwdWs {
  float* lse2;
  float* dsum;
  int2* rows_span;
  int2* cols_span;
  void* tiles;  // tile table (attn_tiles.cu)
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
  w->tiles = take(vlasim_host::tiles_bytes(int64_t(T), a->num_seqs));
  return off;
}

template <int HD>
int launch_bwd(const vlasim_attn_args* a, const vlasim_attn_grads* g, const BwdWs& w, cudaStream_t st) {
  using namespace vlasim_host;
  const int T = int(a->total_tokens), H = a->num_heads, Hkv = a->num_kv_heads;
  const int Tp = (T + 3) & ~3;
  mark_boundary(st);
  k_bwd_pre<HD><<<(T + kPreTokens - 1) / kPreTokens, 256, H * kPreTokens * sizeof(float), st>>>(
      static_cast<const __nv_bfloat16*>(a->o), static_cast<const __nv_bfloat16*>(g->dout), a->lse, w.lse2, w.dsum,
      w.rows_span, w.cols_span, a->cu_seqlens, a->prefix_len, a->num_seqs, a->mask_mode, T, Tp, H);
  VLASIM_LAUNCH_CHECK();
  mark_boundary(st);
  int4* tiles;
  int* ntiles;
  if (int rc = launch_build_tiles(a->cu_seqlens, a->seg_src, a->num_seqs, T, w.tiles, st, &tiles, &ntiles)) return rc;
  mark_boundary(st);
  const int64_t max_tiles = int64_t(T) / 128 + a->num_seqs;
  CUtensorMap tq, tk, tv, tdo;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (int rc = encode_tmap_2d(&tq, a->q, BF, T, uint64_t(H) * HD, uint64_t(H) * HD * 2, 128, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&tdo, g->dout, BF, T, uint64_t(H) * HD, uint64_t(H) * HD * 2, 128, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&tk, a->k, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, 128, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&tv, a->v, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, 128, 64, true)) return rc;
  CUtensorMap tk64, tv64;  // 64-key tiles of the dQ kernel (head_dim 256)
  if (HD == 256) {
    if (int rc = encode_tmap_2d(&tk64, a->k, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, 64, 64, true)) return rc;
    if (int rc = encode_tmap_2d(&tv64, a->v, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, 64, 64, true)) return rc;
  } else {
    tk64 = tk;
    tv64 = tv;
  }
  DkvOutMaps om;  // TMA-store epilogue (single-pass launches, head_dim ≤ 128)
  if (HD <= 128) {
    const uint32_t bh[5] = {128, 64, 32, 16, 8};
    for (int i = 0; i < 5; ++i) {
      if (int rc = encode_tmap_2d(&om.dv[i], g->dv, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, bh[i], 64, true))
        return rc;
      if (int rc = encode_tmap_2d(&om.dk[i], g->dk, BF, T, uint64_t(Hkv) * HD, uint64_t(Hkv) * HD * 2, bh[i], 64, true))
        return rc;
    }
  } else {
    memset(&om, 0, sizeof(om));
  }
  constexpr int UQ = HD == 256 ? 32 : 64;  // query unit of the dK/dV kernel
  CUtensorMap tqu, tdou;                    // UQ-row Q / dO boxes of the dK/dV kernel
  if (int rc = encode_tmap_2d(&tqu, a->q, BF, T, uint64_t(H) * HD, uint64_t(H) * HD * 2, UQ, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&tdou, g->dout, BF, T, uint64_t(H) * HD, uint64_t(H) * HD * 2, UQ, 64, true))
    return rc;
  BwdParams p;
  p.dq = static_cast<__nv_bfloat16*>(g->dq);
  p.dk = static_cast<__nv_bfloat16*>(g->dk);
  p.dv = static_cast<__nv_bfloat16*>(g->dv);
  p.row_map = g->row_map;
  p.lse2 = w.lse2;
  p.dsum = w.dsum;
  p.rows_span = w.rows_span;
  p.cols_span = w.cols_span;
  p.tiles = tiles;
  p.ntiles = ntiles;
  p.T = T;
  p.Tp = Tp;
  p.H = H;
  p.Hkv = Hkv;
  p.vec_copy = int64_t(H) * Tp + 512;
  p.scale = a->softmax_scale;
  p.scale_log2 = a->softmax_scale * kLog2e;
  p.dbg = getenv("VLASIM_DBG") ? atoi(getenv("VLASIM_DBG")) : 0;
  p.ohalf = 0;
  // head_dim 256: a dV pass (MODE 1) and a dK pass (MODE 2) over the full head dim (VLASIM_DKV_HALVES
  // selects the previous two head-dim halves, for comparison); head_dim ≤ 128: one launch (MODE 0)
  const bool halves = HD == 256 && getenv("VLASIM_DKV_HALVES");
  // head_dim ≤ 128: MODE 3 (K / V resident in TMEM); VLASIM_DKV_MODE0 selects the double-buffered
  // MODE 0 kernel for comparison
  static const bool mode0 = getenv("VLASIM_DKV_MODE0") != nullptr;
  const int nlaunch = HD == 256 ? 2 : 1;
  for (int half = 0; half < nlaunch; ++half) {
    const int grid = persistent_grid(max_tiles * Hkv, a->sm_budget);
    p.prof = prof_enabled() ? prof_buffer() : nullptr;
    p.ohalf = halves ? half : 0;
    constexpr int M1 = HD <= 128 ? 3 : 0;  // single-pass mode
    const bool tm = HD <= 128 && !mode0;
    auto kern = HD != 256 || halves
                    ? (tm ? (p.prof ? k_bwd_dkdv<HD, UQ, true, M1> : k_bwd_dkdv<HD, UQ, false, M1>)
                          : (p.prof ? k_bwd_dkdv<HD, UQ, true, 0> : k_bwd_dkdv<HD, UQ, false, 0>))
                : half == 0 ? (p.prof ? k_bwd_dkdv<HD, UQ, true, 1> : k_bwd_dkdv<HD, UQ, false, 1>)
                            : (p.prof ? k_bwd_dkdv<HD, UQ, true, 2> : k_bwd_dkdv<HD, UQ, false, 2>);
    const int smem = HD != 256 || halves ? (tm ? DkvCfg<HD, UQ, M1>::SMEM : DkvCfg<HD, UQ, 0>::SMEM)
                     : half == 0         ? DkvCfg<HD, UQ, 1>::SMEM
                                         : DkvCfg<HD, UQ, 2>::SMEM;
    const int threads = HD != 256 || halves ? (tm ? DkvCfg<HD, UQ, M1>::THREADS : DkvCfg<HD, UQ, 0>::THREADS)
                        : half == 0         ? DkvCfg<HD, UQ, 1>::THREADS
                                            : DkvCfg<HD, UQ, 2>::THREADS;
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, threads, smem, st>>>(tqu, tk, tv, tdou, om, p);
    VLASIM_LAUNCH_CHECK();
    if (p.prof)
      prof_report("k_bwd_dkdv", grid, st,
                  {"prod:qd_empty", "prod:kv_empty", "", "", "", "", "", "prod:total", "mma:kv_full",
                   "mma:qd_full", "", "mma:pt_full", "mma:dkv_empty", "mma:ds_full", "", "mma:total",
                   "smx:s_full", "smx:dp_full", "", "smx:dkv_full", "smx:phaseA", "smx:phaseB", "smx:epilogue", "",
                   "", "", "", "smx:total"});
  }
  mark_boundary(st);
  {
    constexpr int BN = HD == 256 ? 64 : 128;
    constexpr int KS = HD == 64 ? 5 : 3, VS = HD == 64 ? 4 : (HD == 128 ? 2 : 0);  // VS 0: unified K/V ring
    using Cfg = DqCfg<HD, BN, KS, VS>;
    auto kern = p.prof ? k_bwd_dq<HD, BN, KS, VS, true> : k_bwd_dq<HD, BN, KS, VS, false>;
    if (p.prof) prof_buffer();  // fresh counters / trace for this launch
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    const int grid = persistent_grid(max_tiles * H, a->sm_budget);
    kern<<<grid, kDqThreads, Cfg::SMEM, st>>>(tq, BN == 128 ? tk : tk64, BN == 128 ? tv : tv64, tdo, p);
    VLASIM_LAUNCH_CHECK();
    if (p.prof) prof_report("k_bwd_dq", grid, st, {});
  }
  mark_boundary(st);
  return VLASIM_OK;
}

}  // namespace

// FP8 backward: bf16 copies of the dequantised Q / K codes after the backward's own workspace
size_t fp8_bwd_extra(const vlasim_attn_args* a) {
  const size_t T = size_t(a->total_tokens), d = size_t(a->head_dim);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  return up(T * size_t(a->num_heads) * d * 2) + up(T * size_t(a->num_kv_heads) * d * 2);
}

extern "C" size_t vlasim_varlen_attn_workspace_size(const vlasim_attn_args* a, int backward) {
  if (!a) return 0;
  if (!backward) return vlasim_host::fwd_ws_bytes(a);  // forward: per-token visible spans + tiles
  BwdWs w;
  const size_t b = bwd_ws(&w, nullptr, a);
  return backward == 2 ? b + fp8_bwd_extra(a) : b;
}

extern "C" int vlasim_varlen_attn_bwd_cuda(const vlasim_attn_args* a, const vlasim_attn_grads* g, void* ws,
                                           size_t ws_bytes, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = validate_attn_args(a, false)) return rc;
  if (!g || !g->dout || !g->dq || !g->dk || !g->dv) return set_error(VLASIM_ECONFIG, "attention bwd: grads required");
  if (g->row_map && a->seg_src)
    return set_error(VLASIM_ECONFIG, "attention bwd: row_map and seg_src are exclusive (seg_src keeps source order)");
  BwdWs w;
  const size_t need = bwd_ws(&w, nullptr, a);
  if (!ws || ws_bytes < need) return set_error(VLASIM_ECONFIG, "attention bwd: workspace %zu < %zu", ws_bytes, need);
  bwd_ws(&w, ws, a);
  cudaStream_t st = as_stream(stream);
  switch (a->head_dim) {
    case 64: return launch_bwd<64>(a, g, w, st);
    case 128: return launch_bwd<128>(a, g, w, st);
    default: return launch_bwd<256>(a, g, w, st);
  }
}

// Backward of the FP8 Q/K forward (config 4): the gradients of o = attention(deq(q), deq(k), v) with
// deq(x) = value(code) · block scale (the straight-through gradient of the quantiser).  Q and K are
// dequantised once to bf16 (an HBM pass over the codes) and the bf16 backward kernels run on them
// with the FP8 forward's LSE; dQ / dK are with respect to the dequantised operands.
extern "C" int vlasim_varlen_attn_bwd_fp8qk_cuda(const vlasim_attn_args* a, const vlasim_attn_grads* g, void* ws,
                                                 size_t ws_bytes, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = validate_attn_args(a, true)) return rc;
  if (!g || !g->dout || !g->dq || !g->dk || !g->dv) return set_error(VLASIM_ECONFIG, "attention bwd: grads required");
  if (g->row_map && a->seg_src)
    return set_error(VLASIM_ECONFIG, "attention bwd: row_map and seg_src are exclusive (seg_src keeps source order)");
  BwdWs w;
  const size_t base = bwd_ws(&w, nullptr, a), need = base + fp8_bwd_extra(a);
  if (!ws || ws_bytes < need) return set_error(VLASIM_ECONFIG, "attention fp8 bwd: workspace %zu < %zu", ws_bytes, need);
  bwd_ws(&w, ws, a);
  cudaStream_t st = as_stream(stream);
  const int64_t T = a->total_tokens;
  uint8_t* wq = static_cast<uint8_t*>(ws) + base;
  uint8_t* wk = wq + ((size_t(T) * a->num_heads * a->head_dim * 2 + 255) & ~size_t(255));
  if (int rc = launch_fp8_dequant_bf16(static_cast<const uint8_t*>(a->q), a->q_scale, T, a->num_heads, a->head_dim,
                                       wq, st))
    return rc;
  if (int rc = launch_fp8_dequant_bf16(static_cast<const uint8_t*>(a->k), a->k_scale, T, a->num_kv_heads,
                                       a->head_dim, wk, st))
    return rc;
  vlasim_attn_args b = *a;
  b.q = wq;
  b.k = wk;
  b.q_scale = b.k_scale = nullptr;
  switch (a->head_dim) {
    case 64: return launch_bwd<64>(&b, g, w, st);
    case 128: return launch_bwd<128>(&b, g, w, st);
    default: return launch_bwd<256>(&b, g, w, st);
  }
}
