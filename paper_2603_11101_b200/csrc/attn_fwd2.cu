// attn_fwd2.cu — persistent block-diagonal varlen attention forward (sm_100a), head_dim 64/128.
//
// Same math and masking as attn_fwd.cu (vlasim::packed_attention), but
// persistent: grid = #SMs, each CTA walks work items (segment-aligned Q tile of ≤ 128 rows, head;
// attn_tiles.cu) on the boustrophedon schedule; Q is double-buffered so the next item's loads and
// first S MMAs overlap the current item's epilogue.
//
// Warp roles (576 threads):
//   warps 0-15 softmax + epilogue: warp w owns rows 32·(w%4).. (TMEM lane quadrant w%4) and
//              S columns [32·(w/4), +32); the four quarters of a row exchange their partial
//              row max / sum through smem (named barrier per quadrant), P (bf16) is written over
//              the S columns each quarter read, and each quarter handles HD/4 columns of O.
//   warp 16    TMA producer (Q double buffer, K/V ring) and, for bf16, the O stores: an item's
//              epilogue stages O (bf16, SW128) into the item's own Q buffer, idle by then, and
//              the producer writes it with two 128×64 TMA tensor stores before refilling that
//              buffer with the Q tile two items later (no LSU row scatter, no softmax stall).
//              A tile of n < 128 rows is stored as boxes of 64/32/16/8 rows (binary digits of
//              n & ~7); its last n & 7 rows are written by their softmax threads directly.
//   warp 17    TMEM allocator + tcgen05.mma issuer; S_g = Q·K_gᵀ is issued before PV_{g-1}
// TMEM (512 cols): S0 [0,128) · S1 [128,256) · O0 [256, 256+HD) · O1 after O0 (double-buffered so an
// item's epilogue can be deferred past the next item's first tile).
// Visible-key spans per token come from k_fwd_spans (one binary search per token).
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

constexpr float kLazyRescale = 8.0f;  // log2-domain row-max growth tolerated before rescaling O
constexpr int kDefaultPoly = 0;       // pairs of 16 per quarter tile exponentiated on the FMA pipe

__global__ void k_fwd_spans(const int32_t* __restrict__ cu, const int32_t* __restrict__ prefix, int nseq, int mask,
                            int T, int2* __restrict__ rows_span) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const RowSpan r = row_span(cu, prefix, nseq, mask, t, T);
  rows_span[t] = make_int2(r.lo, r.hi);
}

struct Fwd2Params {
  __nv_bfloat16* o;
  float* lse;
  const int2* rows_span;
  const int4* tiles;     // segment-aligned Q tiles {q0, qe, delta}, sorted by cost (attn_tiles.cu)
  const int* ntiles;     // device-side tile count
  const float* q_scale;  // FP8 only: [H, nbt] per-(head, 128-token block) E4M3 scales (d = 128)
  const float* k_scale;  // FP8 only: [Hkv, nbt]
  int T, H, Hkv, nbt;
  float scale_log2;
  unsigned long long* prof;  // [3 roles][8] wait cycles (PROF instantiation only)
};

template <int HD, int KS, int VS, bool FP8>
struct Fwd2Cfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int QK_ELEM = FP8 ? 1 : 2;           // Q/K element bytes (E4M3 codes or bf16)
  static constexpr int QK_BOX = 128 / QK_ELEM;          // elements per 128-B swizzle row
  static constexpr int Q_BYTES = BM * HD * QK_ELEM;
  static constexpr int K_BYTES = BN * HD * QK_ELEM;
  static constexpr int KV_BYTES = BN * HD * 2;          // one V tile (bf16)
  // Q ring of 3: an item's O is staged in its own (idle) Q buffer until the TMA store has read
  // it, so the Q tile two items ahead no longer waits for that store (the MMA waited for Q at
  // item boundaries ~16 % of the time with 2 buffers)
  static constexpr int NQ = 3;
  static constexpr int OFF_Q = 0;                        // [NQ]
  static constexpr int OFF_K = NQ * Q_BYTES;             // [KS] K ring
  static constexpr int OFF_V = OFF_K + KS * K_BYTES;     // [VS] V ring
  // FP8: the E4M3 Q buffer is too small to stage the bf16 O tile, so O gets its own staging tiles,
  // two (items alternate): the producer then has to have issued item k-3's store — not k-2's — before
  // loading item k's Q, so short items' Q / K loads never wait for the previous item's epilogue
  static constexpr int NOST = FP8 ? 2 : 0;
  static constexpr int OST_BYTES = BM * HD * 2;
  static constexpr int OFF_OST = OFF_V + VS * KV_BYTES;
  // row-max / row-sum exchange, 512 B per TMEM lane quadrant: bf16 maxima [2 parity][4 quarter][32
  // rows] for the tiles, fp32 sums [4 quarter][32 rows] once per item over the same bytes
  static constexpr int OFF_XCH = OFF_OST + NOST * OST_BYTES;
  // decoded item descriptors, written by the producer one item ahead (the softmax warps hold no
  // next-item state in registers)
  static constexpr int NDESC = 4;
  static constexpr int OFF_DESC = OFF_XCH + 4 * 512;   // int4 [NDESC][2]
  static constexpr int OFF_BAR = OFF_DESC + NDESC * 32;
  static constexpr int NUM_BARS = 2 * NQ + 2 * KS + 2 * VS + 9 + NQ + 2 + 2 * NDESC;
  // dynamic smem starts 1 KB aligned (no static smem in this kernel): no alignment slack
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr uint32_t S_COL = 0, O_COL = 256;
  static_assert(O_COL + 2 * HD <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
};

// Items are prefetched one ahead with raw span loads only; the key-tile count is derived when
// the item becomes current (fwd_item_cur), so the loads never stall a role at an item boundary.
// q0, qe, kv_lo, kv_hi: packed-stream rows (spans, masks); data rows are those + dl (seg_src).
struct FwdItem {
  int q0, qe, dl, h, kh, kv_lo, kv_hi, nkv;
};
// Item descriptors are built from the tile record (tiles[i / H]) and two span loads indexed by it.
// Roles look ahead so that no load result is consumed within the same item boundary: the tile
// record is fetched one boundary before the span loads that index by it (no dependent-load stall).
__device__ __forceinline__ int4 fwd_tile(const Fwd2Params& p, int i) { return __ldg(&p.tiles[i / p.H]); }
__device__ __forceinline__ FwdItem fwd_item_t(const Fwd2Params& p, int i, int4 t) {
  FwdItem it;
  it.h = i % p.H;
  it.q0 = t.x;
  it.qe = t.y;
  it.dl = t.z;
  it.kh = it.h / (p.H / p.Hkv);
  it.kv_lo = __ldg(&p.rows_span[t.x].x);      // spans are monotone inside a segment
  it.kv_hi = __ldg(&p.rows_span[t.y - 1].y);
  it.nkv = -1;
  return it;
}
__device__ __forceinline__ FwdItem fwd_item(const Fwd2Params& p, int i, int BN) {
  (void)BN;
  return fwd_item_t(p, i, fwd_tile(p, i));
}
__device__ __forceinline__ FwdItem fwd_item_cur(FwdItem it, int BN) {
  it.nkv = max(0, (it.kv_hi - it.kv_lo + BN - 1) / BN);
  return it;
}

constexpr int kFwdThreads = 576;

// The four column quarters' (bf16, rounded-up) maxima of a row, stored row-major [32 rows][4], read
// back as one 8-byte word: one LDS.64 per row instead of four LDS.U16.
__device__ __forceinline__ float xmax4(const __nv_bfloat16* xb, int lane) {
  const uint2 w = *reinterpret_cast<const uint2*>(xb + lane * 4);
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&w.x), b = *reinterpret_cast<const __nv_bfloat162*>(&w.y);
  const __nv_bfloat162 m = __hmax2(a, b);
  return fmaxf(__bfloat162float(m.x), __bfloat162float(m.y));
}

template <int HD, int KS, int VS, bool FP8, bool PROF, int NPOLY = 0>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                     const __grid_constant__ CUtensorMap tmO64, const __grid_constant__ CUtensorMap tmO32,
                     const __grid_constant__ CUtensorMap tmO16, const __grid_constant__ CUtensorMap tmO8,
                     const Fwd2Params p) {
  using Cfg = Fwd2Cfg<HD, KS, VS, FP8>;
  constexpr int BN = Cfg::BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  constexpr int NQ = Cfg::NQ;
  uint64_t* bar_q_full = bars;                          // [NQ]
  uint64_t* bar_q_empty = bars + NQ;                    // [NQ] FP8: the item's last S has read Q
  uint64_t* bar_k_full = bars + 2 * NQ;                 // [KS]
  uint64_t* bar_k_empty = bar_k_full + KS;              // [KS]
  uint64_t* bar_v_full = bar_k_full + 2 * KS;           // [VS]
  uint64_t* bar_v_empty = bar_v_full + VS;              // [VS]
  uint64_t* bar_s_full = bar_v_full + 2 * VS;           // [2]
  uint64_t* bar_p_full = bar_s_full + 2;         // [2] 16 warp arrivals
  uint64_t* bar_o_full = bar_s_full + 4;         // [2] per item: last PV landed in O[k%2]
  uint64_t* bar_o_empty = bar_s_full + 6;        // [2] 16 warp arrivals: epilogue drained O[k%2]
  uint64_t* bar_o_ready = bar_s_full + 8;        // one completion per PV
  uint64_t* bar_o_staged = bar_s_full + 9;       // [NQ] 16 warp arrivals: item's O staged in its Q buffer
  uint64_t* bar_ost_free = bar_o_staged + NQ;    // [2] FP8: O staging tile k&1 has been read by its TMA store
  uint64_t* bar_desc_full = bar_ost_free + 2;    // [NDESC] producer wrote item m's descriptor
  uint64_t* bar_desc_empty = bar_desc_full + Cfg::NDESC;  // [NDESC] 16 warp arrivals: read
  int4* descs = reinterpret_cast<int4*>(smem + Cfg::OFF_DESC);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = __ldg(p.ntiles) * p.H;
  const int i0 = sched_item(0);
  if (tid == 0) {
    for (int s = 0; s < NQ; ++s) {
      mbar_init(&bar_q_full[s], 1);
      mbar_init(&bar_q_empty[s], 1);
      mbar_init(&bar_o_staged[s], 16);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_s_full[s], 1);
      mbar_init(&bar_p_full[s], 16);
    }
    if (smem_u32(smem) & 1023) __trap();  // swizzle atoms need 1 KB alignment
    for (int s = 0; s < KS; ++s) {
      mbar_init(&bar_k_full[s], 1);
      mbar_init(&bar_k_empty[s], 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(&bar_v_full[s], 1);
      mbar_init(&bar_v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_o_full[s], 1);
      mbar_init(&bar_o_empty[s], 16);
    }
    mbar_init(bar_o_ready, 1);
    mbar_init(&bar_ost_free[0], 1);
    mbar_init(&bar_ost_free[1], 1);
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
      WaitProf<PROF> wp;
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      // Load order K0, K1, V0, K2, V1, …: K runs one tile ahead of V, so a K stage (freed as soon
      // as its S MMA completes) is refilled without waiting for the slower-retiring V stages.
      int g = 0, k = 0;
      int pv_g = -1, pv_kh = 0, pv_kv0 = 0;
      auto load_v = [&]() {
        const int vs = pv_g % VS;
        if (pv_g >= VS) wp.template wait<1>(&bar_v_empty[vs], ((pv_g / VS) - 1) & 1);
        uint8_t* sv = smem + Cfg::OFF_V + vs * Cfg::KV_BYTES;
        mbar_expect_tx(&bar_v_full[vs], Cfg::KV_BYTES);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) tma_load_2d(sv + c * BN * 128, &tmV, pv_kh * HD + c * 64, pv_kv0, &bar_v_full[vs]);
      };
      // bf16: item k's O is staged in Q buffer k % NQ; the producer writes it out (two 128×64 TMA
      // stores, or 64/32/16/8-row boxes) as soon as it is staged, and waits for the stores to have
      // read smem only when that buffer takes item k+NQ's Q.  Every item has ≥ 1 key tile (a query
      // sees itself), so every item runs an epilogue.
      int hq0[NQ] = {}, hh[NQ] = {}, hn[NQ] = {};
      int st = 0;  // items < st have had their O stores issued
      auto store_o = [&](int kk) {
        const int b = kk % NQ;
        wp.template wait<0>(&bar_o_staged[b], (kk / NQ) & 1);
        const uint8_t* so = smem + (FP8 ? Cfg::OFF_OST + (kk & 1) * Cfg::OST_BYTES : Cfg::OFF_Q + b * Cfg::Q_BYTES);
        if (hn[b] == 128) {
#pragma unroll
          for (int c = 0; c < HD / 64; ++c) tma_store_2d(&tmO, hh[b] * HD + c * 64, hq0[b], so + c * 16384);
        } else {  // rows [0, n & ~7) as 64/32/16/8-row boxes (1 KB-aligned starts keep the swizzle)
          int r0 = 0;
#pragma unroll
          for (int bh = 64; bh >= 8; bh >>= 1) {
            if (!(hn[b] & bh)) continue;
            const CUtensorMap* m = bh == 64 ? &tmO64 : bh == 32 ? &tmO32 : bh == 16 ? &tmO16 : &tmO8;
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) tma_store_2d(m, hh[b] * HD + c * 64, hq0[b] + r0, so + c * 16384 + r0 * 128);
            r0 += bh;
          }
        }
        bulk_commit();
        if constexpr (FP8) {
          bulk_wait_read0();
          mbar_arrive(&bar_ost_free[kk & 1]);  // item kk+2's O may be staged
        }
      };
      auto try_stores = [&](int upto) {  // O stores of items < upto that are staged already (never blocks)
        while (st < upto && mbar_test_wait(&bar_o_staged[st % NQ], (st / NQ) & 1)) store_o(st++);
      };
      // item ordinal mm's decoded descriptor into the ring: {q0, qe, dl, h}, {kv_lo, kv_hi, nkv, kh}
      auto put_desc = [&](int mm, const FwdItem& it) {
        const int d = mm % Cfg::NDESC;
        if (mm >= Cfg::NDESC) mbar_wait(&bar_desc_empty[d], ((mm / Cfg::NDESC) - 1) & 1);
        descs[2 * d] = make_int4(it.q0, it.qe, it.dl, it.h);
        descs[2 * d + 1] = make_int4(it.kv_lo, it.kv_hi, it.nkv, it.kh);
        mbar_arrive(&bar_desc_full[d]);
      };
      // descriptor m+1 is published at the start of item m (the softmax warps prefetch its row span
      // then), from span loads issued one item earlier; tile records are fetched one item before those
      FwdItem nxt = fwd_item(p, i0 < n_items ? i0 : 0, BN);
      if (i0 < n_items) put_desc(0, fwd_item_cur(nxt, BN));
      FwdItem n1 = fwd_item(p, sched_item(1) < n_items ? sched_item(1) : 0, BN);
      int4 t2 = fwd_tile(p, sched_item(2) < n_items ? sched_item(2) : 0);
      for (int m = 0, i = i0; i < n_items; i = sched_item(++m), ++k) {
        const FwdItem itm = fwd_item_cur(nxt, BN);
        if (sched_item(m + 1) < n_items) {
          put_desc(m + 1, fwd_item_cur(n1, BN));
          nxt = n1;
          if (sched_item(m + 2) < n_items) {
            n1 = fwd_item_t(p, sched_item(m + 2), t2);
            if (sched_item(m + 3) < n_items) t2 = fwd_tile(p, sched_item(m + 3));
          }
        }
        const int qs = k % NQ;
        if (k >= NQ) {  // buffer qs held item k-NQ: its Q reads (FP8) / its O store's reads (bf16) done
          if constexpr (FP8) {
            wp.template wait<0>(&bar_q_empty[qs], ((k / NQ) - 1) & 1);
          } else {
            while (st <= k - NQ) store_o(st++);
            bulk_wait_read0();
          }
        }
        // FP8: staging tile b is released through ost_free[b] (item e's epilogue waits for item e-2's
        // store); the store of item e-2 must be issued while item e is in flight — item e's epilogue
        // runs during item e+1, so the producer issues stores up to k-3 at item k (never a wait on
        // the previous item's epilogue, which would hold back item k's Q and K loads)
        if (FP8 && k >= 3)
          while (st <= k - 3) store_o(st++);
        hq0[qs] = itm.q0 + itm.dl;  // data row of the tile (O stores)
        hh[qs] = itm.h;
        hn[qs] = itm.qe - itm.q0;
        uint8_t* sq = smem + Cfg::OFF_Q + qs * Cfg::Q_BYTES;
        mbar_expect_tx(&bar_q_full[qs], Cfg::Q_BYTES);
#pragma unroll
        for (int c = 0; c < HD / Cfg::QK_BOX; ++c)
          tma_load_2d(sq + c * 128 * 128, &tmQ, itm.h * HD + c * Cfg::QK_BOX, itm.q0 + itm.dl, &bar_q_full[qs]);
        try_stores(k);
        for (int j = 0; j < itm.nkv; ++j, ++g) {
          const int ks = g % KS;
          if (g >= KS) wp.template wait<1>(&bar_k_empty[ks], ((g / KS) - 1) & 1);
          uint8_t* sk = smem + Cfg::OFF_K + ks * Cfg::K_BYTES;
          const int kv0 = itm.kv_lo + j * BN + itm.dl;  // data row
          mbar_expect_tx(&bar_k_full[ks], Cfg::K_BYTES);
#pragma unroll
          for (int c = 0; c < HD / Cfg::QK_BOX; ++c)
            tma_load_2d(sk + c * BN * 128, &tmK, itm.kh * HD + c * Cfg::QK_BOX, kv0, &bar_k_full[ks]);
          if (pv_g >= 0) load_v();
          pv_g = g;
          pv_kh = itm.kh;
          pv_kv0 = kv0;
          try_stores(k);
        }
      }
      if (pv_g >= 0) load_v();
      while (st < k) store_o(st++);
      bulk_wait_all();
      wp.flush(p.prof);
    }
  } else if (warp == 17) {
    // ================================================ MMA issuer (whole warp: descriptors and
    // counters in uniform registers; one elected lane issues)
    {
      constexpr uint32_t idesc_s0 = make_idesc_bf16(128, 0, false, false);  // | N/8 << 17
      constexpr uint32_t idesc_o = make_idesc_bf16(128, HD, false, true);
      constexpr uint32_t Q16 = Cfg::Q_BYTES >> 4, K16 = Cfg::K_BYTES >> 4, V16 = Cfg::KV_BYTES >> 4;
      const uint64_t dQ0 = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_Q), 16, 1024);
      const uint64_t dK0 = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_K), 16, 1024);
      const uint64_t dV0 = make_sdesc_sw128(smem_u32(smem + Cfg::OFF_V), BN * 128, 1024);  // MN-major
      WaitProf<PROF> wp;
      int g = 0, k = 0;
      int ks = 0, vs = 0;                // ring stages of tile g (K) and of the pending PV (V)
      uint32_t kph = 0, vph = 0;
      bool pend = false, pfirst = false, plast = false;  // pending PV (issued one tile late)
      int pg = 0, pk = 0, pnq = 4;  // its tile / item ordinals and active 32-key quarters
      auto do_pv = [&]() {
        wp.template wait<2>(&bar_p_full[pg & 1], (pg >> 1) & 1);
        if (pfirst && pk >= 2) wp.template wait<3>(&bar_o_empty[pk & 1], ((pk >> 1) - 1) & 1);
        wp.template wait<1>(&bar_v_full[vs], vph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_tm = tmem + Cfg::S_COL + (pg & 1) * 128;
          const uint64_t vd = dV0 + vs * V16;
#pragma unroll
          for (int s = 0; s < BN / 16; ++s)  // P: keys 32q..32q+31 packed at S cols 32q .. 32q+15
            if (s < 2 * pnq)
              umma_f16_ts(tmem + Cfg::O_COL + (pk & 1) * HD, a_tm + (s >> 1) * 32 + (s & 1) * 8,
                          sdesc_add(vd, s * 2048), idesc_o, (!pfirst || s > 0) ? 1u : 0u);
          umma_commit(&bar_v_empty[vs]);
          umma_commit(bar_o_ready);
          if (plast) umma_commit(&bar_o_full[pk & 1]);
        }
        __syncwarp();
        if (++vs == VS) { vs = 0; vph ^= 1; }
        pend = false;
      };
      FwdItem nxt = fwd_item(p, i0 < n_items ? i0 : 0, BN);
      int4 tn = fwd_tile(p, sched_item(1) < n_items ? sched_item(1) : 0);  // tile record one item ahead
      for (int m = 0, i = i0; i < n_items; i = sched_item(++m), ++k) {
        const FwdItem itm = fwd_item_cur(nxt, BN);
        if (sched_item(m + 1) < n_items) {  // prefetch (no load result used before the next boundary)
          nxt = fwd_item_t(p, sched_item(m + 1), tn);
          if (sched_item(m + 2) < n_items) tn = fwd_tile(p, sched_item(m + 2));
        }
        const int qs = k % NQ;
        const uint64_t qd = dQ0 + qs * Q16;
        wp.template wait<0>(&bar_q_full[qs], (k / NQ) & 1);
        for (int j = 0; j < itm.nkv; ++j, ++g) {
          wp.template wait<1>(&bar_k_full[ks], kph);
          tc_fence_after();
          const uint32_t d_s = tmem + Cfg::S_COL + (g & 1) * 128;
          const uint64_t kd = dK0 + ks * K16;
          // the item's last tile: N = 32 · ⌈valid keys / 32⌉
          const int nq = j + 1 < itm.nkv ? 4 : (itm.kv_hi - itm.kv_lo - j * BN + 31) >> 5;
          const uint32_t idesc_s = idesc_s0 | (uint32_t(nq * 4) << 17);
          if (elect_one()) {
            if constexpr (FP8) {  // kind::f8f6f4: 32 E4M3 elements (32 B) per K step
              const uint32_t idesc_f8 = make_idesc_e4m3(128, 0) | (uint32_t(nq * 4) << 17);
#pragma unroll
              for (int s = 0; s < HD / 32; ++s)
                umma_f8_ss(d_s, sdesc_add(qd, (s / 4) * 128 * 128 + (s % 4) * 32),
                           sdesc_add(kd, (s / 4) * BN * 128 + (s % 4) * 32), idesc_f8, s > 0);
            } else {
#pragma unroll
              for (int s = 0; s < HD / 16; ++s)
                umma_f16_ss(d_s, sdesc_add(qd, (s / 4) * 128 * 128 + (s % 4) * 32),
                            sdesc_add(kd, (s / 4) * BN * 128 + (s % 4) * 32), idesc_s, s > 0);
            }
            umma_commit(&bar_s_full[g & 1]);
            umma_commit(&bar_k_empty[ks]);
            if (FP8 && j == itm.nkv - 1) umma_commit(&bar_q_empty[qs]);  // bf16: freed by the O store
          }
          __syncwarp();
          if (++ks == KS) { ks = 0; kph ^= 1; }
          if (pend) do_pv();
          pend = true;
          pfirst = j == 0;
          plast = j == itm.nkv - 1;
          pg = g;
          pk = k;
          pnq = nq;
        }
      }
      if (pend) do_pv();
      if (lane == 0) wp.flush(p.prof + 8);
    }
  } else {
    // ================================================ softmax + epilogue warps 0-15
    const int quad = warp & 3, qp = warp >> 2;  // TMEM lane quadrant; column quarter
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int r = quad * 32 + lane;
    const int c0 = qp * 32;
    constexpr int OC = HD / 4;  // O columns per quarter
    __nv_bfloat16* xmax = reinterpret_cast<__nv_bfloat16*>(smem + Cfg::OFF_XCH + quad * 512);  // [2][4][32]
    float* xsum = reinterpret_cast<float*>(smem + Cfg::OFF_XCH + quad * 512);                  // [4][32]
    float sl2 = p.scale_log2;
    // Epilogue of item `ek` is deferred until the first tile of the next item has been handed to
    // the MMA warp, so the tensor core never idles on it (O is double-buffered in TMEM).
    WaitProf<PROF> wp;
    int ek = -1, e_row = 0, e_h = 0, e_n = 0;
    float e_m = 0.f, e_l = 0.f;
    auto epilogue = [&]() {
      const long long te = wp.now();
      wp.template wait<2>(&bar_o_full[ek & 1], (ek >> 1) & 1);
      tc_fence_after();
      uint32_t o[32];
      // OC ≤ 32 columns (HD 64: the upper 16 belong to the next quarter, unused); the row's scalars
      // and the LSE are computed while the TMEM load is in flight
      tmem_ld32(tmem + lane_off + Cfg::O_COL + (ek & 1) * HD + qp * OC, o);
      const bool valid = r < e_n;  // rows past the tile's end belong to the next segment
      const float inv_l = (valid && e_l > 0.f) ? 1.f / e_l : 0.f;
      if (valid && qp == 0)
        p.lse[static_cast<int64_t>(e_h) * p.T + e_row] = (e_m + __log2f(e_l)) * 0.69314718055994530942f;
      // staging tile: bf16 → this item's Q buffer; FP8 → O tile ek&1, once item ek-2's store has read it
      uint8_t* so = smem + (FP8 ? Cfg::OFF_OST + (ek & 1) * Cfg::OST_BYTES : Cfg::OFF_Q + (ek % NQ) * Cfg::Q_BYTES);
      tmem_wait_ld();
      tc_fence_before();
      warp_arrive(&bar_o_empty[ek & 1]);  // O is in registers: the buffer may take item ek+2
      uint32_t pk[16];
#pragma unroll
      for (int t = 0; t < OC / 2; ++t)
        pk[t] = pack_bf16x2(__uint_as_float(o[2 * t]) * inv_l, __uint_as_float(o[2 * t + 1]) * inv_l);
      {  // SW128 staging: 64-column box col / 64, 16-B chunk XOR row
        if (FP8 && ek > 1) wp.template wait<2>(&bar_ost_free[ek & 1], ((ek >> 1) - 1) & 1);
#pragma unroll
        for (int t = 0; t < OC / 8; ++t) {
          const int col = qp * OC + 8 * t;
          *reinterpret_cast<uint4*>(so + (col >> 6) * 16384 + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4)) =
              make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
        }
        fence_proxy_async_smem();
        warp_arrive(&bar_o_staged[ek % NQ]);  // the producer writes the tile out
        if (valid && r >= (e_n & ~7)) {       // the last n & 7 rows: no TMA box, stored here
          uint4* dst = reinterpret_cast<uint4*>(p.o + (int64_t(e_row) * p.H + e_h) * HD + qp * OC);
#pragma unroll
          for (int t = 0; t < OC / 8; ++t) dst[t] = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
        }
      }
      ek = -1;
      wp.template add_since<4>(te);
    };
    int g = 0, k = 0;
    auto get_desc = [&](int mm, FwdItem& it, bool full) {  // item ordinal mm from the producer's ring
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
    float qs_n = 1.f;  // FP8: the next item's row Q block scale (prefetched with its span)
    auto q_scale_of = [&](const FwdItem& f) {
      return __ldg(p.q_scale + int64_t(f.h) * p.nbt + min(f.q0 + r + f.dl, p.T - 1) / 128);
    };
    if (i0 < n_items) {
      FwdItem f;
      get_desc(0, f, false);
      rs_n = f.q0 + r < p.T ? __ldg(p.rows_span + f.q0 + r) : make_int2(0, 0);
      if constexpr (FP8) qs_n = q_scale_of(f);
    }
    for (int m = 0, i = i0; i < n_items; i = sched_item(++m), ++k) {
      FwdItem itm;
      get_desc(m, itm, true);
      __syncwarp();
      warp_arrive(&bar_desc_empty[m % Cfg::NDESC]);
      const int2 rs = rs_n;
      const float qs = qs_n;
      if (sched_item(m + 1) < n_items) {  // prefetch the next item's row span (and FP8 row scale)
        FwdItem f;
        get_desc(m + 1, f, false);
        rs_n = f.q0 + r < p.T ? __ldg(p.rows_span + f.q0 + r) : make_int2(0, 0);
        if constexpr (FP8) qs_n = q_scale_of(f);
      }
      const int row = itm.q0 + r;
      const uint32_t o_tm = tmem + lane_off + Cfg::O_COL + (k & 1) * HD + qp * OC;
      // FP8: the row's Q block scale (a segment-aligned tile may straddle two 128-token blocks)
      if constexpr (FP8) sl2 = p.scale_log2 * qs;
      (void)qs;
      float m_run = -INFINITY, l_run = 0.f;
      // FP8: this quarter's K block scales, one tile ahead in registers.  BN = the 128-token scale
      // block, so tile j of the quarter starts in data-row block kb0 + j at the same offset: the
      // split column cbq (keys before it take block kb0 + j's scale, the rest kb0 + j + 1's) is fixed
      // for the item, and each tile loads one new scale (its second block is the next tile's first)
      static_assert(!FP8 || BN == 128, "FP8 K scales assume 128-key tiles");
      const float* ksc = FP8 ? p.k_scale + int64_t(itm.kh) * p.nbt : nullptr;
      int kb0 = 0, cbq = 128;
      float k0n = 1.f, k1n = 1.f;
      if constexpr (FP8) {
        const int base = itm.kv_lo + c0 + itm.dl;  // data row of the quarter's first key (≥ 0)
        kb0 = base >> 7;
        cbq = 128 - (base & 127);
        k0n = __ldg(ksc + min(kb0, p.nbt - 1));
        k1n = __ldg(ksc + min(kb0 + 1, p.nbt - 1));
      }
      for (int j = 0; j < itm.nkv; ++j, ++g) {
        const uint32_t s_tm = tmem + lane_off + Cfg::S_COL + (g & 1) * 128 + c0;
        const int kv0 = itm.kv_lo + j * BN + c0;
        const float k0s = k0n, k1s = k1n;
        if constexpr (FP8)
          if (j + 1 < itm.nkv) {
            k0n = k1n;
            k1n = __ldg(ksc + min(kb0 + j + 2, p.nbt - 1));
          }
        if (j + 1 == itm.nkv && qp >= ((itm.kv_hi - kv0 + c0 + 31) >> 5)) {
          // The item's last key tile covers only ⌈valid/32⌉ quarters (its S MMA ran with N = 32 of
          // them): this quarter has no S, exponentials or P.  It still takes part in the row-max
          // exchange and the lazy O rescale of its columns.
          wp.template wait<0>(&bar_s_full[g & 1], (g >> 1) & 1);
          __nv_bfloat16* xb = xmax + (g & 1) * 128;
          xb[lane * 4 + qp] = __float2bfloat16_ru(-INFINITY);
          named_bar_sync(1 + quad, 128);
          float mt = xmax4(xb, lane);
          mt = (mt == -INFINITY) ? -INFINITY : mt * sl2;
          const bool grow = mt > m_run + kLazyRescale;
          const float alpha = grow ? ex2_approx(m_run - mt) : 1.f;  // same factor for l and O
          const bool rescale = __any_sync(0xffffffffu, grow && j > 0 && m_run != -INFINITY);
          if (grow) {
            l_run *= alpha;
            m_run = mt;
          }
          if (rescale) {
            wp.template wait<1>(bar_o_ready, (g - 1) & 1);
            tc_fence_after();
            uint32_t o[32];
            tmem_ld32(o_tm, o);
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < OC; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
            if constexpr (OC == 32) {
              tmem_st32(o_tm, o);
            } else {
              uint32_t o16[16];
#pragma unroll
              for (int t = 0; t < 16; ++t) o16[t] = o[t];
              tmem_st16(o_tm, o16);
            }
            tmem_wait_st();
          }
          tc_fence_before();
          warp_arrive(&bar_p_full[g & 1]);
          if (j == 0 && ek >= 0) epilogue();
          continue;
        }
        wp.template wait<0>(&bar_s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        uint32_t x[32];
        tmem_ld32(s_tm, x);
        tmem_wait_ld();
        const int c_lo = rs.x - kv0, c_hi = rs.y - kv0;
        // FP8: K block scale of this quarter.  A quarter inside one 128-key block (≈ 3 in 4) has a
        // uniform scale, folded into the row max and the exponent's multiplier (no per-element
        // work); a quarter straddling two blocks scales its columns (a quarter spans ≤ 2 blocks).
        float ksc = 1.f;
        if constexpr (FP8) {
          ksc = k0s;
          if (cbq < 32) {  // columns ≥ cbq: block kb0+j+1, rescaled by k1/k0 (one predicated FMUL each)
            const float rr = __fdividef(k1s, k0s);
            uint32_t hi;  // opaque to the compiler: bit tests become R2P + predicated FMULs, not 32 compares
            asm("mov.b32 %0, %1;" : "=r"(hi) : "r"(0xFFFFFFFFu << cbq));
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if ((hi >> c) & 1u) x[c] = __float_as_uint(__uint_as_float(x[c]) * rr);
          }
        }
        if (!__all_sync(0xffffffffu, c_lo <= 0 && c_hi >= 32)) {  // some row of the warp is partial
          const int vlo = min(max(c_lo, 0), 32), vhi = min(max(c_hi, 0), 32);
          const uint32_t vis = vhi <= vlo ? 0u : ((vhi >= 32 ? 0xffffffffu : (1u << vhi) - 1u) & ~((1u << vlo) - 1u));
#pragma unroll
          for (int c = 0; c < 32; ++c) x[c] = ((vis >> c) & 1u) ? x[c] : __float_as_uint(-INFINITY);
        }
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // 4 independent max chains (FMNMX3)
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u) mq[u] = fmax3(mq[u], __uint_as_float(x[c + 2 * u]), __uint_as_float(x[c + 2 * u + 1]));
        }
        float mt = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * ksc;  // scales are > 0
        // combine the four column quarters of this row
        // rounded up to bf16: every quarter uses the same offset, ≥ the row max (P ≤ 1)
        __nv_bfloat16* xb = xmax + (g & 1) * 128;
        xb[lane * 4 + qp] = __float2bfloat16_ru(mt);
        {
          const long long tb = wp.now();
          named_bar_sync(1 + quad, 128);
          wp.template add_since<3>(tb);
        }
        mt = xmax4(xb, lane);
        mt = (mt == -INFINITY) ? -INFINITY : mt * sl2;
        const bool grow = mt > m_run + kLazyRescale;
        const float alpha = grow ? ex2_approx(m_run - mt) : 1.f;  // same factor for l and O
        const bool rescale = __any_sync(0xffffffffu, grow && j > 0 && m_run != -INFINITY);
        if (grow) {
          l_run *= alpha;
          m_run = mt;
        }
        const float msub = (m_run == -INFINITY) ? 0.f : m_run;
        float2 lq[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // 4 independent sum chains (FADD2)
        const float2 sl2v = make_float2(sl2 * ksc, sl2 * ksc), nmv = make_float2(-msub, -msub);
        uint32_t pk[16];
        // NPOLY of the 16 pairs take 2^x on the FMA pipe (f2_ex2_poly) when no column of this warp's
        // quarter is masked (warp-uniform): MUFU.EX2 throughput bounds this loop, the FMA pipe has room
        const bool poly_ok = NPOLY > 0 && __all_sync(0xffffffffu, c_lo <= 0 && c_hi >= 32);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const float2 a = f2_fma(make_float2(__uint_as_float(x[2 * t]), __uint_as_float(x[2 * t + 1])), sl2v, nmv);
          float2 pe;
          if (NPOLY > 0 && (t % (16 / (NPOLY > 0 ? NPOLY : 1))) == 16 / (NPOLY > 0 ? NPOLY : 1) - 1 && poly_ok)
            pe = f2_ex2_poly(a);
          else
            pe = make_float2(ex2_approx(a.x), ex2_approx(a.y));
          lq[t & 1] = f2_add(lq[t & 1], pe);
          pk[t] = pack_bf16x2(pe.x, pe.y);
        }
        tmem_st16(s_tm, pk);  // P over the first 16 of this quarter's S columns
        l_run += (lq[0].x + lq[1].x) + (lq[0].y + lq[1].y);
        // lazy O rescale (after the exp pass: x is dead), before PV(g) is released by p_full
        if (rescale) {
          wp.template wait<1>(bar_o_ready, (g - 1) & 1);  // PV_{g-1} has landed in O
          tc_fence_after();
          uint32_t o[32];
          tmem_ld32(o_tm, o);  // OC ≤ 32 columns (HD 64: the upper 16 are rewritten unchanged... scaled)
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < OC; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
          if constexpr (OC == 32) {
            tmem_st32(o_tm, o);
          } else {
            uint32_t o16[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) o16[t] = o[t];
            tmem_st16(o_tm, o16);
          }
        }

        tmem_wait_st();
        tc_fence_before();
        warp_arrive(&bar_p_full[g & 1]);
        if (j == 0 && ek >= 0) epilogue();  // previous item, now that this tile is in flight
      }
      // combine the quarters' row sums and defer this item's epilogue
      // (over the quadrant's max bytes: every quarter has read the last tile's maxima first)
      named_bar_sync(1 + quad, 128);
      xsum[qp * 32 + lane] = l_run;
      named_bar_sync(1 + quad, 128);
      const float l_tot = (xsum[lane] + xsum[32 + lane]) + (xsum[64 + lane] + xsum[96 + lane]);
      named_bar_sync(1 + quad, 128);  // all quarters read before the bytes take the next maxima
      if (ek >= 0) epilogue();         // (only when this item had no tiles)
      if (itm.nkv > 0) {
        ek = k;
        e_row = row + itm.dl;  // data row (lse, tail-row stores)
        e_h = itm.h;
        e_n = itm.qe - itm.q0;
        e_m = m_run;
        e_l = l_tot;
      }
    }
    if (ek >= 0) epilogue();
    if (warp == 0 && lane == 0) wp.flush(p.prof + 16);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 17) tmem_dealloc<512>(tmem);
}

template <int HD, int KS, int VS, bool FP8>
int launch_fwd2(const vlasim_attn_args* a, int2* rows_span, void* tiles_buf, cudaStream_t st) {
  using namespace vlasim_host;
  using Cfg = Fwd2Cfg<HD, KS, VS, FP8>;
  const int T = int(a->total_tokens);
  // All host-side setup (tensor maps, kernel attributes) precedes the first launch: the prep kernels
  // take ~15 µs, and host work between them and the main launch would leave the GPU idle.
  CUtensorMap tq, tk, tv;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const auto QK = FP8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : BF;
  const uint64_t H = a->num_heads, Hkv = a->num_kv_heads;
  if (int rc = encode_tmap_2d(&tq, a->q, QK, T, H * HD, H * HD * Cfg::QK_ELEM, 128, Cfg::QK_BOX, true)) return rc;
  if (int rc = encode_tmap_2d(&tk, a->k, QK, T, Hkv * HD, Hkv * HD * Cfg::QK_ELEM, Cfg::BN, Cfg::QK_BOX, true)) return rc;
  if (int rc = encode_tmap_2d(&tv, a->v, BF, T, Hkv * HD, Hkv * HD * 2, Cfg::BN, 64, true)) return rc;
  CUtensorMap to;  // O tile stores (bf16 path): 128 rows × 64 columns, SW128
  if (int rc = encode_tmap_2d(&to, a->o, BF, T, H * HD, H * HD * 2, 128, 64, true)) return rc;
  CUtensorMap to64, to32, to16, to8;  // partial tiles
  if (int rc = encode_tmap_2d(&to64, a->o, BF, T, H * HD, H * HD * 2, 64, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&to32, a->o, BF, T, H * HD, H * HD * 2, 32, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&to16, a->o, BF, T, H * HD, H * HD * 2, 16, 64, true)) return rc;
  if (int rc = encode_tmap_2d(&to8, a->o, BF, T, H * HD, H * HD * 2, 8, 64, true)) return rc;
  // MUFU offload (f2_ex2_poly pairs of 16 per quarter tile): VLASIM_POLY = 0 / 2 / 4 / 8
  static const int npoly = [] {
    const char* pe = getenv("VLASIM_POLY");
    return pe ? atoi(pe) : kDefaultPoly;
  }();
  const bool prof = prof_enabled();
  auto kern = prof        ? attn_fwd2_kernel<HD, KS, VS, FP8, true>
            : npoly == 8 ? attn_fwd2_kernel<HD, KS, VS, FP8, false, 8>
            : npoly == 4 ? attn_fwd2_kernel<HD, KS, VS, FP8, false, 4>
            : npoly == 2 ? attn_fwd2_kernel<HD, KS, VS, FP8, false, 2>
                         : attn_fwd2_kernel<HD, KS, VS, FP8, false, 0>;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  mark_boundary(st);
  k_fwd_spans<<<(T + 255) / 256, 256, 0, st>>>(a->cu_seqlens, a->prefix_len, a->num_seqs, a->mask_mode, T, rows_span);
  VLASIM_LAUNCH_CHECK();
  int4* tiles;
  int* ntiles;
  if (int rc = launch_build_tiles(a->cu_seqlens, a->seg_src, a->num_seqs, T, tiles_buf, st, &tiles, &ntiles)) return rc;
  mark_boundary(st);
  Fwd2Params p;
  p.o = static_cast<__nv_bfloat16*>(a->o);
  p.lse = a->lse;
  p.rows_span = rows_span;
  p.tiles = tiles;
  p.ntiles = ntiles;
  p.q_scale = a->q_scale;
  p.k_scale = a->k_scale;
  p.T = T;
  p.H = a->num_heads;
  p.Hkv = a->num_kv_heads;
  p.nbt = (T + 127) / 128;
  p.scale_log2 = a->softmax_scale * 1.4426950408889634f;
  // the tile count is known on the device only: one CTA per SM (bounded by the worst case)
  const int64_t max_items = (int64_t(T) / 128 + a->num_seqs) * a->num_heads;
  const int grid = persistent_grid(max_items, a->sm_budget);
  if (prof) {
    p.prof = prof_buffer();
    kern<<<grid, kFwdThreads, Cfg::SMEM, st>>>(tq, tk, tv, to, to64, to32, to16, to8, p);
    VLASIM_LAUNCH_CHECK();
    return prof_report("attn_fwd2", grid, st,
                       {"prod:q_empty", "prod:kv_empty", "", "", "", "", "", "prod:total", "mma:q_full", "mma:k/v_full",
                        "mma:p_full", "mma:o_empty", "", "", "", "mma:total", "smx:s_full", "smx:o_ready",
                        "smx:o_full", "smx:xchg_bar", "smx:epilogue", "", "", "smx:total"});
  }
  p.prof = nullptr;
  kern<<<grid, kFwdThreads, Cfg::SMEM, st>>>(tq, tk, tv, to, to64, to32, to16, to8, p);
  VLASIM_LAUNCH_CHECK();
  mark_boundary(st);
  return VLASIM_OK;
}

}  // namespace

namespace vlasim_host {
// Forward for head_dim 64 / 128; the workspace holds the per-token spans (T int2).
// Forward workspace: per-token spans (T int2, 256-B aligned) then the tile table.
size_t fwd_ws_bytes(const vlasim_attn_args* a) {
  return ((size_t(a->total_tokens) * sizeof(int2) + 255) & ~size_t(255)) + tiles_bytes(a->total_tokens, a->num_seqs);
}
void* fwd_ws_tiles(const vlasim_attn_args* a, void* ws) {
  return static_cast<uint8_t*>(ws) + ((size_t(a->total_tokens) * sizeof(int2) + 255) & ~size_t(255));
}
int launch_fwd_persistent(const vlasim_attn_args* a, void* ws, size_t ws_bytes, cudaStream_t st) {
  const size_t need = fwd_ws_bytes(a);
  if (!ws || ws_bytes < need) return set_error(VLASIM_ECONFIG, "attention fwd: workspace %zu < %zu", ws_bytes, need);
  int2* spans = static_cast<int2*>(ws);
  if (a->head_dim == 64) return launch_fwd2<64, 4, 4, false>(a, spans, fwd_ws_tiles(a, ws), st);
  return launch_fwd2<128, 2, 2, false>(a, spans, fwd_ws_tiles(a, ws), st);
}
}  // namespace vlasim_host

// FP8 Q/K forward (config 4): q/k are E4M3 codes with per-(head, 128-token, 128-d) block scales
// (vlasim_fp8_quant_block_cuda); QKᵀ runs as tcgen05.mma kind::f8f6f4 and the block scales are
// applied to S in the softmax; P·V stays bf16.  head_dim 128 (one d block per head).
extern "C" int vlasim_varlen_attn_fwd_fp8qk_cuda(const vlasim_attn_args* a, void* ws, size_t ws_bytes,
                                                 vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = validate_attn_args(a, true)) return rc;
  if (a->head_dim != 128) return set_error(VLASIM_ECONFIG, "fp8 Q/K attention: head_dim must be 128");
  const size_t need = fwd_ws_bytes(a);
  if (!ws || ws_bytes < need) return set_error(VLASIM_ECONFIG, "attention fwd: workspace %zu < %zu", ws_bytes, need);
  return launch_fwd2<128, 2, 2, true>(a, static_cast<int2*>(ws), fwd_ws_tiles(a, ws), as_stream(stream));
}
