// attn_fwd.cu — block-diagonal varlen attention forward for sm_100a (bf16 in, fp32 accum).
//
// Replaces vlasim::packed_attention (multi-head = looped single head,
// SPEC.md:521) on the packed stream produced by the GPU packer.
//
// One CTA = one segment-aligned Q tile of ≤ 128 rows (attn_tiles.cu) × one head.  The tile's
// key range is the union of its rows' visible intervals; K/V tiles of BN rows are streamed from there, so no key
// block outside [first segment start, last visible key) is ever loaded or multiplied
// (tile skipping at sequence boundaries).  Inside a tile the block-diagonal / causal /
// prefix mask is a per-row interval test.
//
// Warp roles (192 threads):
//   warps 0-3  softmax + epilogue; thread i owns Q row i == TMEM lane i (32x32b loads)
//   warp 4     TMA producer: Q once, K/V ring of STAGES stages (SWIZZLE_128B boxes)
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (512 cols): S double buffer [0, 2·BN), O [2·BN, 2·BN+HD), P (bf16) double buffer
// after O.  Schedule per K tile j: S_j = Q·K_jᵀ (SS) is issued before PV_{j-1}, so the
// tensor core computes S_j while the softmax warps turn S_{j-1} into P_{j-1}.
// O rescaling is lazy: only when a row max grows by more than 2^8 (log2 domain).
#include <cfloat>
#include <climits>

#include "attn_common.cuh"
#include "common.hpp"
#include "sm100.cuh"

using namespace vlasim_dev;

namespace vlasim_host {
void* fwd_ws_tiles(const vlasim_attn_args* a, void* ws);
}

namespace {

struct FwdParams {
  __nv_bfloat16* o;
  float* lse;
  const int32_t* cu;
  const int32_t* prefix;
  const int4* tiles;  // segment-aligned Q tiles {q0, qe, delta}, sorted by cost (attn_tiles.cu)
  const int* ntiles;
  int nseq, T, H, Hkv, mask;
  float scale_log2;
};

template <int HD, int BN, int STAGES>
struct FwdCfg {
  static constexpr int BM = 128;
  static constexpr int Q_BYTES = BM * HD * 2;
  static constexpr int KV_BYTES = BN * HD * 2;  // one of K or V
  static constexpr int SMEM = Q_BYTES + STAGES * 2 * KV_BYTES + 1024;
  static constexpr uint32_t S_COL = 0;
  static constexpr uint32_t O_COL = 2 * BN;
  static constexpr uint32_t P_COL = 2 * BN + HD;
  static_assert(P_COL + BN <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
  static_assert(HD % 64 == 0 && BN % 32 == 0, "tile shape");
};

constexpr float kLazyRescale = 8.0f;  // log2-domain growth tolerated before rescaling O

template <int HD, int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const FwdParams p) {
  using Cfg = FwdCfg<HD, BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + Cfg::Q_BYTES;  // stage s: K at s*2*KV_BYTES, V right after

  __shared__ uint64_t bar_q, bar_kv_full[STAGES], bar_kv_empty[STAGES], bar_s_full[2], bar_p_full[2], bar_o_ready, bar_o_done;
  __shared__ uint32_t tmem_base_s;
  __shared__ int s_kv_lo, s_kv_hi;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (int(blockIdx.x) >= __ldg(p.ntiles) * p.H) return;  // grid sized for the worst-case tile count
  const int h = blockIdx.x % p.H;
  const int4 tile = __ldg(&p.tiles[blockIdx.x / p.H]);
  const int kh = h / (p.H / p.Hkv);
  const int q0 = tile.x, qe = tile.y, dl = tile.z;  // packed rows; data rows are + dl (seg_src)

  if (tid == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bar_kv_full[s], 1);
      mbar_init(&bar_kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_s_full[b], 1);
      mbar_init(&bar_p_full[b], 4);
    }
    mbar_init(&bar_o_ready, 1);
    mbar_init(&bar_o_done, 1);
    s_kv_lo = INT_MAX;
    s_kv_hi = INT_MIN;
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(&tmem_base_s);
  __syncthreads();

  RowSpan rs{0, 0, -1};
  if (tid < 128 && q0 + tid < qe) {  // rows past the tile's end belong to the next segment
    rs = row_span(p.cu, p.prefix, p.nseq, p.mask, q0 + tid, p.T);
    if (rs.lo < rs.hi) {
      atomicMin(&s_kv_lo, rs.lo);
      atomicMax(&s_kv_hi, rs.hi);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const int kv_lo = s_kv_lo;
  const int nkv = (s_kv_hi - kv_lo + BN - 1) / BN;

  if (warp == 4) {
    // ------------------------------------------------ TMA producer
    if (lane == 0 && nkv > 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_expect_tx(&bar_q, Cfg::Q_BYTES);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) tma_load_2d(sQ + c * Cfg::BM * 128, &tmQ, h * HD + c * 64, q0 + dl, &bar_q);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % STAGES;
        if (j >= STAGES) mbar_wait(&bar_kv_empty[st], ((j / STAGES) - 1) & 1);
        uint8_t* sk = sKV + st * 2 * Cfg::KV_BYTES;
        uint8_t* sv = sk + Cfg::KV_BYTES;
        const int kv0 = kv_lo + j * BN + dl;  // data row
        mbar_expect_tx(&bar_kv_full[st], 2 * Cfg::KV_BYTES);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) tma_load_2d(sk + c * BN * 128, &tmK, kh * HD + c * 64, kv0, &bar_kv_full[st]);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) tma_load_2d(sv + c * BN * 128, &tmV, kh * HD + c * 64, kv0, &bar_kv_full[st]);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0 && nkv > 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, BN, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, HD, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(&bar_q, 0);
      for (int j = 0; j <= nkv; ++j) {
        if (j < nkv) {
          const int st = j % STAGES;
          mbar_wait(&bar_kv_full[st], (j / STAGES) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sKV + st * 2 * Cfg::KV_BYTES);
          const uint32_t d_s = tmem + Cfg::S_COL + (j & 1) * BN;
#pragma unroll
          for (int s = 0; s < HD / 16; ++s) {
            const uint64_t a = make_sdesc_sw128(q_addr + (s / 4) * Cfg::BM * 128 + (s % 4) * 32, 16, 1024);
            const uint64_t b = make_sdesc_sw128(k_addr + (s / 4) * BN * 128 + (s % 4) * 32, 16, 1024);
            umma_f16_ss(d_s, a, b, idesc_s, s > 0);
          }
          umma_commit(&bar_s_full[j & 1]);
        }
        if (j > 0) {
          const int jj = j - 1, st = jj % STAGES;
          mbar_wait(&bar_p_full[jj & 1], (jj >> 1) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sKV + st * 2 * Cfg::KV_BYTES + Cfg::KV_BYTES);
          const uint32_t a_tm = tmem + Cfg::P_COL + (jj & 1) * (BN / 2);
#pragma unroll
          for (int s = 0; s < BN / 16; ++s) {
            const uint64_t b = make_sdesc_sw128(v_addr + s * 2048, BN * 128, 1024);
            umma_f16_ts(tmem + Cfg::O_COL, a_tm + s * 8, b, idesc_o, (jj > 0 || s > 0) ? 1u : 0u);
          }
          umma_commit(&bar_kv_empty[st]);
          umma_commit(&bar_o_ready);
          if (jj == nkv - 1) umma_commit(&bar_o_done);
        }
      }
    }
  } else {
    // ------------------------------------------------ softmax (warps 0-3)
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&bar_s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t r[BN];
#pragma unroll
      for (int c = 0; c < BN; c += 32) tmem_ld32(tmem + lane_off + Cfg::S_COL + sb * BN + c, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
      tmem_wait_ld();
      const int kv0 = kv_lo + j * BN;
      const int c_lo = rs.lo - kv0, c_hi = rs.hi - kv0;
      // invisible columns → −∞ in a warp-uniform branch (exp2 → 0); the row max over raw S with 4
      // independent FMNMX3 chains, scaled once (scale > 0)
      if (!__all_sync(0xffffffffu, c_lo <= 0 && c_hi >= BN)) {
#pragma unroll
        for (int c = 0; c < BN; ++c) r[c] = (c >= c_lo && c < c_hi) ? r[c] : __float_as_uint(-INFINITY);
      }
      float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < BN; c += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mq[u] = fmax3(mq[u], __uint_as_float(r[c + 2 * u]), __uint_as_float(r[c + 2 * u + 1]));
      }
      float mt = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
      mt = (mt == -INFINITY) ? -INFINITY : mt * sl2;
      const bool grow = mt > m_run + kLazyRescale;
      const float alpha = grow ? ex2_approx(m_run - mt) : 1.f;  // m_run = -inf → 0
      if (__any_sync(0xffffffffu, grow && j > 0 && m_run != -INFINITY)) {
        mbar_wait(&bar_o_ready, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_off + Cfg::O_COL + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tmem + lane_off + Cfg::O_COL + c, o);
        }
      }
      if (grow) {
        l_run *= alpha;
        m_run = mt;
      }
      const float msub = (m_run == -INFINITY) ? 0.f : m_run;
      // P = exp2(S·scale·log2e − m): FFMA2 for the argument, 4 independent FADD2 sum chains
      const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-msub, -msub);
      float2 lq[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < BN; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 a = f2_fma(make_float2(__uint_as_float(r[c + 2 * i]), __uint_as_float(r[c + 2 * i + 1])), sl2v, nmv);
          const float2 pe = make_float2(ex2_approx(a.x), ex2_approx(a.y));
          lq[i & 1] = f2_add(lq[i & 1], pe);
          pk[i] = pack_bf16x2(pe.x, pe.y);
        }
        tmem_st16(tmem + lane_off + Cfg::P_COL + sb * (BN / 2) + c / 2, pk);
      }
      l_run += (lq[0].x + lq[1].x) + (lq[0].y + lq[1].y);
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(&bar_p_full[sb]);
    }
    // ------------------------------------------------ epilogue: O / l → bf16, LSE
    // o_ready may trail the softmax by two phases here (S(nkv-1) only orders PV(nkv-3)), so its
    // parity is ambiguous: the epilogue waits on the dedicated last-PV barrier
    if (nkv > 0) {
      mbar_wait(&bar_o_done, 0);
      tc_fence_after();
    }
    const int row = q0 + tid;
    const bool valid = row < qe && rs.lo < rs.hi;
    const float inv_l = (valid && l_run > 0.f) ? 1.f / l_run : 0.f;
    __nv_bfloat16* orow = p.o + (static_cast<int64_t>(row + dl) * p.H + h) * HD;
#pragma unroll
    for (int c = 0; c < HD; c += 32) {
      uint32_t o[32];
      tmem_ld32(tmem + lane_off + Cfg::O_COL + c, o);
      tmem_wait_ld();
      if (valid) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * inv_l, __uint_as_float(o[2 * i + 1]) * inv_l);
        uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (valid) p.lse[static_cast<int64_t>(h) * p.T + row + dl] = (m_run + __log2f(l_run)) * 0.69314718055994530942f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc<512>(tmem);
}

template <int HD, int BN, int STAGES>
int launch_fwd(const vlasim_attn_args* a, void* tiles_buf, cudaStream_t st) {
  using namespace vlasim_host;
  using Cfg = FwdCfg<HD, BN, STAGES>;
  CUtensorMap tq, tk, tv;
  const uint64_t T = a->total_tokens;
  if (int rc = encode_tmap_2d(&tq, a->q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, T, uint64_t(a->num_heads) * HD,
                              uint64_t(a->num_heads) * HD * 2, 128, 64, true))
    return rc;
  if (int rc = encode_tmap_2d(&tk, a->k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, T, uint64_t(a->num_kv_heads) * HD,
                              uint64_t(a->num_kv_heads) * HD * 2, BN, 64, true))
    return rc;
  if (int rc = encode_tmap_2d(&tv, a->v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, T, uint64_t(a->num_kv_heads) * HD,
                              uint64_t(a->num_kv_heads) * HD * 2, BN, 64, true))
    return rc;
  FwdParams p;
  p.o = static_cast<__nv_bfloat16*>(a->o);
  p.lse = a->lse;
  p.cu = a->cu_seqlens;
  p.prefix = a->prefix_len;
  mark_boundary(st);
  if (int rc = launch_build_tiles(a->cu_seqlens, a->seg_src, a->num_seqs, int64_t(T), tiles_buf, st,
                                  const_cast<int4**>(&p.tiles), const_cast<int**>(&p.ntiles)))
    return rc;
  mark_boundary(st);
  p.nseq = a->num_seqs;
  p.T = static_cast<int>(T);
  p.H = a->num_heads;
  p.Hkv = a->num_kv_heads;
  p.mask = a->mask_mode;
  p.scale_log2 = a->softmax_scale * 1.4426950408889634f;
  auto kern = attn_fwd_kernel<HD, BN, STAGES>;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int64_t max_tiles = int64_t(T) / 128 + a->num_seqs;
  kern<<<max_tiles * a->num_heads, 192, Cfg::SMEM, st>>>(tq, tk, tv, p);
  VLASIM_LAUNCH_CHECK();
  mark_boundary(st);
  return VLASIM_OK;
}

// ---------------------------------------------------------------------------------------------
// Persistent variant (head_dim 256, config 3): grid = min(#SMs, items, sm_budget); each CTA walks
// the cost-sorted items (segment-aligned Q tile, head) on the boustrophedon schedule with the same
// three roles.  Every pipeline runs on CONTINUOUS counters across items, so an item boundary costs
// no prologue: the next item's Q tile loads as soon as the current item's last S MMA has read the
// Q buffer (bar_q_empty), its K/V tiles stream through the same ring, its first S MMA issues while
// the softmax warps drain the current O, and only its first P·V waits for that drain (bar_o_free):
// O (256 columns) is single-buffered — S[2] (2·BN) + O (HD) + P[2] (BN) = 448 of 512 columns.
// Visible-key spans per token come from k_spans_p (the forward workspace's span table).
__global__ void k_spans_p(const int32_t* __restrict__ cu, const int32_t* __restrict__ prefix, int nseq, int mask,
                          int T, int2* __restrict__ rows_span) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const RowSpan r = row_span(cu, prefix, nseq, mask, t, T);
  rows_span[t] = make_int2(r.lo, r.hi);
}

// Persistent layout: Q | K ring (KS) | V ring (VS).  K and V have separate rings: a K stage is
// released as soon as its S MMA has read it and a V stage after its P·V, so the K/V streaming from
// L2 — the limiter of this kernel (128 flop per K/V byte at d = 256, BN = 64) — is not held up by
// the softmax of the tile.  The producer issues V one tile behind K.
template <int HD, int BN, int KS, int VS>
struct FwdPCfg {
  static constexpr int BM = 128;
  static constexpr int Q_BYTES = BM * HD * 2;
  static constexpr int KV_BYTES = BN * HD * 2;
  static constexpr int OFF_K = Q_BYTES, OFF_V = OFF_K + KS * KV_BYTES;
  static constexpr int SMEM = OFF_V + VS * KV_BYTES + 1024;
  // TMEM: S[2] [0, 2·BN) with P (bf16) written over its S buffer, O [2·BN, 2·BN + HD), and the item's
  // Q tile [Q_COL, +HD/2): copied from smem by tcgen05.cp at the item start, so S = Q·Kᵀ takes A
  // from TMEM — the 64 KB Q tile is not re-read from smem for every key tile, and its smem buffer is
  // released as soon as it is copied (the next item's Q loads during this item)
  static constexpr uint32_t S_COL = 0, O_COL = 2 * BN, Q_COL = 2 * BN + HD;
  static_assert(Q_COL + HD / 2 <= 512, "TMEM budget");
  static_assert(SMEM <= 232448 - 1024, "smem budget");
};

struct FwdPParams {
  __nv_bfloat16* o;
  float* lse;
  const int2* rows_span;
  const int4* tiles;
  const int* ntiles;
  int T, H, Hkv;
  float scale_log2;
};

struct FwdPItem {
  int q0, qe, dl, h, kh, kv_lo, kv_hi, nkv;
};
// Every role walks the items with a look-ahead: the tile record (tiles[i / H]) two items ahead, the
// span loads that index by it one item ahead, and the derived count when the item becomes current —
// no load result is consumed at the boundary where it is issued (no dependent-load stall per item).
struct FwdPCursor {
  int m = 0, i = 0, n = 0;
  FwdPItem nx;
  int4 tn;
  __device__ __forceinline__ int4 tile(const FwdPParams& p, int mm) const {
    const int ii = sched_item(mm);
    return ii < n ? __ldg(&p.tiles[ii / p.H]) : make_int4(0, 1, 0, 0);
  }
  __device__ __forceinline__ FwdPItem raw(const FwdPParams& p, int ii, int4 t) const {
    FwdPItem it;
    it.h = ii % p.H;
    it.q0 = t.x;
    it.qe = t.y;
    it.dl = t.z;
    it.kh = it.h / (p.H / p.Hkv);
    it.kv_lo = __ldg(&p.rows_span[t.x].x);  // spans are monotone inside a segment
    it.kv_hi = __ldg(&p.rows_span[t.y - 1].y);
    it.nkv = -1;
    return it;
  }
  __device__ __forceinline__ void start(const FwdPParams& p, int nitems) {
    n = nitems;
    m = 0;
    i = sched_item(0);
    if (i < n) nx = raw(p, i, tile(p, 0));
    tn = tile(p, 1);
  }
  // the current item (m), then the look-ahead advances; false past the last item
  template <int BN>
  __device__ __forceinline__ bool take(const FwdPParams& p, FwdPItem& it) {
    if (i >= n) return false;
    it = nx;
    it.nkv = max(0, (it.kv_hi - it.kv_lo + BN - 1) / BN);
    i = sched_item(++m);
    if (i < n) {
      nx = raw(p, i, tn);
      tn = tile(p, m + 1);
    }
    return true;
  }
};

template <int HD, int BN, int KS, int VS>
__global__ void __launch_bounds__(192, 1)
    attn_fwd_p_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const FwdPParams p) {
  using Cfg = FwdPCfg<HD, BN, KS, VS>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;

  __shared__ uint64_t bar_q_full, bar_q_empty, bar_k_full[KS], bar_k_empty[KS], bar_v_full[VS], bar_v_empty[VS],
      bar_s_full[2], bar_p_full[2], bar_o_ready, bar_o_done, bar_o_free;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nitems = __ldg(p.ntiles) * p.H;
  if (tid == 0) {
    mbar_init(&bar_q_full, 1);
    mbar_init(&bar_q_empty, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(&bar_k_full[s], 1);
      mbar_init(&bar_k_empty[s], 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(&bar_v_full[s], 1);
      mbar_init(&bar_v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_s_full[b], 1);
      mbar_init(&bar_p_full[b], 4);
    }
    mbar_init(&bar_o_ready, 1);
    mbar_init(&bar_o_done, 1);
    mbar_init(&bar_o_free, 4);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    // ------------------------------------------------ TMA producer (V one tile behind K)
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      int gk = 0, gv = 0, k = 0;
      int pv_row = -1, pv_kh = 0;  // the V tile still to load (data row, kv head)
      auto load_v = [&]() {
        const int st = gv % VS;
        if (gv >= VS) mbar_wait(&bar_v_empty[st], ((gv / VS) - 1) & 1);
        mbar_expect_tx(&bar_v_full[st], Cfg::KV_BYTES);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          tma_load_2d(sV + st * Cfg::KV_BYTES + c * BN * 128, &tmV, pv_kh * HD + c * 64, pv_row, &bar_v_full[st]);
        ++gv;
        pv_row = -1;
      };
      FwdPCursor cur;
      cur.start(p, nitems);
      for (FwdPItem it; cur.take<BN>(p, it);) {
        if (k > 0) mbar_wait(&bar_q_empty, (k - 1) & 1);  // the previous item's last S has read Q
        mbar_expect_tx(&bar_q_full, Cfg::Q_BYTES);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          tma_load_2d(sQ + c * Cfg::BM * 128, &tmQ, it.h * HD + c * 64, it.q0 + it.dl, &bar_q_full);
        for (int j = 0; j < it.nkv; ++j, ++gk) {
          const int st = gk % KS;
          if (gk >= KS) mbar_wait(&bar_k_empty[st], ((gk / KS) - 1) & 1);
          const int kv0 = it.kv_lo + j * BN + it.dl;  // data row
          mbar_expect_tx(&bar_k_full[st], Cfg::KV_BYTES);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_2d(sK + st * Cfg::KV_BYTES + c * BN * 128, &tmK, it.kh * HD + c * 64, kv0, &bar_k_full[st]);
          if (pv_row >= 0) load_v();
          pv_row = kv0;
          pv_kh = it.kh;
        }
        ++k;
      }
      if (pv_row >= 0) load_v();
    }
  } else if (warp == 5) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, BN, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, HD, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      int g = 0, k = 0;
      FwdPCursor cur;
      cur.start(p, nitems);
      for (FwdPItem itc; cur.take<BN>(p, itc);) {
        const int nkv = itc.nkv;
        mbar_wait(&bar_q_full, k & 1);
        tc_fence_after();
        // Q → TMEM (one tcgen05.cp per 16-element K-step; in issue order after the previous item's
        // last S MMA), then Q's smem buffer is free
#pragma unroll
        for (int s = 0; s < HD / 16; ++s)
          tmem_cp_128x256b(tmem + Cfg::Q_COL + 8 * s,
                           make_sdesc_sw128(q_addr + (s / 4) * Cfg::BM * 128 + (s % 4) * 32, 16, 1024));
        umma_commit(&bar_q_empty);
        if (nkv == 0) umma_commit(&bar_o_done);  // (no visible key: cannot happen) keep the phases aligned
        for (int j = 0; j <= nkv; ++j) {
          if (j < nkv) {
            const int gj = g + j, st = gj % KS;
            mbar_wait(&bar_k_full[st], (gj / KS) & 1);
            tc_fence_after();
            const uint32_t k_addr = smem_u32(sK + st * Cfg::KV_BYTES);
            const uint32_t d_s = tmem + Cfg::S_COL + (gj & 1) * BN;
#pragma unroll
            for (int s = 0; s < HD / 16; ++s) {
              const uint64_t b = make_sdesc_sw128(k_addr + (s / 4) * BN * 128 + (s % 4) * 32, 16, 1024);
              umma_f16_ts(d_s, tmem + Cfg::Q_COL + 8 * s, b, idesc_s, s > 0 ? 1u : 0u);
            }
            umma_commit(&bar_s_full[gj & 1]);
            umma_commit(&bar_k_empty[st]);
          }
          if (j > 0) {
            const int gj = g + j - 1, st = gj % VS;
            mbar_wait(&bar_p_full[gj & 1], (gj >> 1) & 1);
            if (j == 1 && k > 0) mbar_wait(&bar_o_free, (k - 1) & 1);  // previous item's O drained
            mbar_wait(&bar_v_full[st], (gj / VS) & 1);
            tc_fence_after();
            const uint32_t v_addr = smem_u32(sV + st * Cfg::KV_BYTES);
            const uint32_t a_tm = tmem + Cfg::S_COL + (gj & 1) * BN;  // P over its S buffer
#pragma unroll
            for (int s = 0; s < BN / 16; ++s) {
              const uint64_t b = make_sdesc_sw128(v_addr + s * 2048, BN * 128, 1024);
              umma_f16_ts(tmem + Cfg::O_COL, a_tm + s * 8, b, idesc_o, (j > 1 || s > 0) ? 1u : 0u);
            }
            umma_commit(&bar_v_empty[st]);
            umma_commit(&bar_o_ready);
            if (j == nkv) umma_commit(&bar_o_done);
          }
        }
        g += nkv;
        ++k;
      }
    }
  } else {
    // ------------------------------------------------ softmax + epilogue (warps 0-3, thread = row)
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float sl2 = p.scale_log2;
    int g = 0, k = 0;
    FwdPCursor cur;
    cur.start(p, nitems);
    auto row_span_of = [&](const FwdPItem& f) {  // rows past the tile: none
      return f.q0 + tid < f.qe ? __ldg(&p.rows_span[f.q0 + tid]) : make_int2(0, 0);
    };
    int2 rs_n = cur.i < cur.n ? row_span_of(cur.nx) : make_int2(0, 0);
    for (FwdPItem it; cur.take<BN>(p, it);) {
      const int row = it.q0 + tid;
      const int2 rs = rs_n;  // loaded one item ahead
      if (cur.i < cur.n) rs_n = row_span_of(cur.nx);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < it.nkv; ++j) {
        const int gj = g + j, sb = gj & 1;
        mbar_wait(&bar_s_full[sb], (gj >> 1) & 1);
        tc_fence_after();
        uint32_t r[BN];
#pragma unroll
        for (int c = 0; c < BN; c += 32)
          tmem_ld32(tmem + lane_off + Cfg::S_COL + sb * BN + c, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
        tmem_wait_ld();
        const int kv0 = it.kv_lo + j * BN;
        const int c_lo = rs.x - kv0, c_hi = rs.y - kv0;
        if (!__all_sync(0xffffffffu, c_lo <= 0 && c_hi >= BN)) {
#pragma unroll
          for (int c = 0; c < BN; ++c) r[c] = (c >= c_lo && c < c_hi) ? r[c] : __float_as_uint(-INFINITY);
        }
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < BN; c += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            mq[u] = fmax3(mq[u], __uint_as_float(r[c + 2 * u]), __uint_as_float(r[c + 2 * u + 1]));
        }
        float mt = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        mt = (mt == -INFINITY) ? -INFINITY : mt * sl2;
        const bool grow = mt > m_run + kLazyRescale;
        const float alpha = grow ? ex2_approx(m_run - mt) : 1.f;
        if (__any_sync(0xffffffffu, grow && j > 0 && m_run != -INFINITY)) {
          mbar_wait(&bar_o_ready, (gj - 1) & 1);  // P·V of the previous tile has landed in O
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < HD; c += 32) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_off + Cfg::O_COL + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 32; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * alpha);
            tmem_st32(tmem + lane_off + Cfg::O_COL + c, o);
          }
        }
        if (grow) {
          l_run *= alpha;
          m_run = mt;
        }
        const float msub = (m_run == -INFINITY) ? 0.f : m_run;
        const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-msub, -msub);
        float2 lq[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < BN; c += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float2 a2 = f2_fma(make_float2(__uint_as_float(r[c + 2 * q]), __uint_as_float(r[c + 2 * q + 1])),
                                     sl2v, nmv);
            const float2 pe = make_float2(ex2_approx(a2.x), ex2_approx(a2.y));
            lq[q & 1] = f2_add(lq[q & 1], pe);
            pk[q] = pack_bf16x2(pe.x, pe.y);
          }
          tmem_st16(tmem + lane_off + Cfg::S_COL + sb * BN + c / 2, pk);  // P over the S it was read from
        }
        l_run += (lq[0].x + lq[1].x) + (lq[0].y + lq[1].y);
        tmem_wait_st();
        tc_fence_before();
        warp_arrive(&bar_p_full[sb]);
      }
      // epilogue: O / l → bf16 (direct row stores), LSE; then hand O back to the MMA warp
      mbar_wait(&bar_o_done, k & 1);
      tc_fence_after();
      const bool valid = row < it.qe && rs.x < rs.y;
      const float inv_l = (valid && l_run > 0.f) ? 1.f / l_run : 0.f;
      __nv_bfloat16* orow = p.o + (static_cast<int64_t>(row + it.dl) * p.H + it.h) * HD;
#pragma unroll
      for (int c = 0; c < HD; c += 32) {
        uint32_t o[32];
        tmem_ld32(tmem + lane_off + Cfg::O_COL + c, o);
        tmem_wait_ld();
        if (valid) {
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            pk[q] = pack_bf16x2(__uint_as_float(o[2 * q]) * inv_l, __uint_as_float(o[2 * q + 1]) * inv_l);
          uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      tc_fence_before();
      warp_arrive(&bar_o_free);
      if (valid)
        p.lse[static_cast<int64_t>(it.h) * p.T + row + it.dl] = (m_run + __log2f(l_run)) * 0.69314718055994530942f;
      g += it.nkv;
      ++k;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc<512>(tmem);
}

template <int HD, int BN, int KS, int VS>
int launch_fwd_p(const vlasim_attn_args* a, void* ws, cudaStream_t st) {
  using namespace vlasim_host;
  using Cfg = FwdPCfg<HD, BN, KS, VS>;
  CUtensorMap tq, tk, tv;
  const uint64_t T = a->total_tokens;
  if (int rc = encode_tmap_2d(&tq, a->q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, T, uint64_t(a->num_heads) * HD,
                              uint64_t(a->num_heads) * HD * 2, 128, 64, true))
    return rc;
  if (int rc = encode_tmap_2d(&tk, a->k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, T, uint64_t(a->num_kv_heads) * HD,
                              uint64_t(a->num_kv_heads) * HD * 2, BN, 64, true))
    return rc;
  if (int rc = encode_tmap_2d(&tv, a->v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, T, uint64_t(a->num_kv_heads) * HD,
                              uint64_t(a->num_kv_heads) * HD * 2, BN, 64, true))
    return rc;
  FwdPParams p;
  p.o = static_cast<__nv_bfloat16*>(a->o);
  p.lse = a->lse;
  int2* spans = static_cast<int2*>(ws);
  p.rows_span = spans;
  mark_boundary(st);
  k_spans_p<<<int((T + 255) / 256), 256, 0, st>>>(a->cu_seqlens, a->prefix_len, a->num_seqs, a->mask_mode, int(T),
                                                  spans);
  if (int rc = launch_build_tiles(a->cu_seqlens, a->seg_src, a->num_seqs, int64_t(T), fwd_ws_tiles(a, ws), st,
                                  const_cast<int4**>(&p.tiles), const_cast<int**>(&p.ntiles)))
    return rc;
  mark_boundary(st);
  p.T = static_cast<int>(T);
  p.H = a->num_heads;
  p.Hkv = a->num_kv_heads;
  p.scale_log2 = a->softmax_scale * 1.4426950408889634f;
  auto kern = attn_fwd_p_kernel<HD, BN, KS, VS>;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int64_t max_tiles = int64_t(T) / 128 + a->num_seqs;
  kern<<<persistent_grid(max_tiles * a->num_heads, a->sm_budget), 192, Cfg::SMEM, st>>>(tq, tk, tv, p);
  VLASIM_LAUNCH_CHECK();
  mark_boundary(st);
  return VLASIM_OK;
}

}  // namespace

namespace vlasim_host {
int validate_attn_args(const vlasim_attn_args* a, bool fp8) {
  if (!a) return set_error(VLASIM_ECONFIG, "attention: null args");
  if (!a->q || !a->k || !a->v || !a->o || !a->lse || !a->cu_seqlens)
    return set_error(VLASIM_ECONFIG, "attention: q, k, v, o, lse, cu_seqlens are required");
  if (a->total_tokens < 1 || a->total_tokens >= INT_MAX)
    return set_error(VLASIM_ECONFIG, "attention: total_tokens=%lld out of range", (long long)a->total_tokens);
  if (a->num_seqs < 1) return set_error(VLASIM_ECONFIG, "attention: num_seqs must be >= 1");
  if (a->num_heads < 1 || a->num_kv_heads < 1 || a->num_heads % a->num_kv_heads)
    return set_error(VLASIM_ECONFIG, "attention: num_kv_heads (%d) must divide num_heads (%d)", a->num_kv_heads,
                     a->num_heads);
  if (a->head_dim != 64 && a->head_dim != 128 && a->head_dim != 256)
    return set_error(VLASIM_ECONFIG, "attention: head_dim %d unsupported (64, 128, 256)", a->head_dim);
  if (a->mask_mode < 0 || a->mask_mode > 2) return set_error(VLASIM_ECONFIG, "attention: bad mask_mode");
  if (a->mask_mode == VLASIM_MASK_PREFIX && !a->prefix_len)
    return set_error(VLASIM_ECONFIG, "attention: prefix mask needs prefix_len");
  if (fp8 && (!a->q_scale || !a->k_scale)) return set_error(VLASIM_ECONFIG, "attention: fp8 path needs scales");
  const uintptr_t al = reinterpret_cast<uintptr_t>(a->q) | reinterpret_cast<uintptr_t>(a->k) |
                       reinterpret_cast<uintptr_t>(a->v) | reinterpret_cast<uintptr_t>(a->o);
  if (al & 15) return set_error(VLASIM_ECONFIG, "attention: q/k/v/o must be 16-byte aligned");
  return VLASIM_OK;
}
}  // namespace vlasim_host

namespace vlasim_host {
int launch_fwd_persistent(const vlasim_attn_args* a, void* ws, size_t ws_bytes, cudaStream_t st);
void* fwd_ws_tiles(const vlasim_attn_args* a, void* ws);
}

// head_dim 64/128: persistent kernel (attn_fwd2.cu, needs the span workspace);
// head_dim 256: the persistent single-O kernel above (attn_fwd_p_kernel; VLASIM_FWD_V1 selects the
// one-tile-per-CTA kernel for comparison).
extern "C" int vlasim_varlen_attn_fwd_cuda(const vlasim_attn_args* a, void* ws, size_t ws_bytes,
                                           vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = validate_attn_args(a, false)) return rc;
  cudaStream_t st = as_stream(stream);
  const size_t need = fwd_ws_bytes(a);
  if (!ws || ws_bytes < need) return set_error(VLASIM_ECONFIG, "attention fwd: workspace %zu < %zu", ws_bytes, need);
  if (a->head_dim == 256)
    return getenv("VLASIM_FWD_V1") ? launch_fwd<256, 64, 2>(a, fwd_ws_tiles(a, ws), st)
                                   : launch_fwd_p<256, 64, 3, 2>(a, ws, st);
  if (getenv("VLASIM_FWD_V1"))
    return a->head_dim == 64 ? launch_fwd<64, 128, 4>(a, fwd_ws_tiles(a, ws), st)
                             : launch_fwd<128, 128, 3>(a, fwd_ws_tiles(a, ws), st);
  return launch_fwd_persistent(a, ws, ws_bytes, st);
}
