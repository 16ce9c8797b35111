// pack.cu — GPU packer: length histogram → stable class ranks → class-wise first-fit-
// decreasing → packed-stream layout (cu_seqlens, member order, token ids) → token-row
// gather/scatter.  Bit-exact with the reference's sequential FFD under
// the pinned order (length desc, id asc) — see DESIGN.md §2 for the equivalence proof:
//
//   All items of one length L are placed in id order; each lands in the lowest-index bin
//   with rem >= L, and after it lands every lower-index bin has rem < L.  Hence class L
//   fills open bins in index order, bin b taking min(floor(rem_b / L), remaining) items,
//   and the leftover opens new bins of floor(cap / L) items each.  FFD = a sequence of
//   per-class exclusive scans over the open bins, driven by the length histogram.
//
// Kernels (one launch each, all stream-ordered, no host sync unless SYNC_CHECK):
//   k_init        status / per-bin counters
//   k_hist        validate 1 <= len <= cap, per-chunk histogram in smem
//   k_class_scan  per-class exclusive base across chunks (stable rank offsets) + counts
//   k_ffd         single CTA: class-wise FFD over the open-bin list (smem), emits "runs"
//   k_assign      stable rank inside class → run → (bin, slot, token offset)
//   k_scan_*      exclusive scans: bin member/token offsets, source offsets
//   k_layout      member order, global + per-bin cu_seqlens
#include <algorithm>
#include <climits>

#include "common.hpp"
#include "scan.cuh"

using namespace vlasim_dev;

namespace {

constexpr int kChunk = 4096;         // items per histogram / rank chunk
constexpr int kRankThreads = 1024;   // k_assign block (4 rounds of 1024 items)
constexpr int kScanItems = 4096;     // items per scan block (1024 threads × 4)
constexpr int kMaxActiveBins = 16384;  // open bins kept in k_ffd shared memory (then spilled to HBM)
constexpr int kSmemHistMaxCap = 40959;  // (cap + 1) int32 counters in smem; larger caps count in HBM
constexpr int kGreedyDeepMaxBins = 1 << 20;  // 4-level 32-ary room tree, level 0 in HBM

struct PackWs {
  int32_t* chunk_hist;       // [C][cap+1]   → exclusive per-class base after k_class_scan
  int32_t* class_count;      // [cap+1]
  int32_t* class_run_start;  // [cap+1]
  int32_t* class_nruns;      // [cap+1]
  int32_t* run_bin;          // [n]
  int32_t* run_cum;          // [n]  items of the class placed before this run
  int32_t* run_tok;          // [n]  bin fill (tokens) before this run
  int32_t* run_mem;          // [n]  bin member count before this run
  int64_t* scan_part;        // [3][num_scan_blocks + 1]
  int32_t* mode;             // [1]     1: k_ffd_warp placed the batch (k_ffd returns at once)
  int32_t* spill;            // [3][n]  k_ffd open-bin list once it outgrows shared memory;
                             //         k_greedy level-0 room / count ([2][min(n, 2^20)])
};

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

inline int64_t num_chunks(int64_t n) { return (n + kChunk - 1) / kChunk; }
inline int64_t num_scan_blocks(int64_t n) { return (n + 1 + kScanItems - 1) / kScanItems; }

size_t carve(PackWs* w, void* base, int64_t n, int cap) {
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* r = p ? p + off : nullptr;
    off += align_up(bytes);
    return r;
  };
  const size_t nc = size_t(cap) + 1;
  w->chunk_hist = reinterpret_cast<int32_t*>(take(size_t(num_chunks(n)) * nc * 4));
  w->class_count = reinterpret_cast<int32_t*>(take(nc * 4));
  w->class_run_start = reinterpret_cast<int32_t*>(take(nc * 4));
  w->class_nruns = reinterpret_cast<int32_t*>(take(nc * 4));
  w->run_bin = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
  w->run_cum = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
  w->run_tok = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
  w->run_mem = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
  w->scan_part = reinterpret_cast<int64_t*>(take(size_t(3) * (num_scan_blocks(n) + 1) * 8));
  w->mode = reinterpret_cast<int32_t*>(take(4));
  w->spill = reinterpret_cast<int32_t*>(take(size_t(3) * ((n + 31) & ~int64_t(31)) * 4));
  return off;
}

// ------------------------------------------------------------------ init / validate
__global__ void k_init(vlasim_pack_out out, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i == 0) {
    out.status[0] = 0;
    out.status[1] = INT_MAX;
    *out.num_bins = 0;
  }
  if (i < n) {
    out.bin_count[i] = 0;
    out.bin_fill[i] = 0;
  }
}

// kGlobal (cap > kSmemHistMaxCap): the chunk's counters live in its chunk_hist row (zeroed by
// the host-side memset) and are incremented with HBM atomics.
template <bool kGlobal>
__global__ void k_hist(const int32_t* __restrict__ len, int64_t n, int cap, int32_t* __restrict__ chunk_hist,
                       int32_t* status) {
  extern __shared__ int32_t sh_[];
  int32_t* sh = kGlobal ? chunk_hist + size_t(blockIdx.x) * (cap + 1) : sh_;
  if (!kGlobal) {
    for (int i = threadIdx.x; i <= cap; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  const int64_t base = int64_t(blockIdx.x) * kChunk;
  for (int j = threadIdx.x; j < kChunk; j += blockDim.x) {
    const int64_t i = base + j;
    if (i >= n) break;
    const int L = len[i];
    if (L < 1 || L > cap) {
      atomicMin(&status[1], int(i));
      status[0] = VLASIM_ECONFIG;
      continue;
    }
    atomicAdd(&sh[L], 1);
  }
  if (kGlobal) return;
  __syncthreads();
  int32_t* o = chunk_hist + size_t(blockIdx.x) * (cap + 1);
  for (int i = threadIdx.x; i <= cap; i += blockDim.x) o[i] = sh[i];
}

// One thread per length class: exclusive base over chunks (in chunk order = id order).
__global__ void k_class_scan(int32_t* __restrict__ chunk_hist, int64_t nchunks, int cap,
                             int32_t* __restrict__ class_count) {
  const int L = blockIdx.x * blockDim.x + threadIdx.x;
  if (L > cap) return;
  int32_t run = 0;
  int64_t c = 0;
  for (; c + 8 <= nchunks; c += 8) {  // 8 independent loads in flight, then the running sums
    int32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = chunk_hist[size_t(c + u) * (cap + 1) + L];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      chunk_hist[size_t(c + u) * (cap + 1) + L] = run;
      run += v[u];
    }
  }
  for (; c < nchunks; ++c) {
    int32_t* p = chunk_hist + size_t(c) * (cap + 1) + L;
    const int32_t v = *p;
    *p = run;
    run += v;
  }
  class_count[L] = run;
}

// ------------------------------------------------------------------ class-wise FFD
// Single CTA.  Open ("active") bins are kept in shared memory sorted by bin id:
// act_id / act_rem / act_cnt.  A bin whose remaining room is below the smallest length
// still to come can never receive an item again; it is retired (final count/fill written)
// during compaction, which preserves the id order of the survivors.  When more than
// kMaxActiveBins bins stay open even after retirement, the list moves to the workspace
// (`spill`, n entries per array — FFD never opens more bins than items) and the kernel carries
// on there: any input the reference packs, the GPU packs (no open-bin limit).
__global__ void __launch_bounds__(1024, 1) k_ffd(int n, int cap, PackWs ws, vlasim_pack_out out) {
  extern __shared__ int32_t sm[];
  int32_t* act_id = sm;
  int32_t* act_rem = sm + kMaxActiveBins;
  int32_t* act_cnt = sm + 2 * kMaxActiveBins;
  int32_t* cls = sm + 3 * kMaxActiveBins;  // [1024] compacted class list of the current L-chunk
  int act_cap = kMaxActiveBins;            // uniform: capacity of the current open-bin arrays
  __shared__ int32_t scratch[33];
  __shared__ int32_t s_ncls, s_lmin;
  const int tid = threadIdx.x, nt = blockDim.x;

  if (out.status[0] != 0) return;  // validation failed upstream
  if (*ws.mode == 1) return;       // k_ffd_warp placed this batch (at most kWarpMaxBins bins)

  // smallest present length (retirement threshold)
  int lmin_local = INT_MAX;
  for (int L = 1 + tid; L <= cap; L += nt)
    if (ws.class_count[L] > 0) lmin_local = min(lmin_local, L);
  for (int o = 16; o > 0; o >>= 1) lmin_local = min(lmin_local, __shfl_xor_sync(0xffffffffu, lmin_local, o));
  if (tid == 0) s_lmin = INT_MAX;
  __syncthreads();
  if ((tid & 31) == 0) atomicMin(&s_lmin, lmin_local);
  __syncthreads();
  const int lmin = s_lmin;

  int nact = 0, nb = 0, nruns = 0;  // uniform across the block
  int32_t tot;

  for (int hi = cap; hi >= 1; hi -= 1024) {
    // ---- compact the non-empty classes of L ∈ (hi-1024, hi] in descending order
    const int span = min(1024, hi);
    const int per_c = (span + nt - 1) / nt;
    int mine = 0;
    for (int j = tid * per_c; j < min(span, (tid + 1) * per_c); ++j) mine += ws.class_count[hi - j] > 0;
    int pos = block_exclusive_scan<int32_t>(mine, scratch, &tot);
    for (int j = tid * per_c; j < min(span, (tid + 1) * per_c); ++j)
      if (ws.class_count[hi - j] > 0) cls[pos++] = hi - j;
    if (tid == 0) s_ncls = tot;
    __syncthreads();
    const int ncls = s_ncls;

    for (int ci = 0; ci < ncls; ++ci) {
      const int L = cls[ci];
      const int c = ws.class_count[L];
      const int runs_before = nruns;

      // ---- phase A: existing open bins, in id order
      const int per = (nact + nt - 1) / nt;
      const int b0 = min(nact, tid * per), b1 = min(nact, b0 + per);
      int sumq = 0;
      for (int b = b0; b < b1; ++b) sumq += act_rem[b] / L;
      int32_t totq;
      const int exq = block_exclusive_scan<int32_t>(sumq, scratch, &totq);
      int running = exq, nr = 0;
      for (int b = b0; b < b1 && running < c; ++b) {
        const int q = act_rem[b] / L;
        if (q > 0) ++nr;
        running += q;
      }
      int32_t nr_tot;
      int ridx = nruns + block_exclusive_scan<int32_t>(nr, scratch, &nr_tot);
      running = exq;
      for (int b = b0; b < b1 && running < c; ++b) {
        const int rem = act_rem[b];
        const int q = rem / L;
        if (q > 0) {
          const int take = min(q, c - running);
          ws.run_bin[ridx] = act_id[b];
          ws.run_cum[ridx] = running;
          ws.run_tok[ridx] = cap - rem;
          ws.run_mem[ridx] = act_cnt[b];
          ++ridx;
          act_rem[b] = rem - take * L;
          act_cnt[b] += take;
        }
        running += q;
      }
      nruns += nr_tot;
      const int placed = min(c, totq);
      const int r = c - placed;

      // ---- phase B: new bins of floor(cap / L) items each
      if (r > 0) {
        const int k = cap / L;
        const int nnew = (r + k - 1) / k;
        if (nact + nnew > act_cap) {
          // (smem mode only: in the spilled arrays nact + nnew <= bins opened <= n = act_cap)
          // retire bins that can never be used again, then re-check; per <= 16 here
          __syncthreads();
          int keep = 0;
          for (int b = b0; b < b1; ++b) keep += act_rem[b] >= lmin;
          int32_t kept;
          int kpos = block_exclusive_scan<int32_t>(keep, scratch, &kept);
          int32_t tid_buf[32], rem_buf[32], cnt_buf[32];  // per <= kMaxActiveBins / 1024 = 16
          int nk = 0;
          for (int b = b0; b < b1; ++b) {
            if (act_rem[b] >= lmin) {
              tid_buf[nk] = act_id[b];
              rem_buf[nk] = act_rem[b];
              cnt_buf[nk] = act_cnt[b];
              ++nk;
            } else {
              out.bin_count[act_id[b]] = act_cnt[b];
              out.bin_fill[act_id[b]] = cap - act_rem[b];
            }
          }
          __syncthreads();
          for (int j = 0; j < nk; ++j) {
            act_id[kpos + j] = tid_buf[j];
            act_rem[kpos + j] = rem_buf[j];
            act_cnt[kpos + j] = cnt_buf[j];
          }
          nact = kept;
          __syncthreads();
          if (nact + nnew > act_cap) {  // spill the open-bin list to the workspace, id order kept
            const int64_t stride = (int64_t(n) + 31) & ~int64_t(31);
            int32_t* g_id = ws.spill;
            int32_t* g_rem = ws.spill + stride;
            int32_t* g_cnt = ws.spill + 2 * stride;
            for (int b = tid; b < nact; b += nt) {
              g_id[b] = act_id[b];
              g_rem[b] = act_rem[b];
              g_cnt[b] = act_cnt[b];
            }
            __syncthreads();
            act_id = g_id;
            act_rem = g_rem;
            act_cnt = g_cnt;
            act_cap = n;
          }
        }
        for (int j = tid; j < nnew; j += nt) {
          const int take = min(k, r - j * k);
          ws.run_bin[nruns + j] = nb + j;
          ws.run_cum[nruns + j] = placed + j * k;
          ws.run_tok[nruns + j] = 0;
          ws.run_mem[nruns + j] = 0;
          act_id[nact + j] = nb + j;
          act_rem[nact + j] = cap - take * L;
          act_cnt[nact + j] = take;
        }
        nb += nnew;
        nact += nnew;
        nruns += nnew;
      }
      if (tid == 0) {
        ws.class_run_start[L] = runs_before;
        ws.class_nruns[L] = nruns - runs_before;
      }
      __syncthreads();
    }
  }
  // final state of the still-open bins
  for (int b = tid; b < nact; b += nt) {
    out.bin_count[act_id[b]] = act_cnt[b];
    out.bin_fill[act_id[b]] = cap - act_rem[b];
  }
  if (tid == 0) *out.num_bins = nb;
}

// Warp-synchronous variant of k_ffd for batches whose bins fit in shared memory: one warp,
// class counts staged in smem, bins visited 32 at a time with early exit once the class is
// placed (no block barriers on the per-class critical path).
constexpr int kWarpMaxBins = 16384;
constexpr int kWarpCntMaxCap = 24575;  // 2 × 64 KB of bins + (cap + 1) counters + 2 KB within 227 KB
// floor(a / b) for 0 <= a, 1 <= b <= 2^15 via the fp32 reciprocal, corrected to the exact quotient
// (the estimate is off by at most one either way at these magnitudes).
__device__ __forceinline__ int udiv_small(int a, int b, float inv_b) {
  int q = __float2int_rz(__int2float_rn(a) * inv_b);
  q -= q * b > a;
  q += (q + 1) * b <= a;
  return q;
}
__global__ void __launch_bounds__(32, 1) k_ffd_warp(int64_t n, int cap, PackWs ws, vlasim_pack_out out) {
  extern __shared__ int32_t sm[];
  int32_t* act_rem = sm;                    // bins are never retired here: id == index
  int32_t* act_cnt = sm + kWarpMaxBins;
  // [cap + 1] class counts: staged in smem up to kWarpCntMaxCap, read from the workspace beyond
  const bool cnt_smem = cap <= kWarpCntMaxCap;
  int32_t* cnt = cnt_smem ? sm + 2 * kWarpMaxBins : ws.class_count;
  const int lane = threadIdx.x;
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  if (out.status[0] != 0) return;
  // class counts → smem: a single warp, so keep 32 loads in flight per lane (latency-bound otherwise)
  long long tok = 0;  // Σ lengths, for the bin-count bound below
#pragma unroll 32
  for (int L = lane; L <= cap; L += 32) {
    const int c = __ldg(ws.class_count + L);
    if (cnt_smem) cnt[L] = c;
    tok += static_cast<long long>(c) * L;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tok += __shfl_xor_sync(full, tok, o);
  __syncwarp();
  // Any first-fit packing keeps every bin but one more than half full, so it opens fewer than
  // 2·Σl/cap + 1 bins (and never more than n): when that bound fits the smem bin arrays this warp
  // places the batch (config 5: 1M samples, ≈ 6.4k bins); otherwise the 1024-thread k_ffd does.
  const long long bound = min(static_cast<long long>(n), 2 * tok / cap + 1);
  if (bound > kWarpMaxBins) {
    if (lane == 0) *ws.mode = 0;
    return;
  }
  if (lane == 0) *ws.mode = 1;
  // Register-resident fast path: FFD never opens more than 2·Σl/cap + 1 bins (every pair of
  // consecutive bins holds more than cap tokens), so when that bound is ≤ 64 the open bins live
  // in registers, two per lane (bins lane and 32 + lane).  Each run of a class is one first-fit
  // step: two ballots for the lowest bin with room, the bin's room and member count broadcast
  // from its owner lane, min(⌊room/L⌋, left) items taken at once (the class-wise argument).
  if (2 * tok <= 63LL * cap) {
    // (1) the present classes, largest first, compacted into smem (the bin arrays are unused on
    //     this path; n ≤ kWarpMaxBins bounds the class count)
    int2* cls = reinterpret_cast<int2*>(act_rem);
    int ncls = 0;
#pragma unroll 4
    for (int hi = cap; hi >= 1; hi -= 32) {
      const int myL = hi - lane;
      const int c = myL >= 1 ? cnt[myL] : 0;
      const unsigned pm = __ballot_sync(full, c > 0);
      if (c > 0) cls[ncls + __popc(pm & lt)] = make_int2(myL, c);
      ncls += __popc(pm);
    }
    __syncwarp();
    // (2) placement.  Bins not yet opened hold room = cap, so the lowest bin with room ≥ L is the
    //     first fit when one exists and otherwise the next fresh bin: two ballots, no bin count
    //     test on the critical path.  Classes are read 32 at a time into registers; the owner lane
    //     of the chosen bin records the run in an smem ring (one 16-B store) that the warp flushes
    //     to the run arrays every 32 runs, and the per-class run ranges are written once per 32
    //     classes — a single-warp loop is latency-bound, so every instruction on it counts.
    int4* ring = reinterpret_cast<int4*>(act_cnt);  // [32] run records (bin, cum, tok, mem)
    auto flush = [&](int base, int cnt) {
      __syncwarp();
      if (lane < cnt) {
        const int4 rr = ring[lane];
        ws.run_bin[base + lane] = rr.x;
        ws.run_cum[base + lane] = rr.y;
        ws.run_tok[base + lane] = rr.z;
        ws.run_mem[base + lane] = rr.w;
      }
      __syncwarp();
    };
    int rem[2] = {cap, cap}, mem[2] = {0, 0};
    int nb = 0, nruns = 0;
    for (int base = 0; base < ncls; base += 32) {
      const int2 my = base + lane < ncls ? cls[base + lane] : make_int2(0, 0);
      const int ne = min(32, ncls - base);
      int my_start = 0;  // first run of class base + lane
      for (int e = 0; e < ne; ++e) {
        const int L = __shfl_sync(full, my.x, e), c = __shfl_sync(full, my.y, e);
        if (lane == e) my_start = nruns;
        int placed = 0;
        while (true) {  // one run per iteration
          const unsigned m0 = __ballot_sync(full, rem[0] >= L);
          const unsigned m1 = __ballot_sync(full, rem[1] >= L);
          const int b = m0 ? __ffs(m0) - 1 : 31 + __ffs(m1);
          // branch-free owner update (selects, one predicated store): no divergence on the chain
          const bool h = m0 == 0, own = lane == (b & 31);
          const int rb = h ? rem[1] : rem[0], cb = h ? mem[1] : mem[0];
          int take = 1;  // room ≥ L is guaranteed (first fit or a fresh bin): one item needs no division
          if (c - placed > 1) take = min(udiv_small(rb, L, __frcp_rn(float(L))), c - placed);  // uniform test
          if (own) ring[nruns & 31] = make_int4(b, placed, cap - rb, cb);
          rem[0] = own && !h ? rb - take * L : rem[0];
          rem[1] = own && h ? rb - take * L : rem[1];
          mem[0] = own && !h ? cb + take : mem[0];
          mem[1] = own && h ? cb + take : mem[1];
          nb = max(nb, b + 1);
          if ((++nruns & 31) == 0) flush(nruns - 32, 32);
          if (c == 1) break;  // c is warp-uniform
          placed += __shfl_sync(full, take, b & 31);
          if (placed >= c) break;
        }
      }
      const int nxt = __shfl_down_sync(full, my_start, 1);
      if (lane < ne) {
        ws.class_run_start[my.x] = my_start;
        ws.class_nruns[my.x] = (lane + 1 < ne ? nxt : nruns) - my_start;
      }
    }
    flush(nruns & ~31, nruns & 31);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (32 * h + lane < nb) {
        out.bin_count[32 * h + lane] = mem[h];
        out.bin_fill[32 * h + lane] = cap - rem[h];
      }
    if (lane == 0) *out.num_bins = nb;
    return;
  }
  // General path: the open bins in smem with a per-32-bin maximum of the room (cmax), so a class
  // visits only the chunks that have room for it — 32 chunk maxima per ballot — instead of every
  // bin from the first (1M long-tailed samples: ~487 classes over ~6.4k bins).
  int32_t* cmax = sm + 2 * kWarpMaxBins + (cnt_smem ? cap + 1 : 0);  // [kWarpMaxBins / 32]
  auto chunk_max = [&](int ch, int nbins) {  // recompute cmax[ch] from the bins themselves
    const int b = ch * 32 + lane;
    const int v = __reduce_max_sync(full, unsigned(b < nbins ? act_rem[b] : 0));  // REDUX: one instruction
    if (lane == 0) cmax[ch] = v;
  };
  int nb = 0, nruns = 0;
  for (int hi = cap; hi >= 1; hi -= 32) {
    const int myL = hi - lane;
    unsigned present = __ballot_sync(full, myL >= 1 && cnt[myL > 0 ? myL : 0] > 0);
    while (present) {
      const int k = __ffs(present) - 1;  // lowest lane = largest L
      present &= present - 1;
      const int L = hi - k;
      const int c = cnt[L];
      const float invL = __frcp_rn(float(L));
      const int runs_before = nruns;
      int running = 0;  // items of class L accounted for by bins visited so far (Σq)
      const int nch = (nb + 31) >> 5;
      for (int g0 = 0; g0 < nch && running < c; g0 += 32) {
        unsigned cm = __ballot_sync(full, g0 + lane < nch && cmax[g0 + lane] >= L);
        while (cm && running < c) {
          const int ch = g0 + __ffs(cm) - 1;
          cm &= cm - 1;
          const int b = ch * 32 + lane;
          const int rem = b < nb ? act_rem[b] : 0;
          const int q = udiv_small(rem, L, invL);
          int inc = q;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(full, inc, o);
            if (lane >= o) inc += t;
          }
          const int before = running + inc - q;
          const bool takes = q > 0 && before < c;
          const unsigned tm = __ballot_sync(full, takes);
          int nrem = rem;
          if (takes) {
            const int take = min(q, c - before);
            const int r = nruns + __popc(tm & lt);
            ws.run_bin[r] = b;
            ws.run_cum[r] = before;
            ws.run_tok[r] = cap - rem;
            ws.run_mem[r] = act_cnt[b];
            nrem = rem - take * L;
            act_rem[b] = nrem;
            act_cnt[b] += take;
          }
          nruns += __popc(tm);
          running += __shfl_sync(full, inc, 31);
          const int mx = __reduce_max_sync(full, unsigned(nrem));
          if (lane == 0) cmax[ch] = mx;
          __syncwarp();
        }
      }
      const int placed = min(c, running);
      const int r = c - placed;
      if (r > 0) {
        const int kk = udiv_small(cap, L, invL);
        const int nnew = udiv_small(r + kk - 1, kk, __frcp_rn(float(kk)));
        if (nb + nnew > kWarpMaxBins) {  // (unreachable: nb stays below the bound checked above)
          if (lane == 0) {
            out.status[0] = VLASIM_ECONFIG;
            out.status[1] = -2;
          }
          return;
        }
        for (int j = lane; j < nnew; j += 32) {
          const int take = min(kk, r - j * kk);
          ws.run_bin[nruns + j] = nb + j;
          ws.run_cum[nruns + j] = placed + j * kk;
          ws.run_tok[nruns + j] = 0;
          ws.run_mem[nruns + j] = 0;
          act_rem[nb + j] = cap - take * L;
          act_cnt[nb + j] = take;
        }
        __syncwarp();
        for (int ch = nb >> 5; ch <= (nb + nnew - 1) >> 5; ++ch) chunk_max(ch, nb + nnew);
        __syncwarp();
        nb += nnew;
        nruns += nnew;
      }
      if (lane == 0) {
        ws.class_run_start[L] = runs_before;
        ws.class_nruns[L] = nruns - runs_before;
      }
      __syncwarp();
    }
  }
  for (int b = lane; b < nb; b += 32) {
    out.bin_count[b] = act_cnt[b];
    out.bin_fill[b] = cap - act_rem[b];
  }
  if (lane == 0) *out.num_bins = nb;
}

// ------------------------------------------------------------------ stable ranks → bins
// kGlobal (cap > kSmemHistMaxCap): the running ranks advance in the chunk's own chunk_hist row
// (the exclusive class base; nothing reads it afterwards).
template <bool kGlobal>
__global__ void __launch_bounds__(kRankThreads) k_assign(const int32_t* __restrict__ len, int64_t n, int cap,
                                                          PackWs ws, vlasim_pack_out out) {
  extern __shared__ int32_t cnt_[];  // [cap+1] running per-class rank inside this chunk
  if (out.status[0] != 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t* base = ws.chunk_hist + size_t(blockIdx.x) * (cap + 1);
  int32_t* cnt = kGlobal ? base : cnt_;
  if (!kGlobal) {
    for (int i = tid; i <= cap; i += blockDim.x) cnt[i] = base[i];
    __syncthreads();
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int round = 0; round < kChunk / kRankThreads; ++round) {
    if (int64_t(blockIdx.x) * kChunk + round * kRankThreads >= n) break;  // uniform
    const int64_t i = int64_t(blockIdx.x) * kChunk + round * kRankThreads + tid;
    const bool valid = i < n;
    const int L = valid ? len[i] : -1 - lane;  // invalid lanes never match anyone
    const unsigned peers = __match_any_sync(0xffffffffu, L);
    const int leader = __ffs(peers) - 1;
    const int before = __popc(peers & lt_mask);
    int rank0 = 0;
    for (int w = 0; w < kRankThreads / 32; ++w) {
      if (w == warp && valid && lane == leader) {
        rank0 = cnt[L];
        cnt[L] = rank0 + __popc(peers);
      }
      __syncthreads();
    }
    rank0 = __shfl_sync(0xffffffffu, rank0, leader);
    if (!valid) continue;
    const int rank = rank0 + before;
    // binary search the run of class L containing `rank`
    int lo = ws.class_run_start[L], hi = lo + ws.class_nruns[L] - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ws.run_cum[mid] <= rank) lo = mid; else hi = mid - 1;
    }
    const int within = rank - ws.run_cum[lo];
    out.bin_of[i] = ws.run_bin[lo];
    out.slot[i] = ws.run_mem[lo] + within;
    out.tok_off[i] = ws.run_tok[lo] + within * L;
  }
}

// ------------------------------------------------------------------ greedy (arrival order)
// Streaming first-fit in id order: sample i goes to the lowest-index bin whose
// remaining room is >= len[i] (a fresh bin has room cap, so the first unopened bin always
// qualifies).  Inherently sequential; one warp walks a 32-ary max-tree of remaining room:
//   n <= 32768 : 3 levels in shared memory (bins = level 0, 32768 of them);
//   n >  32768 : 4 levels (2^20 bins) — level 0 (room, count) in the workspace (L2-resident),
//                levels 1-3 in shared memory; one coalesced 128-B load per sample.
// Each descent step is one ballot; the update walks back up with warp max-reductions over the
// 32 values each lane already holds in registers (no re-read after the owner's store).
constexpr int kGreedyMaxBins = 32768;
constexpr size_t kGreedySmem = (2 * kGreedyMaxBins + 1024 + 32) * sizeof(uint16_t);
constexpr size_t kGreedyDeepSmem = (kGreedyMaxBins + 1024 + 32) * sizeof(uint16_t);

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void k_greedy_fill(int32_t* __restrict__ rem0, int32_t* __restrict__ cnt0, int64_t nb, int cap) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < nb) {
    rem0[i] = cap;
    cnt0[i] = 0;
  }
}

template <bool kDeep>
__global__ void __launch_bounds__(32, 1) k_greedy(const int32_t* __restrict__ len, int64_t n, int cap,
                                                  PackWs ws, vlasim_pack_out out) {
  extern __shared__ uint16_t gsm[];
  // shallow: rem0/cnt = bins in smem; deep: g_rem/g_cnt = bins in HBM, rem0 = level-1 maxima
  uint16_t* rem0 = gsm;                                      // [32768]
  uint16_t* cnt = kDeep ? nullptr : rem0 + kGreedyMaxBins;   // [32768] (shallow)
  uint16_t* rem1 = rem0 + (kDeep ? 1 : 2) * kGreedyMaxBins;  // [1024]
  uint16_t* rem2 = rem1 + 1024;                              // [32]
  const int64_t gstride = (n + 31) & ~int64_t(31);
  int32_t* g_rem = ws.spill;
  int32_t* g_cnt = ws.spill + gstride;
  const int lane = threadIdx.x;
  if (out.status[0] != 0) return;  // invalid lengths (k_hist)
  for (int i = lane; i < kGreedyMaxBins; i += 32) {
    rem0[i] = uint16_t(cap);
    if (!kDeep) cnt[i] = 0;
  }
  for (int i = lane; i < 1024; i += 32) rem1[i] = uint16_t(cap);
  rem2[lane] = uint16_t(cap);
  __syncwarp();
  int nb = 0;
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t my = base + lane;
    const int lm = my < n ? len[my] : 0;
    const int cntv = int(n - base < 32 ? n - base : 32);
    int ob = 0, os = 0, ot = 0;  // results of sample base + lane
    for (int j = 0; j < cntv; ++j) {
      const int L = __shfl_sync(0xffffffffu, lm, j);
      const unsigned m2 = __ballot_sync(0xffffffffu, rem2[lane] >= L);
      if (m2 == 0) {  // every bin of the tree is too full: out of tree capacity
        if (lane == 0) {
          out.status[1] = -4;
          out.status[0] = VLASIM_ECONFIG;
        }
        return;
      }
      const int j2 = __ffs(m2) - 1;
      const int j1 = j2 * 32 + __ffs(__ballot_sync(0xffffffffu, rem1[j2 * 32 + lane] >= L)) - 1;
      int v0 = rem0[j1 * 32 + lane];
      int b = j1 * 32 + __ffs(__ballot_sync(0xffffffffu, v0 >= L)) - 1;
      int r, c;
      if (kDeep) {  // one more level: the 32 bins under node b live in HBM
        const int64_t g = int64_t(b) * 32 + lane;
        const int vg = g < gstride ? g_rem[g] : 0;
        const unsigned mg = __ballot_sync(0xffffffffu, vg >= L);
        const int jg = __ffs(mg) - 1;  // node b has max >= L, so some bin under it qualifies
        const int64_t bb = int64_t(b) * 32 + jg;
        r = __shfl_sync(0xffffffffu, vg, jg);
        c = lane == 0 ? g_cnt[bb] : 0;
        c = __shfl_sync(0xffffffffu, c, 0);
        const int vg2 = lane == jg ? vg - L : vg;
        if (lane == jg) g_rem[bb] = vg2;
        if (lane == 0) g_cnt[bb] = c + 1;
        const int mx = warp_max(vg2);  // new maximum of node b
        if (lane == (b & 31)) v0 = mx;
        if (lane == 0) rem0[b] = uint16_t(mx);
        b = int(bb);
      } else {
        r = __shfl_sync(0xffffffffu, v0, b & 31);
        c = cnt[b];
        if (lane == (b & 31)) v0 -= L;
        __syncwarp();
        if (lane == 0) {
          rem0[b] = uint16_t(r - L);
          cnt[b] = uint16_t(c + 1);
        }
      }
      const int v1 = warp_max(v0);
      __syncwarp();
      if (lane == 0) rem1[j1] = uint16_t(v1);
      __syncwarp();
      const int v2 = warp_max(rem1[j2 * 32 + lane]);
      if (lane == 0) rem2[j2] = uint16_t(v2);
      __syncwarp();
      if (lane == j) {
        ob = b;
        os = c;
        ot = cap - r;
      }
      nb = max(nb, b + 1);
    }
    if (my < n) {
      out.bin_of[my] = ob;
      out.slot[my] = os;
      out.tok_off[my] = ot;
    }
  }
  for (int b = lane; b < nb; b += 32) {
    out.bin_count[b] = kDeep ? g_cnt[b] : cnt[b];
    out.bin_fill[b] = cap - (kDeep ? g_rem[b] : rem0[b]);
  }
  if (lane == 0) *out.num_bins = nb;
}

// ------------------------------------------------------------------ device-wide scans
// Exclusive scan of int32 in[0..n) (+ total at out[n]) in three passes; partial sums int64.
__global__ void k_scan_reduce(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ part) {
  __shared__ int64_t scratch[33];
  int64_t s = 0;
  const int64_t b = int64_t(blockIdx.x) * kScanItems;
  for (int j = threadIdx.x; j < kScanItems; j += blockDim.x) {
    const int64_t i = b + j;
    if (i < n) s += in[i];
  }
  int64_t tot;
  block_exclusive_scan<int64_t>(s, scratch, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}
__global__ void k_scan_parts(int64_t* part, int64_t nparts, int64_t* total_out) {
  __shared__ int64_t scratch[33];
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nparts; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < nparts ? part[i] : 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan<int64_t>(v, scratch, &tot);
    if (i < nparts) part[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}
template <typename OutT>
__global__ void k_scan_apply(const int32_t* __restrict__ in, int64_t n, const int64_t* __restrict__ part,
                             OutT* __restrict__ out, int32_t* status) {
  __shared__ int64_t scratch[33];
  const int64_t b = int64_t(blockIdx.x) * kScanItems;
  const int64_t i0 = b + threadIdx.x * 4;
  int64_t v[4], s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[j] = (i0 + j < n) ? in[i0 + j] : 0;
    s += v[j];
  }
  int64_t tot;
  int64_t run = part[blockIdx.x] + block_exclusive_scan<int64_t>(s, scratch, &tot);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t i = i0 + j;
    if (i <= n) {
      if (run > INT_MAX && status) {
        status[0] = VLASIM_ECONFIG;
        status[1] = -3;  // token count overflows int32 cu_seqlens
      }
      out[i] = OutT(run);
    }
    run += v[j];
  }
}

// ------------------------------------------------------------------ layout
// On a device-side input error (status set upstream; the caller may not synchronise — the CUDA
// graph path) the plan is left DEFINED and empty: every cu_seqlens entry 0 and num_bins 0, so
// kernels stream-ordered after the packer see zero-length segments and do no work.
__global__ void k_layout(const int32_t* __restrict__ len, int64_t n, vlasim_pack_out out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (out.status[0] != 0) {
    if (i < n) out.cu_seqlens[i] = 0;
    if (i == 0) {
      out.cu_seqlens[n] = 0;
      *out.num_bins = 0;
    }
    return;
  }
  if (i >= n) return;
  const int b = out.bin_of[i], s = out.slot[i], t = out.tok_off[i];
  const int mo = out.bin_member_off[b];
  const int m = mo + s;
  out.member_ids[m] = int32_t(i);
  out.cu_seqlens[m] = out.bin_token_off[b] + t;
  int32_t* cb = out.cu_seqlens_bins + mo + b;
  cb[s + 1] = t + len[i];
  if (s == 0) cb[0] = 0;
  if (i == 0) out.cu_seqlens[n] = out.bin_token_off[n];
}

__global__ void k_token_ids(const int32_t* __restrict__ len, vlasim_pack_out out, int64_t n, int32_t* pos_ids,
                            int32_t* seg_ids, int32_t* gather_idx) {
  // one warp per segment (grid-stride)
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t m = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32; m < n; m += warps) {
    const int id = out.member_ids[m];
    const int start = out.cu_seqlens[m];
    const int L = len[id];
    const int src = out.src_off[id];
    for (int p = lane; p < L; p += 32) {
      if (pos_ids) pos_ids[start + p] = p;
      if (seg_ids) seg_ids[start + p] = int32_t(m);
      if (gather_idx) gather_idx[start + p] = src + p;
    }
  }
}

// One CTA per segment: contiguous copy of len × row_bytes with 16-byte vectors, 4 in flight.
template <bool kGather>
__global__ void __launch_bounds__(256) k_copy_rows(const uint4* __restrict__ a, uint4* __restrict__ b,
                                                   int64_t row_vecs, const int32_t* __restrict__ len,
                                                   vlasim_pack_out out) {
  const int64_t m = blockIdx.x;
  const int id = out.member_ids[m];
  const int64_t nvec = int64_t(len[id]) * row_vecs;
  const int64_t packed = int64_t(out.cu_seqlens[m]) * row_vecs;
  const int64_t source = int64_t(out.src_off[id]) * row_vecs;
  const uint4* src = a + (kGather ? source : packed);
  uint4* dst = b + (kGather ? packed : source);
  const int64_t stride = 4 * blockDim.x;
  int64_t j = threadIdx.x;
  for (; j + 3 * blockDim.x < nvec; j += stride) {
    uint4 v0 = __ldcs(src + j), v1 = __ldcs(src + j + blockDim.x), v2 = __ldcs(src + j + 2 * blockDim.x),
          v3 = __ldcs(src + j + 3 * blockDim.x);
    __stcs(dst + j, v0);
    __stcs(dst + j + blockDim.x, v1);
    __stcs(dst + j + 2 * blockDim.x, v2);
    __stcs(dst + j + 3 * blockDim.x, v3);
  }
  for (; j < nvec; j += blockDim.x) __stcs(dst + j, __ldcs(src + j));
}

int run_scan(const int32_t* in, int64_t n, int32_t* out, int64_t* part, int64_t* total, int32_t* status,
             cudaStream_t st) {
  const int64_t nb = num_scan_blocks(n);
  k_scan_reduce<<<nb, 1024, 0, st>>>(in, n, part);
  k_scan_parts<<<1, 1024, 0, st>>>(part, nb, total);
  k_scan_apply<int32_t><<<nb, 1024, 0, st>>>(in, n, part, out, status);
  return 0;
}

// validation + per-chunk length histogram (smem counters up to kSmemHistMaxCap, HBM beyond)
int launch_hist(const int32_t* d_len, int64_t n, int cap, const PackWs& w, const vlasim_pack_out* out,
                cudaStream_t st) {
  const int64_t nchunks = num_chunks(n);
  if (cap <= kSmemHistMaxCap) {
    if ((cap + 1) * 4 > 48 * 1024)
      VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_hist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (cap + 1) * 4));
    k_hist<false><<<nchunks, 512, (cap + 1) * 4, st>>>(d_len, n, cap, w.chunk_hist, out->status);
  } else {
    VLASIM_CUDA_TRY(cudaMemsetAsync(w.chunk_hist, 0, size_t(nchunks) * (cap + 1) * 4, st));
    k_hist<true><<<nchunks, 512, 0, st>>>(d_len, n, cap, w.chunk_hist, out->status);
  }
  return VLASIM_OK;
}

int check_out(const vlasim_pack_out* o) {
  if (!o || !o->bin_of || !o->slot || !o->tok_off || !o->bin_count || !o->bin_fill || !o->bin_member_off ||
      !o->bin_token_off || !o->member_ids || !o->cu_seqlens || !o->cu_seqlens_bins || !o->src_off || !o->num_bins ||
      !o->total_tokens || !o->status)
    return vlasim_host::set_error(VLASIM_ECONFIG, "vlasim_pack_out: every output pointer must be set");
  return 0;
}

int finish(const vlasim_pack_out* out, int64_t n, uint32_t flags, cudaStream_t st) {
  using namespace vlasim_host;
  if (!(flags & VLASIM_PACK_SYNC_CHECK)) return VLASIM_OK;
  int32_t h[2];
  VLASIM_CUDA_TRY(cudaMemcpyAsync(h, out->status, sizeof(h), cudaMemcpyDeviceToHost, st));
  VLASIM_CUDA_TRY(cudaStreamSynchronize(st));
  if (h[0] == 0) return VLASIM_OK;
  if (h[1] == -3) return set_error(VLASIM_ECONFIG, "GPU packer: total tokens exceed int32 cu_seqlens range");
  if (h[1] == -4) return set_error(VLASIM_ECONFIG, "greedy packer: more than %d bins", kGreedyDeepMaxBins);
  return set_error(VLASIM_ECONFIG, "oversize or empty sample: id %d (length must be in [1, capacity])", h[1]);
}

}  // namespace

extern "C" size_t vlasim_pack_workspace_size(int64_t n, int32_t capacity) {
  PackWs w;
  return carve(&w, nullptr, n < 1 ? 1 : n, capacity < 1 ? 1 : capacity);
}

extern "C" int vlasim_pack_ffd_cuda(const int32_t* d_len, int64_t n, int32_t cap, const vlasim_pack_out* out,
                                    void* d_ws, size_t ws_bytes, uint32_t flags, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = check_out(out)) return rc;
  if (n < 1) return set_error(VLASIM_ECONFIG, "pack_ffd: need at least one sample (n=%lld)", (long long)n);
  if (n >= INT_MAX) return set_error(VLASIM_ECONFIG, "pack_ffd: n=%lld exceeds int32 ids", (long long)n);
  if (cap < 1 || cap > VLASIM_PACK_MAX_CAPACITY)
    return set_error(VLASIM_ECONFIG, "pack_ffd: capacity %d outside [1, %d]", cap, VLASIM_PACK_MAX_CAPACITY);
  PackWs w;
  const size_t need = carve(&w, nullptr, n, cap);
  if (!d_ws || ws_bytes < need)
    return set_error(VLASIM_ECONFIG, "pack_ffd: workspace too small (%zu < %zu)", ws_bytes, need);
  carve(&w, d_ws, n, cap);
  cudaStream_t st = as_stream(stream);
  const int64_t nchunks = num_chunks(n);

  k_init<<<(n + 255) / 256, 256, 0, st>>>(*out, n);
  if (int rc = launch_hist(d_len, n, cap, w, out, st)) return rc;
  k_class_scan<<<(cap + 1 + 255) / 256, 256, 0, st>>>(w.chunk_hist, nchunks, cap, w.class_count);
  {  // the warp packer takes every batch whose bin count is bounded by its smem bin arrays
    const size_t wsm = (2 * kWarpMaxBins + (cap <= kWarpCntMaxCap ? cap + 1 : 0) + kWarpMaxBins / 32) * 4;
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_ffd_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
    k_ffd_warp<<<1, 32, wsm, st>>>(n, cap, w, *out);
  }
  if (n > kWarpMaxBins) {  // the 1024-thread packer (returns at once when the warp placed the batch)
    const size_t ffd_smem = (3 * kMaxActiveBins + 1024) * 4;
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_ffd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ffd_smem));
    k_ffd<<<1, 1024, ffd_smem, st>>>(int(n), cap, w, *out);
  }
  if (cap <= kSmemHistMaxCap) {
    const size_t as_smem = (cap + 1) * 4;
    if (as_smem > 48 * 1024)
      VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_assign<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)as_smem));
    k_assign<false><<<nchunks, kRankThreads, as_smem, st>>>(d_len, n, cap, w, *out);
  } else {
    k_assign<true><<<nchunks, kRankThreads, 0, st>>>(d_len, n, cap, w, *out);
  }
  const int64_t nsb = num_scan_blocks(n) + 1;
  run_scan(out->bin_count, n, out->bin_member_off, w.scan_part, nullptr, nullptr, st);
  run_scan(out->bin_fill, n, out->bin_token_off, w.scan_part + nsb, nullptr, out->status, st);
  run_scan(d_len, n, out->src_off, w.scan_part + 2 * nsb, out->total_tokens, out->status, st);
  k_layout<<<(n + 255) / 256, 256, 0, st>>>(d_len, n, *out);
  VLASIM_LAUNCH_CHECK();
  return finish(out, n, flags, st);
}

extern "C" int vlasim_pack_token_ids_cuda(const int32_t* d_len, const vlasim_pack_out* out, int64_t n,
                                          int64_t total_tokens, int32_t* d_pos, int32_t* d_seg, int32_t* d_gather,
                                          vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = check_out(out)) return rc;
  if (n < 1 || total_tokens < 1) return set_error(VLASIM_ECONFIG, "token_ids: empty input");
  const int64_t warps_needed = n;
  const int64_t blocks = std::min<int64_t>((warps_needed + 7) / 8, int64_t(num_sms()) * 16);
  k_token_ids<<<blocks, 256, 0, as_stream(stream)>>>(d_len, *out, n, d_pos, d_seg, d_gather);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

static int copy_rows(bool gather, const void* a, void* b, int64_t row_bytes, const int32_t* d_len,
                     const vlasim_pack_out* out, int64_t n, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = check_out(out)) return rc;
  if (row_bytes <= 0 || row_bytes % 16) return set_error(VLASIM_ECONFIG, "row_bytes must be a positive multiple of 16");
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)
    return set_error(VLASIM_ECONFIG, "gather/scatter buffers must be 16-byte aligned");
  if (n < 1) return VLASIM_OK;
  auto kern = gather ? k_copy_rows<true> : k_copy_rows<false>;
  kern<<<n, 256, 0, as_stream(stream)>>>(static_cast<const uint4*>(a), static_cast<uint4*>(b), row_bytes / 16, d_len,
                                        *out);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

extern "C" int vlasim_gather_rows_cuda(const void* d_src, void* d_dst, int64_t row_bytes, const int32_t* d_len,
                                       const vlasim_pack_out* out, int64_t n, vlasim_stream_t stream) {
  return copy_rows(true, d_src, d_dst, row_bytes, d_len, out, n, stream);
}
extern "C" int vlasim_scatter_rows_cuda(const void* d_packed, void* d_dst, int64_t row_bytes, const int32_t* d_len,
                                        const vlasim_pack_out* out, int64_t n, vlasim_stream_t stream) {
  return copy_rows(false, d_packed, d_dst, row_bytes, d_len, out, n, stream);
}

// seg_src[m] = src_off[member_ids[m]]: source row of packed segment m (attention's seg_src).
__global__ void k_seg_src(const int32_t* __restrict__ member_ids, const int32_t* __restrict__ src_off, int64_t n,
                          int32_t* __restrict__ seg_src) {
  const int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (m < n) seg_src[m] = __ldg(src_off + __ldg(member_ids + m));
}

extern "C" int vlasim_pack_seg_src_cuda(const vlasim_pack_out* out, int64_t n, int32_t* d_seg_src,
                                        vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = check_out(out)) return rc;
  if (!d_seg_src) return set_error(VLASIM_ECONFIG, "pack_seg_src: output required");
  if (n < 1) return VLASIM_OK;
  k_seg_src<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(out->member_ids, out->src_off, n, d_seg_src);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

extern "C" int vlasim_pack_greedy_cuda(const int32_t* d_len, int64_t n, int32_t cap, const vlasim_pack_out* out,
                                       void* d_ws, size_t ws_bytes, uint32_t flags, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (int rc = check_out(out)) return rc;
  if (n < 1) return set_error(VLASIM_ECONFIG, "pack_greedy: need at least one sample (n=%lld)", (long long)n);
  if (n >= INT_MAX) return set_error(VLASIM_ECONFIG, "pack_greedy: n=%lld exceeds int32 ids", (long long)n);
  if (cap < 1 || cap > VLASIM_PACK_MAX_CAPACITY)
    return set_error(VLASIM_ECONFIG, "pack_greedy: capacity %d outside [1, %d]", cap, VLASIM_PACK_MAX_CAPACITY);
  PackWs w;
  const size_t need = carve(&w, nullptr, n, cap);
  if (!d_ws || ws_bytes < need)
    return set_error(VLASIM_ECONFIG, "pack_greedy: workspace too small (%zu < %zu)", ws_bytes, need);
  carve(&w, d_ws, n, cap);
  cudaStream_t st = as_stream(stream);
  k_init<<<(n + 255) / 256, 256, 0, st>>>(*out, n);
  if (int rc = launch_hist(d_len, n, cap, w, out, st)) return rc;  // validation
  if (n <= kGreedyMaxBins) {  // at most n bins: the 3-level smem tree holds them all
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_greedy<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGreedySmem));
    k_greedy<false><<<1, 32, kGreedySmem, st>>>(d_len, n, cap, w, *out);
  } else {
    const int64_t gstride = (n + 31) & ~int64_t(31);
    const int64_t nfill = std::min<int64_t>(gstride, kGreedyDeepMaxBins);
    k_greedy_fill<<<(nfill + 255) / 256, 256, 0, st>>>(w.spill, w.spill + gstride, nfill, cap);
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_greedy<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGreedyDeepSmem));
    k_greedy<true><<<1, 32, kGreedyDeepSmem, st>>>(d_len, n, cap, w, *out);
  }
  const int64_t nsb = num_scan_blocks(n) + 1;
  run_scan(out->bin_count, n, out->bin_member_off, w.scan_part, nullptr, nullptr, st);
  run_scan(out->bin_fill, n, out->bin_token_off, w.scan_part + nsb, nullptr, out->status, st);
  run_scan(d_len, n, out->src_off, w.scan_part + 2 * nsb, out->total_tokens, out->status, st);
  k_layout<<<(n + 255) / 256, 256, 0, st>>>(d_len, n, *out);
  VLASIM_LAUNCH_CHECK();
  return finish(out, n, flags, st);
}
