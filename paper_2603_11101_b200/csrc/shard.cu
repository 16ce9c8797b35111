// shard.cu — length-balanced sharding of packs across ranks, on the device.
//
// Packs are independent (block-diagonal attention never crosses a pack), so the
// path shards by pack with no collective on the attention path.  After the single all-gather of the
// per-rank lengths every rank runs the same GPU FFD and then this kernel, which computes the same
// deterministic LPT assignment on every rank and this rank's share of the packed stream — without a
// host round trip, so the whole per-step sharding stays stream-ordered (and graph-capturable):
//
//   cost(b)  = Σ l² over the members of bin b (bidirectional visible pairs, the attention work)
//   LPT      bins by (cost desc, bin asc), each to the least-loaded rank (ties: lowest rank)
//            — the same rule as paper_2603_11101_b200/dist.py:lpt (host, tests)
//   local    the rank's bins in bin-index order, members in order: local cu_seqlens, the member
//            sample ids, each local sample's row in the rank's sample-major layout (samples in id
//            order) and each local segment's source row (vlasim_attn_args.seg_src)
//
// Bin level in one CTA of 1024 threads (k_shard_bins): per-bin costs one warp per bin, a bitonic sort
// of ≤ 16384 64-bit bin keys in shared memory, the greedy assignment by one thread (loads in
// registers, world ≤ 16), block scans over the bins.  Sample level device-wide (k_shard_scan_*): the
// local sample-major offsets by a three-pass scan and the scatter of every local sample to its
// segment slot.  Metadata only (a few bytes per sample).
#include <algorithm>
#include <climits>

#include "common.hpp"
#include "scan.cuh"

using namespace vlasim_dev;

namespace {

constexpr int kShardThreads = 1024;
constexpr int kMaxShardBins = 16384;
constexpr int kMaxWorld = 16;

struct ShardIn {
  const int32_t* len;
  const int32_t* bin_of;
  const int32_t* slot;
  const int32_t* tok_off;
  const int32_t* bin_count;
  const int32_t* bin_fill;
  const int32_t* bin_member_off;
  const int32_t* member_ids;
  const int32_t* num_bins;
};

// Block-wide exclusive scan of `count` int64 values produced by f(i), chunked per thread (each thread
// owns a contiguous range).  Calls out(i, exclusive_prefix) for every i; returns the total.
template <typename F, typename G>
__device__ int64_t block_scan_chunked(int64_t count, F f, G out, int64_t* scratch) {
  const int64_t per = (count + kShardThreads - 1) / kShardThreads;
  const int64_t b0 = per * int64_t(threadIdx.x), b = b0 < count ? b0 : count, e = b + per < count ? b + per : count;
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += f(i);
  int64_t total;
  int64_t run = block_exclusive_scan<int64_t>(s, scratch, &total);
  for (int64_t i = b; i < e; ++i) {
    const int64_t v = f(i);
    out(i, run);
    run += v;
  }
  __syncthreads();
  return total;
}

// ---- 0: per-bin cost Σ l² over the whole grid (integer atomics: order-independent, deterministic)
__global__ void k_shard_cost(ShardIn in, int64_t n, unsigned long long* __restrict__ cost) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long l = unsigned(in.len[i]);
    atomicAdd(cost + in.bin_of[i], l * l);
  }
}

// ---- 1: bin keys (cost, bin) sorted descending in shared memory by one CTA (bitonic)
__global__ void __launch_bounds__(kShardThreads) k_shard_bins(ShardIn in, vlasim_shard_out o,
                                                              unsigned long long* __restrict__ cost) {
  extern __shared__ unsigned long long keys[];  // [P] sort keys, P = next pow2 >= bins
  unsigned long long* sorted = cost;            // the sorted keys replace the costs in place
  const int B = *in.num_bins;
  if (B > kMaxShardBins) {
    if (threadIdx.x == 0) o.status[0] = VLASIM_ECONFIG, o.status[1] = B;
    return;
  }
  if (threadIdx.x == 0) o.status[0] = 0, o.status[1] = 0;
  int P = 1;
  while (P < B) P <<= 1;
  // key = cost · 2^32 + (2^32 − 1 − b): descending order = (cost desc, b asc); cost from k_shard_cost
  for (int b = threadIdx.x; b < P; b += kShardThreads)
    keys[b] = b < B ? (cost[b] << 32) | (0xFFFFFFFFull - unsigned(b)) : 0ull;
  __syncthreads();
  // bitonic sort, descending
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += kShardThreads) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          const unsigned long long a = keys[i], c = keys[j];
          if (desc ? a < c : a > c) keys[i] = c, keys[j] = a;
        }
      }
      __syncthreads();
    }
  for (int b = threadIdx.x; b < B; b += kShardThreads) sorted[b] = keys[b];
}

// ---- 2: greedy LPT over the sorted keys (staged in shared memory by the warp), one thread with the
// rank loads in registers
// W = world (the per-bin chain is one thread's, so its width is compiled for the rank count).
template <int W>
__global__ void __launch_bounds__(32, 1) k_shard_lpt(ShardIn in, int world, vlasim_shard_out o,
                                                     const unsigned long long* __restrict__ gkeys) {
  extern __shared__ unsigned long long keys[];
  if (o.status[0]) return;
  const int B = *in.num_bins;
  for (int b = threadIdx.x; b < B; b += 32) keys[b] = gkeys[b];
  __syncwarp();
  if (threadIdx.x != 0) return;
  // greedy LPT (one thread): rank r's load packed with its index, key_r = load_r · 16 + r, so the
  // least-loaded rank (ties: lowest rank) is the minimum key — 15 independent 64-bit mins per bin
  // (a 4-level tree) after one predicated add; unused ranks hold UINT64_MAX.
  unsigned long long kr[W];
#pragma unroll
  for (int r = 0; r < W; ++r) kr[r] = r < world ? static_cast<unsigned long long>(r) : ~0ull;
  constexpr int P2 = W <= 1 ? 1 : W <= 2 ? 2 : W <= 4 ? 4 : W <= 8 ? 8 : 16;
  auto argmin = [&]() {  // a log2-level tree of independent 64-bit mins (padded to a power of two)
    unsigned long long t[P2];
#pragma unroll
    for (int j = 0; j < P2; ++j) t[j] = j < W ? kr[j] : ~0ull;
#pragma unroll
    for (int w = P2 / 2; w >= 1; w /= 2)
#pragma unroll
      for (int j = 0; j < w; ++j) t[j] = min(t[2 * j], t[2 * j + 1]);
    return t[0];
  };
  // Narrow path: greedy LPT keeps max − min rank load ≤ the largest bin cost (keys[0], the first
  // key), so with that cost below 2^27 the keys relative to the current minimum load fit 32 bits.
  // The W keys are kept SORTED in registers: the least-loaded rank is s[0]; after its load grows it
  // is re-inserted (W−1 independent compares, two selects per slot) and every key is rebased on
  // the new minimum — no min tree and no per-rank predicated add on the per-bin chain.
  if (B > 0 && (keys[0] >> 32) < (1ull << 27)) {
    uint32_t sk[W];
#pragma unroll
    for (int r = 0; r < W; ++r) sk[r] = uint32_t(r);  // load 0, rank r: sorted
    unsigned long long base = 0;  // absolute load (without the ×16) of the relative zero
    unsigned long long k = keys[0];
    for (int i = 0; i < B; ++i) {
      const unsigned long long kn = i + 1 < B ? keys[i + 1] : 0ull;
      o.bin_rank[int(0xFFFFFFFFull - (k & 0xFFFFFFFFull))] = int(sk[0] & 15);
      const uint32_t x = sk[0] + (uint32_t(k >> 32) << 4);
      bool lt[W + 1];  // lt[j]: sk[j] < x (monotone: a true prefix of 1..W−1)
      lt[0] = true;
#pragma unroll
      for (int j = 1; j < W; ++j) lt[j] = sk[j] < x;
      lt[W] = false;
      uint32_t ns[W];
#pragma unroll
      for (int q = 0; q < W; ++q) ns[q] = lt[q + 1] ? sk[q + 1 < W ? q + 1 : q] : (lt[q] ? x : sk[q]);
      const uint32_t sub = ns[0] & ~15u;  // rebase on the new minimum load
#pragma unroll
      for (int q = 0; q < W; ++q) sk[q] = ns[q] - sub;
      base += sub >> 4;
      k = kn;
    }
#pragma unroll
    for (int q = 0; q < W; ++q) o.rank_load[sk[q] & 15] = static_cast<long long>(base + (sk[q] >> 4));
    return;
  }
  unsigned long long m = argmin();
  unsigned long long k = B > 0 ? keys[0] : 0ull;
  for (int i = 0; i < B; ++i) {
    const unsigned long long kn = i + 1 < B ? keys[i + 1] : 0ull;  // next key's load in flight
    const int best = int(m & 15);
    o.bin_rank[int(0xFFFFFFFFull - (k & 0xFFFFFFFFull))] = best;
    const unsigned long long add = (k >> 32) << 4;
#pragma unroll
    for (int r = 0; r < W; ++r) kr[r] += r == best ? add : 0ull;
    m = argmin();
    k = kn;
  }
#pragma unroll
  for (int r = 0; r < W; ++r)
    if (r < world) o.rank_load[r] = static_cast<long long>(kr[r] >> 4);
}

// ---- 3: this rank's bins in index order: local member / token offsets per bin
__global__ void __launch_bounds__(kShardThreads) k_shard_binscan(ShardIn in, int rank, vlasim_shard_out o,
                                                                 int32_t* __restrict__ lmo, int32_t* __restrict__ lto) {
  __shared__ int64_t scratch[33];
  if (o.status[0]) return;
  const int B = *in.num_bins;
  // this rank's bins in index order: local member / token offsets per bin
  const int64_t nseg = block_scan_chunked(
      B, [&](int64_t b) -> int64_t { return o.bin_rank[b] == rank ? in.bin_count[b] : 0; },
      [&](int64_t b, int64_t x) { lmo[b] = int32_t(x); }, scratch);
  const int64_t ntok = block_scan_chunked(
      B, [&](int64_t b) -> int64_t { return o.bin_rank[b] == rank ? in.bin_fill[b] : 0; },
      [&](int64_t b, int64_t x) { lto[b] = int32_t(x); }, scratch);
  if (threadIdx.x == 0) {
    *o.local_nseg = int32_t(nseg);
    *o.local_tokens = ntok;
  }
}

// ---- 4: sample level, device-wide: local_src_off = exclusive scan of the local samples' lengths
// in id order (−1 for samples of other ranks), three passes over 4096-sample blocks.
constexpr int kScanItems = 4096;

__device__ __forceinline__ int64_t local_len(const ShardIn& in, const vlasim_shard_out& o, int rank, int64_t i) {
  return o.bin_rank[in.bin_of[i]] == rank ? in.len[i] : 0;
}

__global__ void __launch_bounds__(1024) k_shard_scan_reduce(ShardIn in, int64_t n, int rank, vlasim_shard_out o,
                                                            int64_t* __restrict__ part) {
  __shared__ int64_t scratch[33];
  if (o.status[0]) return;
  int64_t s = 0;
  const int64_t b = int64_t(blockIdx.x) * kScanItems;
  for (int j = threadIdx.x; j < kScanItems; j += blockDim.x) {
    const int64_t i = b + j;
    if (i < n) s += local_len(in, o, rank, i);
  }
  int64_t tot;
  block_exclusive_scan<int64_t>(s, scratch, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_shard_scan_parts(int64_t* part, int64_t nparts, const int32_t* status) {
  __shared__ int64_t scratch[33];
  if (status[0]) return;
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nparts; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < nparts ? part[i] : 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan<int64_t>(v, scratch, &tot);
    if (i < nparts) part[i] = carry + ex;
    carry += tot;
  }
}

// applies the scan and scatters every local sample to its local segment position
__global__ void __launch_bounds__(1024) k_shard_scan_apply(ShardIn in, int64_t n, int rank, vlasim_shard_out o,
                                                           const int64_t* __restrict__ part,
                                                           const int32_t* __restrict__ lmo,
                                                           const int32_t* __restrict__ lto) {
  __shared__ int64_t scratch[33];
  if (o.status[0]) return;
  const int64_t b = int64_t(blockIdx.x) * kScanItems;
  const int64_t i0 = b + threadIdx.x * 4;
  int64_t v[4], s = 0;
  int bin[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t i = i0 + j;
    bin[j] = i < n ? in.bin_of[i] : 0;
    v[j] = (i < n && o.bin_rank[bin[j]] == rank) ? in.len[i] : -1;
    s += v[j] > 0 ? v[j] : 0;
  }
  int64_t tot;
  int64_t run = part[blockIdx.x] + block_exclusive_scan<int64_t>(s, scratch, &tot);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t i = i0 + j;
    if (i >= n) break;
    if (v[j] < 0) {
      o.local_src_off[i] = -1;
      continue;
    }
    const int32_t src = int32_t(run);
    o.local_src_off[i] = src;
    const int jj = lmo[bin[j]] + in.slot[i];
    o.local_ids[jj] = int32_t(i);
    o.local_cu[jj] = lto[bin[j]] + in.tok_off[i];
    o.local_seg_src[jj] = src;
    run += v[j];
  }
}

// segments past the local count: zero length at the end of the stream
__global__ void k_shard_tail(int64_t n, vlasim_shard_out o) {
  if (o.status[0]) return;
  const int64_t nseg = *o.local_nseg, ntok = *o.local_tokens;
  for (int64_t j = nseg + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j <= n; j += int64_t(gridDim.x) * blockDim.x)
    o.local_cu[j] = int32_t(ntok);
}

}  // namespace

extern "C" size_t vlasim_shard_scratch_size(int64_t n) {
  if (n < 1) n = 1;
  const int64_t nblk = (n + kScanItems - 1) / kScanItems;
  return size_t(n) * 4 + size_t((n + 1) & ~int64_t(1)) * 4 + size_t(nblk + 1) * 8 + size_t(n) * 8;
}

extern "C" int vlasim_shard_lpt_cuda(const int32_t* d_len, const vlasim_pack_out* plan, int64_t n, int32_t world,
                                     int32_t rank, const vlasim_shard_out* out, uint32_t flags,
                                     vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (!d_len || !plan || !out) return set_error(VLASIM_ECONFIG, "shard_lpt: null argument");
  if (n < 1 || n >= INT_MAX) return set_error(VLASIM_ECONFIG, "shard_lpt: n=%lld out of range", (long long)n);
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return set_error(VLASIM_ECONFIG, "shard_lpt: world %d / rank %d out of range (world <= %d)", world, rank,
                     kMaxWorld);
  if (!out->bin_rank || !out->rank_load || !out->local_ids || !out->local_cu || !out->local_seg_src ||
      !out->local_src_off || !out->local_nseg || !out->local_tokens || !out->status)
    return set_error(VLASIM_ECONFIG, "shard_lpt: every output buffer is required");
  if (!out->scratch) return set_error(VLASIM_ECONFIG, "shard_lpt: scratch (vlasim_shard_scratch_size) is required");
  ShardIn in{d_len, plan->bin_of, plan->slot, plan->tok_off, plan->bin_count, plan->bin_fill, plan->bin_member_off,
             plan->member_ids, plan->num_bins};
  cudaStream_t st = as_stream(stream);
  int32_t* lmo = out->scratch;
  int32_t* lto = lmo + n;
  int64_t* part = reinterpret_cast<int64_t*>(lto + ((n + 1) & ~int64_t(1)));
  const int64_t nblk = (n + kScanItems - 1) / kScanItems;
  unsigned long long* cost = reinterpret_cast<unsigned long long*>(part + nblk + 1);
  VLASIM_CUDA_TRY(cudaMemsetAsync(cost, 0, size_t(n) * 8, st));
  k_shard_cost<<<int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8)), 256, 0, st>>>(in, n, cost);
  const size_t smem = size_t(kMaxShardBins) * 8;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_shard_bins, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  k_shard_bins<<<1, kShardThreads, smem, st>>>(in, *out, cost);
  using LptKernel = void (*)(ShardIn, int, vlasim_shard_out, const unsigned long long*);
  static const LptKernel lpts[kMaxWorld] = {k_shard_lpt<1>,  k_shard_lpt<2>,  k_shard_lpt<3>,  k_shard_lpt<4>,
                                            k_shard_lpt<5>,  k_shard_lpt<6>,  k_shard_lpt<7>,  k_shard_lpt<8>,
                                            k_shard_lpt<9>,  k_shard_lpt<10>, k_shard_lpt<11>, k_shard_lpt<12>,
                                            k_shard_lpt<13>, k_shard_lpt<14>, k_shard_lpt<15>, k_shard_lpt<16>};
  const LptKernel lpt = lpts[world - 1];
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(lpt, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  lpt<<<1, 32, smem, st>>>(in, world, *out, cost);
  k_shard_binscan<<<1, kShardThreads, 0, st>>>(in, rank, *out, lmo, lto);
  k_shard_scan_reduce<<<nblk, 1024, 0, st>>>(in, n, rank, *out, part);
  k_shard_scan_parts<<<1, 1024, 0, st>>>(part, nblk, out->status);
  k_shard_scan_apply<<<nblk, 1024, 0, st>>>(in, n, rank, *out, part, lmo, lto);
  k_shard_tail<<<int(std::min<int64_t>((n + 256) / 256, 1024)), 256, 0, st>>>(n, *out);
  VLASIM_LAUNCH_CHECK();
  if (flags & VLASIM_SYNC_CHECK) {
    int32_t h[2];
    VLASIM_CUDA_TRY(cudaMemcpyAsync(h, out->status, sizeof(h), cudaMemcpyDeviceToHost, st));
    VLASIM_CUDA_TRY(cudaStreamSynchronize(st));
    if (h[0]) return set_error(h[0], "shard_lpt: %d bins exceed the device LPT limit of %d", h[1], kMaxShardBins);
  }
  return VLASIM_OK;
}
