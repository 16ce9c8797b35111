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
// One CTA of 1024 threads: a bitonic sort of ≤ 16384 64-bit bin keys in shared memory, the greedy
// assignment by one thread (loads in registers, world ≤ 16), and chunked block scans over bins and
// samples.  Metadata only (a few bytes per sample): latency-bound, a few µs at the bench's sizes.
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

__global__ void __launch_bounds__(kShardThreads) k_shard_plan(ShardIn in, int64_t n, int world, int rank,
                                                              vlasim_shard_out o) {
  extern __shared__ unsigned long long keys[];  // [P] sort keys, P = next pow2 >= bins
  __shared__ int64_t scratch[33];
  const int B = *in.num_bins;
  if (B > kMaxShardBins) {
    if (threadIdx.x == 0) o.status[0] = VLASIM_ECONFIG, o.status[1] = B;
    return;
  }
  if (threadIdx.x == 0) o.status[0] = 0, o.status[1] = 0;
  int P = 1;
  while (P < B) P <<= 1;
  // cost of every bin; key = cost · 2^32 + (2^32 − 1 − b): descending order = (cost desc, b asc)
  for (int b = threadIdx.x; b < P; b += kShardThreads) {
    unsigned long long k = 0;
    if (b < B) {
      long long c = 0;
      for (int m = in.bin_member_off[b]; m < in.bin_member_off[b + 1]; ++m) {
        const long long l = in.len[in.member_ids[m]];
        c += l * l;
      }
      k = (static_cast<unsigned long long>(c) << 32) | (0xFFFFFFFFull - unsigned(b));
    }
    keys[b] = k;
  }
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
  // greedy LPT (one thread; world ≤ 16 loads in registers)
  if (threadIdx.x == 0) {
    long long ld[kMaxWorld];
#pragma unroll
    for (int r = 0; r < kMaxWorld; ++r) ld[r] = r < world ? 0 : LLONG_MAX;
    for (int i = 0; i < B; ++i) {
      const unsigned long long k = keys[i];
      const int b = int(0xFFFFFFFFull - (k & 0xFFFFFFFFull));
      int best = 0;
      long long bl = ld[0];
#pragma unroll
      for (int r = 1; r < kMaxWorld; ++r)
        if (ld[r] < bl) bl = ld[r], best = r;
#pragma unroll
      for (int r = 0; r < kMaxWorld; ++r)
        if (r == best) ld[r] += static_cast<long long>(k >> 32);
      o.bin_rank[b] = best;
    }
#pragma unroll
    for (int r = 0; r < kMaxWorld; ++r)
      if (r < world) o.rank_load[r] = ld[r];
  }
  __syncthreads();
  // this rank's bins in index order: local member / token offsets per bin
  int32_t* lmo = reinterpret_cast<int32_t*>(keys);  // reuse smem: [B] local member offset
  int32_t* lto = lmo + kMaxShardBins;              // [B] local token offset (bins ≤ 16384 → 128 KB)
  const int64_t nseg = block_scan_chunked(
      B, [&](int64_t b) -> int64_t { return o.bin_rank[b] == rank ? in.bin_count[b] : 0; },
      [&](int64_t b, int64_t x) { lmo[b] = int32_t(x); }, scratch);
  const int64_t ntok = block_scan_chunked(
      B, [&](int64_t b) -> int64_t { return o.bin_rank[b] == rank ? in.bin_fill[b] : 0; },
      [&](int64_t b, int64_t x) { lto[b] = int32_t(x); }, scratch);
  // the rank's sample-major layout: local samples in id order
  block_scan_chunked(
      n, [&](int64_t i) -> int64_t { return o.bin_rank[in.bin_of[i]] == rank ? in.len[i] : 0; },
      [&](int64_t i, int64_t x) { o.local_src_off[i] = o.bin_rank[in.bin_of[i]] == rank ? int32_t(x) : -1; },
      scratch);
  for (int64_t i = threadIdx.x; i < n; i += kShardThreads) {
    const int b = in.bin_of[i];
    if (o.bin_rank[b] != rank) continue;
    const int j = lmo[b] + in.slot[i];
    o.local_ids[j] = int32_t(i);
    o.local_cu[j] = lto[b] + in.tok_off[i];
    o.local_seg_src[j] = o.local_src_off[i];
  }
  // segments past the local count: zero length at the end of the stream
  for (int64_t j = nseg + threadIdx.x; j <= n; j += kShardThreads) o.local_cu[j] = int32_t(ntok);
  if (threadIdx.x == 0) {
    *o.local_nseg = int32_t(nseg);
    *o.local_tokens = ntok;
  }
}

}  // namespace

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
  ShardIn in{d_len, plan->bin_of, plan->slot, plan->tok_off, plan->bin_count, plan->bin_fill, plan->bin_member_off,
             plan->member_ids, plan->num_bins};
  cudaStream_t st = as_stream(stream);
  const size_t smem = size_t(kMaxShardBins) * 8;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_shard_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  k_shard_plan<<<1, kShardThreads, smem, st>>>(in, n, world, rank, *out);
  VLASIM_LAUNCH_CHECK();
  if (flags & VLASIM_SYNC_CHECK) {
    int32_t h[2];
    VLASIM_CUDA_TRY(cudaMemcpyAsync(h, out->status, sizeof(h), cudaMemcpyDeviceToHost, st));
    VLASIM_CUDA_TRY(cudaStreamSynchronize(st));
    if (h[0]) return set_error(h[0], "shard_lpt: %d bins exceed the device LPT limit of %d", h[1], kMaxShardBins);
  }
  return VLASIM_OK;
}
