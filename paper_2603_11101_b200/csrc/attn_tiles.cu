// attn_tiles.cu — segment-aligned 128-row tiles of the packed stream, ordered by cost.
//
// Every attention kernel walks work items (tile, head).  A tile is a run of ≤ 128 consecutive
// rows of ONE segment: segment [s, e) of the packed stream (cu_seqlens) is cut
// into ⌈(e−s)/128⌉ tiles [s + 128k, min(s + 128(k+1), e)).  Because a tile never straddles a
// segment boundary, its key range is that one segment's visible keys — no block of another
// segment is loaded or multiplied (for U[16,512] packs the computed pairs drop by ≈ 10 % against
// tiles on the global 128-row grid).  The rows of the 128-row TMA box beyond the
// tile's end belong to the next segment; the kernels mask them like any invisible pair and never
// store them.
//
// Order: tiles are sorted by their segment's tile count, descending (stable: a segment's tiles
// stay adjacent, and equal-cost segments keep stream order, so concurrently running items share
// K/V in L2).  With the persistent kernels' boustrophedon schedule (sched_item) the per-CTA work
// sums stay balanced — the heaviest items run first and the tail is made of the lightest.
//
// Each tile also carries its segment's source offset (vlasim_attn_args.seg_src): data row of
// packed row t = t + delta, one constant for the tile's rows and for all its keys (a segment's
// keys are its own rows), so the gather into the packed stream is a TMA coordinate shift.
//
// One CTA of 1024 threads: pass 1 histograms the tile counts per cost bucket, pass 2 places each
// segment's tiles at (bucket offset + weighted rank among the earlier segments of its bucket).
#include <cstdint>

#include "common.hpp"

namespace {

constexpr int kTilesThreads = 1024;
constexpr int kBuckets = 128;  // cost bucket = min(tiles of the segment, 127)

__global__ void __launch_bounds__(kTilesThreads) k_build_tiles(const int32_t* __restrict__ cu,
                                                               const int32_t* __restrict__ seg_src, int nseq,
                                                               int4* __restrict__ tiles, int* __restrict__ ntiles) {
  __shared__ int boff[kBuckets];          // first position of each bucket's next tile
  __shared__ int wsum[32][kBuckets];      // per-warp, per-bucket tile counts → exclusive scan over warps
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < kBuckets; b += kTilesThreads) boff[b] = 0;
  __syncthreads();
  for (int s = tid; s < nseq; s += kTilesThreads) {
    const int c = (__ldg(cu + s + 1) - __ldg(cu + s) + 127) >> 7;
    if (c > 0) atomicAdd(&boff[min(c, kBuckets - 1)], c);
  }
  __syncthreads();
  if (tid == 0) {  // descending cost: bucket kBuckets-1 first
    int run = 0;
    for (int b = kBuckets - 1; b >= 0; --b) {
      const int n = boff[b];
      boff[b] = run;
      run += n;
    }
    *ntiles = run;
  }
  __syncthreads();
  for (int base = 0; base < nseq; base += kTilesThreads) {
    const int s = base + tid;
    const int lo = s < nseq ? __ldg(cu + s) : 0, hi = s < nseq ? __ldg(cu + s + 1) : 0;
    const int c = (hi - lo + 127) >> 7;
    const int b = min(c, kBuckets - 1);
    for (int x = tid; x < 32 * kBuckets; x += kTilesThreads) (&wsum[0][0])[x] = 0;
    __syncthreads();
    int acc = 0;  // tiles of the earlier lanes of this warp in the same bucket
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const int cj = __shfl_sync(0xffffffffu, c, j), bj = __shfl_sync(0xffffffffu, b, j);
      acc += (j < lane && bj == b) ? cj : 0;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    if (31 - __clz(peers) == lane) wsum[warp][b] = acc + c;  // the bucket's last lane in this warp
    __syncthreads();
    int total = 0;
    if (tid < kBuckets) {
      for (int w = 0; w < 32; ++w) {
        const int t = wsum[w][tid];
        wsum[w][tid] = total;
        total += t;
      }
    }
    __syncthreads();
    if (c > 0) {
      const int pos = boff[b] + wsum[warp][b] + acc;
      const int dl = seg_src ? __ldg(seg_src + s) - lo : 0;
      for (int k = 0; k < c; ++k) tiles[pos + k] = make_int4(lo + 128 * k, min(lo + 128 * (k + 1), hi), dl, 0);
    }
    __syncthreads();
    if (tid < kBuckets) boff[tid] += total;
  }
}

}  // namespace

namespace vlasim_host {

// Upper bound of the tile count: Σ⌈l/128⌉ ≤ ⌊T/128⌋ + nseq.
size_t tiles_bytes(int64_t T, int nseq) { return (size_t(T / 128) + size_t(nseq) + 1) * sizeof(int4) + 16; }

// tiles: {q0, qe, delta, 0} per tile, followed by the tile count (int) in the last 16 bytes.
int launch_build_tiles(const int32_t* cu, const int32_t* seg_src, int nseq, int64_t T, void* buf, cudaStream_t st,
                       int4** tiles, int** ntiles) {
  *tiles = static_cast<int4*>(buf);
  *ntiles = reinterpret_cast<int*>(static_cast<uint8_t*>(buf) + tiles_bytes(T, nseq) - 16);
  k_build_tiles<<<1, kTilesThreads, 0, st>>>(cu, seg_src, nseq, *tiles, *ntiles);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

}  // namespace vlasim_host
