// attn_common.cuh — shared pieces of the varlen attention kernels: segment lookup and
// the visible-key interval of a query row under the three mask modes.
//
// Mask semantics (SPEC.md:496, 514, 520 give the bidirectional block-
// diagonal case): for query t in segment [s, e) with prefix P,
//   visible keys = [s, min(e, max(s + P, t + 1)))
//   bidirectional: P = e - s ; causal: P = 0 ; prefix: P = prefix_len[seg].
#pragma once
#include <cstdint>

namespace vlasim_dev {

struct RowSpan {
  int lo, hi;  // visible keys [lo, hi) in packed-stream coordinates; lo == hi → none
  int seg;
};

// Largest s with cu[s] <= t (cu strictly increasing, cu[0] = 0, cu[nseq] <= T: rows of the tensors
// past cu[nseq] — e.g. the pad rows of a dynamically padded batch read through seg_src — belong to
// no segment).
__device__ __forceinline__ int find_segment(const int32_t* __restrict__ cu, int nseq, int t) {
  int lo = 0, hi = nseq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(cu + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ RowSpan row_span(const int32_t* __restrict__ cu, const int32_t* __restrict__ prefix,
                                            int nseq, int mask_mode, int t, int T) {
  RowSpan r{0, 0, -1};
  if (t < 0 || t >= T || t >= __ldg(cu + nseq)) return r;  // rows past the last segment: none
  const int s = find_segment(cu, nseq, t);
  const int b = __ldg(cu + s), e = __ldg(cu + s + 1);
  int P = e - b;
  if (mask_mode == 1) P = 0;
  else if (mask_mode == 2) P = min(e - b, max(0, __ldg(prefix + s)));
  r.lo = b;
  r.hi = min(e, max(b + P, t + 1));
  r.seg = s;
  return r;
}

// Queries that can see key j of segment [b, e) with prefix P: [j < b + P ? b : j, e).
__device__ __forceinline__ RowSpan key_span(const int32_t* __restrict__ cu, const int32_t* __restrict__ prefix,
                                            int nseq, int mask_mode, int j, int T) {
  RowSpan r{0, 0, -1};
  if (j < 0 || j >= T || j >= __ldg(cu + nseq)) return r;
  const int s = find_segment(cu, nseq, j);
  const int b = __ldg(cu + s), e = __ldg(cu + s + 1);
  int P = e - b;
  if (mask_mode == 1) P = 0;
  else if (mask_mode == 2) P = min(e - b, max(0, __ldg(prefix + s)));
  r.lo = (j < b + P) ? b : j;
  r.hi = e;
  r.seg = s;
  return r;
}

// Persistent static schedule over work items sorted by decreasing cost (attn_tiles.cu): round m
// of CTA b takes item m·G + b on even rounds and m·G + (G−1−b) on odd rounds (boustrophedon), so
// no CTA takes the heaviest item of every round.
__device__ __forceinline__ int sched_item(int m) {
  const int G = gridDim.x, b = blockIdx.x;
  return m * G + ((m & 1) ? G - 1 - b : b);
}

}  // namespace vlasim_dev
