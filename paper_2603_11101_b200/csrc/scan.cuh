// scan.cuh — warp / block prefix sums used by the packer (hand-written; no CUB).
#pragma once
#include <cstdint>

namespace vlasim_dev {

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_reduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan. `scratch` must hold >= 33 T.  Returns the exclusive prefix;
// *total receives the block sum.  All threads of the block must call it.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* scratch, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < nwarps) ? scratch[lane] : T(0);
    T winc = warp_inclusive_scan(w);
    scratch[lane] = winc - w;
    if (lane == 31) scratch[32] = winc;
  }
  __syncthreads();
  T res = scratch[warp] + inc - v;
  *total = scratch[32];
  __syncthreads();
  return res;
}

}  // namespace vlasim_dev
