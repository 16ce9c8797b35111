// pad.cu — π0.5 dynamic padding on the GPU: the step before
// packing in the paper's π0.5 pipeline, and the fixed-length baseline it is compared against.
//
//   vlasim_dynamic_pad_cuda   pad_to = max(lengths) of the batch (dynamic_pad_length),
//                             cu_seqlens of the valid tokens (exclusive scan of the lengths) and
//                             seg_src[i] = i·pad_to, so the varlen attention kernels run directly on
//                             the padded [n, pad_to, ...] storage: each sample's valid rows are one
//                             segment (its pad keys are never visible, no pad query is computed)
//   vlasim_pad_rows_cuda      sample-major rows → padded [n, pad_to, row] with zero fill
//   vlasim_unpad_rows_cuda    the inverse (valid rows only)
// The copies are HBM-bound: one CTA per sample, 16-byte vectors, 4 in flight per thread.
#include <climits>

#include "common.hpp"
#include "scan.cuh"

namespace {

using vlasim_dev::block_exclusive_scan;

// One CTA of 1024 threads: validation, max, exclusive scan (chunked with a carry), seg_src.
__global__ void __launch_bounds__(1024) k_dynamic_pad(const int32_t* __restrict__ len, int64_t n,
                                                      int32_t* __restrict__ pad_to, int32_t* __restrict__ cu,
                                                      int32_t* __restrict__ seg_src, int32_t* __restrict__ status) {
  __shared__ int64_t scratch[33];
  __shared__ int s_max, s_bad;
  if (threadIdx.x == 0) {
    s_max = 0;
    s_bad = INT_MAX;
  }
  __syncthreads();
  int mx = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int L = len[i];
    if (L < 1) atomicMin(&s_bad, int(i));
    mx = max(mx, L);
  }
  atomicMax(&s_max, mx);
  __syncthreads();
  const int P = s_max;
  if (s_bad != INT_MAX) {
    if (threadIdx.x == 0) {
      status[0] = VLASIM_ECONFIG;
      status[1] = s_bad;
      *pad_to = 0;
    }
    return;
  }
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < n; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < n ? len[i] : 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan<int64_t>(v, scratch, &tot);
    if (i < n) {
      cu[i] = int32_t(carry + ex);
      seg_src[i] = int32_t(i * P);
    }
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cu[n] = int32_t(carry);
    *pad_to = P;
    status[0] = (carry > INT_MAX || int64_t(n) * P > INT_MAX) ? VLASIM_ECONFIG : 0;
    status[1] = status[0] ? -3 : 0;
  }
}

// kPad: src sample-major (sample i at rows [off[i], off[i] + len[i])) → dst [n, pad_to] rows,
// zero-filled; !kPad: the inverse for the valid rows.
template <bool kPad>
__global__ void __launch_bounds__(256) k_pad_rows(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                  int64_t row_vecs, const int32_t* __restrict__ len,
                                                  const int32_t* __restrict__ off, const int32_t* __restrict__ pad_to) {
  const int64_t i = blockIdx.x;
  const int64_t L = len[i], P = *pad_to;
  const int64_t nvalid = L * row_vecs, ntot = kPad ? P * row_vecs : nvalid;
  const uint4* s = src + (kPad ? int64_t(off[i]) : i * P) * row_vecs;
  uint4* d = dst + (kPad ? i * P : int64_t(off[i])) * row_vecs;
  const int64_t stride = 4 * blockDim.x;
  int64_t j = threadIdx.x;
  for (; j + 3 * blockDim.x < nvalid; j += stride) {
    const uint4 v0 = __ldcs(s + j), v1 = __ldcs(s + j + blockDim.x), v2 = __ldcs(s + j + 2 * blockDim.x),
                v3 = __ldcs(s + j + 3 * blockDim.x);
    __stcs(d + j, v0);
    __stcs(d + j + blockDim.x, v1);
    __stcs(d + j + 2 * blockDim.x, v2);
    __stcs(d + j + 3 * blockDim.x, v3);
  }
  for (; j < nvalid; j += blockDim.x) __stcs(d + j, __ldcs(s + j));
  if (kPad)
    for (int64_t z = nvalid + threadIdx.x; z < ntot; z += blockDim.x) __stcs(d + z, make_uint4(0, 0, 0, 0));
}

int check_rows(const void* a, const void* b, int64_t row_bytes) {
  using vlasim_host::set_error;
  if (row_bytes <= 0 || row_bytes % 16) return set_error(VLASIM_ECONFIG, "row_bytes must be a positive multiple of 16");
  if (!a || !b || ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15))
    return set_error(VLASIM_ECONFIG, "pad/unpad buffers must be non-null and 16-byte aligned");
  return VLASIM_OK;
}

}  // namespace

extern "C" int vlasim_dynamic_pad_cuda(const int32_t* d_len, int64_t n, int32_t* d_pad_to, int32_t* d_cu_seqlens,
                                       int32_t* d_seg_src, int32_t* d_status, uint32_t flags, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (n < 1) return set_error(VLASIM_ECONFIG, "dynamic_pad_length: empty batch");
  if (n >= INT_MAX) return set_error(VLASIM_ECONFIG, "dynamic_pad: n exceeds int32");
  if (!d_len || !d_pad_to || !d_cu_seqlens || !d_seg_src || !d_status)
    return set_error(VLASIM_ECONFIG, "dynamic_pad: null buffer");
  cudaStream_t st = as_stream(stream);
  k_dynamic_pad<<<1, 1024, 0, st>>>(d_len, n, d_pad_to, d_cu_seqlens, d_seg_src, d_status);
  VLASIM_LAUNCH_CHECK();
  if (!(flags & VLASIM_SYNC_CHECK)) return VLASIM_OK;
  int32_t h[2];
  VLASIM_CUDA_TRY(cudaMemcpyAsync(h, d_status, sizeof(h), cudaMemcpyDeviceToHost, st));
  VLASIM_CUDA_TRY(cudaStreamSynchronize(st));
  if (h[0] == 0) return VLASIM_OK;
  if (h[1] == -3) return set_error(VLASIM_ECONFIG, "dynamic_pad: padded batch exceeds int32 rows");
  return set_error(VLASIM_ECONFIG, "dynamic_pad: empty sample: id %d (length must be >= 1)", h[1]);
}

extern "C" int vlasim_pad_rows_cuda(const void* d_src, void* d_padded, int64_t row_bytes, const int32_t* d_len,
                                    const int32_t* d_src_off, const int32_t* d_pad_to, int64_t n,
                                    vlasim_stream_t stream) {
  if (int rc = check_rows(d_src, d_padded, row_bytes)) return rc;
  if (n < 1) return VLASIM_OK;
  k_pad_rows<true><<<n, 256, 0, vlasim_host::as_stream(stream)>>>(
      static_cast<const uint4*>(d_src), static_cast<uint4*>(d_padded), row_bytes / 16, d_len, d_src_off, d_pad_to);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

extern "C" int vlasim_unpad_rows_cuda(const void* d_padded, void* d_dst, int64_t row_bytes, const int32_t* d_len,
                                      const int32_t* d_src_off, const int32_t* d_pad_to, int64_t n,
                                      vlasim_stream_t stream) {
  if (int rc = check_rows(d_padded, d_dst, row_bytes)) return rc;
  if (n < 1) return VLASIM_OK;
  k_pad_rows<false><<<n, 256, 0, vlasim_host::as_stream(stream)>>>(
      static_cast<const uint4*>(d_padded), static_cast<uint4*>(d_dst), row_bytes / 16, d_len, d_src_off, d_pad_to);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}
