// quant.cu — the general E4M3 quantizer: PerTensor, PerChannel(axis) and
// PerBlock(128, 128 over the last two dims) granularity over an fp32 or bf16 tensor of any shape,
// dequantize, and quant_error with a per-group breakdown.  The per-head block quantiser of the FP8
// attention path (fp8.cu) is the PerBlock case specialised to [T, heads, d] bf16.
//
//   scale_g = RN_fp32(amax_g / 448)  (1 for an all-zero group)
//   code    = RNE onto E4M3 of the REAL quotient |x|·448 / amax_g, saturating to ±448
//                                                                         SPEC.md:583, 618-619
//   non-finite input → VLASIM_ECONFIG naming the flat index
//
// Exactness of the codes (the oracle is an exhaustive nearest-value search):
// X64 = (|x|·448) / amax in fp64 — the numerator is exact (≤ 27 significant bits), the division
// correctly rounded.  A midpoint M between two E4M3 values has ≤ 5 significant bits, so M·amax has
// ≤ 29 and a quotient X ≠ M sits at relative distance > 2^-30 from M, while X64 is within 2^-53 of X:
// the round-half-even decision on X64 (rint on the binade grid, exact scaling by a power of two) is
// the decision on X.  fp64 costs ~10 DFMA per element: far below HBM time on B200.
//
// Passes (all stream-ordered, one HBM read each):
//   k_amax    per-group absolute maximum (atomicMax on the fp32 bit pattern — order-independent,
//             hence deterministic); non-finite detection
//   k_scales  scale_g from amax_g
//   k_codes   the codes (8 consecutive elements per thread, one 8-B store when aligned)
// quant_error reduces per group in a FIXED order (one CTA per group, or fixed 64 K-element chunks
// for PerTensor + an ordered second pass): bit-identical metrics run to run.
#include <cuda_bf16.h>

#include <algorithm>
#include <climits>

#include "common.hpp"

namespace {

constexpr int kElems = 8;  // consecutive elements per thread in the element-wise passes

// Flat index → group, advanced incrementally (no 64-bit division per element).
struct GroupMap {
  int kind;                   // VLASIM_GRAN_*
  int64_t n;                  // elements
  int64_t ch, inner;          // PerChannel: [outer, ch, inner]
  int64_t rows, cols;         // PerBlock:   [batch, rows, cols]
  int64_t nbr, nbc;           //             ⌈rows/128⌉, ⌈cols/128⌉
  int64_t groups;
};

struct GroupCursor {
  int64_t a, b, c;  // PerChannel: (outer, channel, inner); PerBlock: (batch, row, col)
  __device__ void seek(const GroupMap& m, int64_t i) {
    if (m.kind == VLASIM_GRAN_CHANNEL) {
      c = i % m.inner;
      const int64_t t = i / m.inner;
      b = t % m.ch;
      a = t / m.ch;
    } else if (m.kind == VLASIM_GRAN_BLOCK) {
      c = i % m.cols;
      const int64_t t = i / m.cols;
      b = t % m.rows;
      a = t / m.rows;
    } else {
      a = b = c = 0;
    }
  }
  __device__ int64_t group(const GroupMap& m) const {
    if (m.kind == VLASIM_GRAN_CHANNEL) return b;
    if (m.kind == VLASIM_GRAN_BLOCK) return (a * m.nbr + (b >> 7)) * m.nbc + (c >> 7);
    return 0;
  }
  __device__ void next(const GroupMap& m) {
    if (m.kind == VLASIM_GRAN_CHANNEL) {
      if (++c == m.inner) {
        c = 0;
        if (++b == m.ch) b = 0, ++a;
      }
    } else if (m.kind == VLASIM_GRAN_BLOCK) {
      if (++c == m.cols) {
        c = 0;
        if (++b == m.rows) b = 0, ++a;
      }
    }
  }
};

template <typename T>
__device__ __forceinline__ float load_f(const T* p, int64_t i);
template <>
__device__ __forceinline__ float load_f<float>(const float* p, int64_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ float load_f<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

// RNE onto E4M3 (codes 0..0x7E) of X >= 0, saturating at 448.  Binade E = ⌊log2 X⌋ clamped to
// −6 (subnormals share the 2^-9 spacing of the first normal binade); spacing u = 2^(E−3);
// N = rint(X / u) ∈ [0, 16] (exact scaling, ties to even); code = (E + 6)·8 + N, so N = 16 carries
// into the next binade and an even N is an even code (ties to the even mantissa).
__device__ __forceinline__ uint32_t e4m3_rne_f64(double X) {
  if (X >= 448.0) return 0x7E;
  if (X <= 0.0009765625) return 0;  // ≤ 2^-10: below (or tied with) half the smallest subnormal
  int E = int((__double2hiint(X) >> 20) & 0x7FF) - 1023;
  E = E < -6 ? -6 : E;
  const double N = rint(X * __hiloint2double((1023 - (E - 3)) << 20, 0));  // X · 2^(3−E), exact
  return uint32_t((E + 6) * 8 + int(N));
}

__device__ __forceinline__ float e4m3_value(uint32_t c) {
  const int e = (c >> 3) & 0xF, m = c & 7;
  float v;
  if (e == 0) v = ldexpf(float(m) / 8.f, -6);
  else if (e == 15 && m == 7) v = __int_as_float(0x7fc00000);
  else v = ldexpf(1.f + float(m) / 8.f, e - 7);
  return (c & 0x80) ? -v : v;
}

__device__ __forceinline__ void report_bad(int32_t* status, int64_t i) {
  if (!status) return;
  atomicMin(status + 1, int32_t(i < INT_MAX ? i : INT_MAX));
  atomicExch(status, VLASIM_ECONFIG);
}

// ---- pass 1: per-group amax.  Runs of one group are folded in registers and flushed with one
// atomicMax; PerChannel with inner == 1 (the channel is the fastest dim: the group changes every
// element) folds into a shared-memory copy of the channel maxima first.
template <typename T>
__global__ void __launch_bounds__(256) k_amax(const T* __restrict__ x, GroupMap m, uint32_t* __restrict__ amax,
                                              int32_t* __restrict__ status, int smem_ch) {
  extern __shared__ uint32_t s_amax[];
  for (int i = threadIdx.x; i < smem_ch; i += blockDim.x) s_amax[i] = 0;
  if (smem_ch) __syncthreads();
  uint32_t* dst = smem_ch ? s_amax : amax;
  const int64_t nchunks = (m.n + kElems - 1) / kElems;
  for (int64_t ck = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ck < nchunks;
       ck += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i0 = ck * kElems;
    GroupCursor cur;
    cur.seek(m, i0);
    int64_t g = cur.group(m);
    float run = 0.f;
#pragma unroll
    for (int j = 0; j < kElems; ++j) {
      const int64_t i = i0 + j;
      if (i >= m.n) break;
      const int64_t gj = cur.group(m);
      if (gj != g) {
        atomicMax(dst + g, __float_as_uint(run));
        g = gj;
        run = 0.f;
      }
      const float v = load_f(x, i);
      if (!isfinite(v)) report_bad(status, i);
      run = fmaxf(run, fabsf(v));
      cur.next(m);
    }
    atomicMax(dst + g, __float_as_uint(run));
  }
  if (smem_ch) {
    __syncthreads();
    for (int i = threadIdx.x; i < smem_ch; i += blockDim.x)
      if (s_amax[i]) atomicMax(amax + i, s_amax[i]);
  }
}

__global__ void k_scales(const uint32_t* __restrict__ amax, int64_t groups, float* __restrict__ scales) {
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (g < groups) {
    const float a = __uint_as_float(amax[g]);
    scales[g] = a == 0.f ? 1.f : __fdiv_rn(a, 448.f);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_codes(const T* __restrict__ x, GroupMap m, const uint32_t* __restrict__ amax,
                                               uint8_t* __restrict__ codes, const int32_t* __restrict__ status) {
  if (status && status[0] != 0) return;  // non-finite input: no codes written
  const int64_t nchunks = (m.n + kElems - 1) / kElems;
  for (int64_t ck = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ck < nchunks;
       ck += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i0 = ck * kElems;
    GroupCursor cur;
    cur.seek(m, i0);
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < kElems; ++j) {
      const int64_t i = i0 + j;
      if (i >= m.n) break;
      const float v = load_f(x, i);
      const float a = __uint_as_float(__ldg(amax + cur.group(m)));
      // all-zero group: scale 1, the code of ±0; otherwise the exact RNE code of |x|·448/amax
      const uint32_t mag = a == 0.f ? 0u : e4m3_rne_f64(__ddiv_rn(double(fabsf(v)) * 448.0, double(a)));
      w[j >> 2] |= (mag | (signbit(v) ? 0x80u : 0u)) << (8 * (j & 3));
      cur.next(m);
    }
    if (i0 + kElems <= m.n) {
      *reinterpret_cast<uint2*>(codes + i0) = make_uint2(w[0], w[1]);
    } else {
      for (int j = 0; i0 + j < m.n; ++j) codes[i0 + j] = uint8_t(w[j >> 2] >> (8 * (j & 3)));
    }
  }
}

__global__ void __launch_bounds__(256) k_dequant(const uint8_t* __restrict__ codes, const float* __restrict__ scales,
                                                 GroupMap m, float* __restrict__ out) {
  const int64_t nchunks = (m.n + kElems - 1) / kElems;
  for (int64_t ck = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ck < nchunks;
       ck += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i0 = ck * kElems;
    GroupCursor cur;
    cur.seek(m, i0);
#pragma unroll
    for (int j = 0; j < kElems; ++j) {
      const int64_t i = i0 + j;
      if (i >= m.n) break;
      out[i] = __fmul_rn(e4m3_value(codes[i]), __ldg(scales + cur.group(m)));
      cur.next(m);
    }
  }
}

// ---- quant_error: per element deq = fp32(value(code)·scale), diff = fp32(deq − x),
// squared in fp64; relative error fp32(|diff| / |x|) over elements in E4M3's normal range
// (|fp32(x / scale)| >= 2^-6).  Fixed-order reductions.
struct ErrAcc {
  float mx;
  double sse;
};

template <typename T>
__device__ __forceinline__ void err_elem(const T* x, const uint8_t* codes, float scale, int64_t i, ErrAcc& acc) {
  const float xv = load_f(x, i);
  const float diff = __fsub_rn(__fmul_rn(e4m3_value(codes[i]), scale), xv);
  acc.sse += double(diff) * double(diff);
  if (fabsf(__fdiv_rn(xv, scale)) >= 0.015625f) acc.mx = fmaxf(acc.mx, __fdiv_rn(fabsf(diff), fabsf(xv)));
}

// block-wide reduction in a fixed order (shuffle tree, then warps 0..7 in order)
__device__ ErrAcc block_reduce(ErrAcc a) {
  __shared__ float smx[8];
  __shared__ double ssse[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a.mx = fmaxf(a.mx, __shfl_xor_sync(0xffffffffu, a.mx, o));
    a.sse += __shfl_xor_sync(0xffffffffu, a.sse, o);
  }
  if ((threadIdx.x & 31) == 0) {
    smx[threadIdx.x >> 5] = a.mx;
    ssse[threadIdx.x >> 5] = a.sse;
  }
  __syncthreads();
  ErrAcc r{0.f, 0.0};
  for (int w = 0; w < int(blockDim.x >> 5); ++w) {
    r.mx = fmaxf(r.mx, smx[w]);
    r.sse += ssse[w];
  }
  __syncthreads();
  return r;
}

constexpr int64_t kErrChunk = 1 << 16;  // PerTensor: elements per first-pass CTA (fixed → deterministic)

// One CTA per group (PerChannel, PerBlock) or per fixed chunk (PerTensor, partial results).
template <typename T>
__global__ void __launch_bounds__(256) k_quant_err(const T* __restrict__ x, const uint8_t* __restrict__ codes,
                                                   const float* __restrict__ scales, GroupMap m,
                                                   float* __restrict__ gmax, double* __restrict__ gsse,
                                                   int64_t* __restrict__ gcnt) {
  const int64_t g = blockIdx.x;
  ErrAcc acc{0.f, 0.0};
  int64_t count = 0;
  if (m.kind == VLASIM_GRAN_TENSOR) {
    const float s = scales[0];
    const int64_t i0 = g * kErrChunk, i1 = m.n < i0 + kErrChunk ? m.n : i0 + kErrChunk;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) err_elem(x, codes, s, i, acc);
    count = i1 - i0;
  } else if (m.kind == VLASIM_GRAN_CHANNEL) {
    const float s = scales[g];
    const int64_t outer = m.n / (m.ch * m.inner), per = outer * m.inner;
    for (int64_t e = threadIdx.x; e < per; e += blockDim.x) {
      const int64_t o = e / m.inner, in = e - o * m.inner;
      err_elem(x, codes, s, (o * m.ch + g) * m.inner + in, acc);
    }
    count = per;
  } else {
    const float s = scales[g];
    const int64_t bc = g % m.nbc, br = (g / m.nbc) % m.nbr, b = g / (m.nbc * m.nbr);
    const int64_t r0 = br * 128, c0 = bc * 128;
    const int nr = int(m.rows - r0 < 128 ? m.rows - r0 : 128), nc = int(m.cols - c0 < 128 ? m.cols - c0 : 128);
    for (int e = threadIdx.x; e < nr * 128; e += blockDim.x) {
      const int r = e >> 7, c = e & 127;
      if (c < nc) err_elem(x, codes, s, (b * m.rows + r0 + r) * m.cols + c0 + c, acc);
    }
    count = int64_t(nr) * nc;
  }
  const ErrAcc r = block_reduce(acc);
  if (threadIdx.x == 0) {
    gmax[g] = r.mx;
    gsse[g] = r.sse;
    gcnt[g] = count;
  }
}

// PerTensor second pass: the chunk partials in index order (one thread — there are n / 65536).
__global__ void k_quant_err_tensor(int64_t nparts, float* gmax, double* gsse, int64_t* gcnt) {
  float mx = 0.f;
  double sse = 0.0;
  int64_t cnt = 0;
  for (int64_t p = 0; p < nparts; ++p) {
    mx = fmaxf(mx, gmax[p]);
    sse += gsse[p];
    cnt += gcnt[p];
  }
  gmax[0] = mx;
  gsse[0] = sse;
  gcnt[0] = cnt;
}

int make_map(const int64_t* shape, int32_t ndim, int32_t gran, int32_t axis, GroupMap* m) {
  using vlasim_host::set_error;
  if (!shape || ndim < 1 || ndim > 8) return set_error(VLASIM_ECONFIG, "quantize: 1 <= ndim <= 8 required");
  int64_t n = 1;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 1) return set_error(VLASIM_ECONFIG, "quantize: dimension %d is %lld (must be >= 1)", i,
                                       (long long)shape[i]);
    n *= shape[i];
  }
  *m = GroupMap{};
  m->kind = gran;
  m->n = n;
  if (gran == VLASIM_GRAN_TENSOR) {
    m->groups = 1;
  } else if (gran == VLASIM_GRAN_CHANNEL) {
    if (axis < 0) axis += ndim;
    if (axis < 0 || axis >= ndim) return set_error(VLASIM_ECONFIG, "quantize: channel axis out of range");
    m->ch = shape[axis];
    m->inner = 1;
    for (int i = axis + 1; i < ndim; ++i) m->inner *= shape[i];
    m->groups = m->ch;
  } else if (gran == VLASIM_GRAN_BLOCK) {
    if (ndim < 2) return set_error(VLASIM_ECONFIG, "quantize: PerBlock needs a tensor of >= 2 dims");  // SPEC pre
    m->rows = shape[ndim - 2];
    m->cols = shape[ndim - 1];
    m->nbr = (m->rows + 127) / 128;
    m->nbc = (m->cols + 127) / 128;
    m->groups = (n / (m->rows * m->cols)) * m->nbr * m->nbc;
  } else {
    return set_error(VLASIM_ECONFIG, "quantize: unknown granularity %d", gran);
  }
  return VLASIM_OK;
}

int grid_for(int64_t n) {
  const int64_t chunks = (n + kElems - 1) / kElems;
  const int64_t want = (chunks + 255) / 256;
  const int64_t cap = int64_t(vlasim_host::num_sms()) * 8;
  return int(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" int64_t vlasim_fp8_groups(const int64_t* shape, int32_t ndim, int32_t granularity, int32_t axis) {
  GroupMap m;
  if (make_map(shape, ndim, granularity, axis, &m)) return -1;
  return m.groups;
}

extern "C" size_t vlasim_fp8_quantize_workspace_size(const int64_t* shape, int32_t ndim, int32_t granularity,
                                                     int32_t axis) {
  GroupMap m;
  if (make_map(shape, ndim, granularity, axis, &m)) return 0;
  return size_t(m.groups) * 4;
}

extern "C" int vlasim_fp8_quantize_cuda(const void* d_x, int32_t dtype, const int64_t* shape, int32_t ndim,
                                        int32_t granularity, int32_t axis, uint8_t* d_codes, float* d_scales,
                                        int32_t* d_status, void* d_workspace, size_t workspace_bytes, uint32_t flags,
                                        vlasim_stream_t stream) {
  using namespace vlasim_host;
  GroupMap m;
  if (int rc = make_map(shape, ndim, granularity, axis, &m)) return rc;
  if (dtype != VLASIM_DTYPE_F32 && dtype != VLASIM_DTYPE_BF16)
    return set_error(VLASIM_ECONFIG, "quantize: input dtype must be fp32 or bf16");
  if (!d_x || !d_codes || !d_scales) return set_error(VLASIM_ECONFIG, "quantize: null buffer");
  if ((flags & VLASIM_SYNC_CHECK) && !d_status) return set_error(VLASIM_ECONFIG, "quantize: sync check needs d_status");
  if (!d_workspace || workspace_bytes < size_t(m.groups) * 4)
    return set_error(VLASIM_ECONFIG, "quantize: workspace too small (%zu < %zu)", workspace_bytes,
                     size_t(m.groups) * 4);
  cudaStream_t st = as_stream(stream);
  uint32_t* amax = static_cast<uint32_t*>(d_workspace);
  VLASIM_CUDA_TRY(cudaMemsetAsync(amax, 0, size_t(m.groups) * 4, st));
  if (d_status) {
    const int32_t init[2] = {0, INT_MAX};
    VLASIM_CUDA_TRY(cudaMemcpyAsync(d_status, init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  const int smem_ch = (m.kind == VLASIM_GRAN_CHANNEL && m.inner == 1 && m.ch <= 12288) ? int(m.ch) : 0;
  const int grid = grid_for(m.n);
  const int grid1 = smem_ch ? std::min(grid, num_sms()) : grid;
  if (smem_ch * 4 > 48 * 1024) {
    VLASIM_CUDA_TRY(cudaFuncSetAttribute(k_amax<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ch * 4));
    VLASIM_CUDA_TRY(
        cudaFuncSetAttribute(k_amax<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ch * 4));
  }
  if (dtype == VLASIM_DTYPE_F32) {
    const float* x = static_cast<const float*>(d_x);
    k_amax<float><<<grid1, 256, smem_ch * 4, st>>>(x, m, amax, d_status, smem_ch);
    k_scales<<<int((m.groups + 255) / 256), 256, 0, st>>>(amax, m.groups, d_scales);
    k_codes<float><<<grid, 256, 0, st>>>(x, m, amax, d_codes, d_status);
  } else {
    const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(d_x);
    k_amax<__nv_bfloat16><<<grid1, 256, smem_ch * 4, st>>>(x, m, amax, d_status, smem_ch);
    k_scales<<<int((m.groups + 255) / 256), 256, 0, st>>>(amax, m.groups, d_scales);
    k_codes<__nv_bfloat16><<<grid, 256, 0, st>>>(x, m, amax, d_codes, d_status);
  }
  VLASIM_LAUNCH_CHECK();
  if (!(flags & VLASIM_SYNC_CHECK)) return VLASIM_OK;
  int32_t h[2];
  VLASIM_CUDA_TRY(cudaMemcpyAsync(h, d_status, sizeof(h), cudaMemcpyDeviceToHost, st));
  VLASIM_CUDA_TRY(cudaStreamSynchronize(st));
  if (h[0] != 0) return set_error(VLASIM_ECONFIG, "quantize: non-finite input at flat index %d", h[1]);
  return VLASIM_OK;
}

extern "C" int vlasim_fp8_dequantize_cuda(const uint8_t* d_codes, const float* d_scales, const int64_t* shape,
                                          int32_t ndim, int32_t granularity, int32_t axis, float* d_out,
                                          vlasim_stream_t stream) {
  using namespace vlasim_host;
  GroupMap m;
  if (int rc = make_map(shape, ndim, granularity, axis, &m)) return rc;
  if (!d_codes || !d_scales || !d_out) return set_error(VLASIM_ECONFIG, "dequantize: null buffer");
  k_dequant<<<grid_for(m.n), 256, 0, as_stream(stream)>>>(d_codes, d_scales, m, d_out);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

extern "C" int64_t vlasim_fp8_error_groups(const int64_t* shape, int32_t ndim, int32_t granularity, int32_t axis) {
  GroupMap m;
  if (make_map(shape, ndim, granularity, axis, &m)) return -1;
  return m.kind == VLASIM_GRAN_TENSOR ? (m.n + kErrChunk - 1) / kErrChunk : m.groups;
}

extern "C" int vlasim_fp8_quant_error_general_cuda(const void* d_x, int32_t dtype, const uint8_t* d_codes,
                                                   const float* d_scales, const int64_t* shape, int32_t ndim,
                                                   int32_t granularity, int32_t axis, float* d_group_maxrel,
                                                   double* d_group_sse, int64_t* d_group_count,
                                                   vlasim_stream_t stream) {
  using namespace vlasim_host;
  GroupMap m;
  if (int rc = make_map(shape, ndim, granularity, axis, &m)) return rc;
  if (dtype != VLASIM_DTYPE_F32 && dtype != VLASIM_DTYPE_BF16)
    return set_error(VLASIM_ECONFIG, "quant_error: input dtype must be fp32 or bf16");
  if (!d_x || !d_codes || !d_scales || !d_group_maxrel || !d_group_sse || !d_group_count)
    return set_error(VLASIM_ECONFIG, "quant_error: null buffer");
  cudaStream_t st = as_stream(stream);
  const int64_t nblk = m.kind == VLASIM_GRAN_TENSOR ? (m.n + kErrChunk - 1) / kErrChunk : m.groups;
  if (nblk > INT_MAX) return set_error(VLASIM_ECONFIG, "quant_error: too many groups");
  if (dtype == VLASIM_DTYPE_F32)
    k_quant_err<float><<<int(nblk), 256, 0, st>>>(static_cast<const float*>(d_x), d_codes, d_scales, m, d_group_maxrel,
                                                  d_group_sse, d_group_count);
  else
    k_quant_err<__nv_bfloat16><<<int(nblk), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(d_x), d_codes, d_scales,
                                                          m, d_group_maxrel, d_group_sse, d_group_count);
  if (m.kind == VLASIM_GRAN_TENSOR) k_quant_err_tensor<<<1, 1, 0, st>>>(nblk, d_group_maxrel, d_group_sse, d_group_count);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}
