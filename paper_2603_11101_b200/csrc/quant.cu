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
// Exactness of the codes (the oracle is an exhaustive nearest-value search): the fp32
// quotient q of |x|·448 by amax (one Markstein correction) is within ~2 ulps of the real X, so
// cvt.rn(q) is the RNE code of X unless q lies within 64 ulps of a midpoint between two E4M3 values
// (below 2^-6: within 2^-22 of an odd multiple of 2^-10); only those (rare) elements are re-decided
// by exact fp64 comparisons (e4m3_fix: |x|·448 has ≤ 27 significant bits, midpoint·amax ≤ 29).
// Groups whose maximum lies outside 2^±100 take the fp64 decision for every element (group_rcp).
// A per-element fp64 division (the first version) made the code pass FP64-bound on B200.
//
// Kernels by granularity (every warp load one contiguous span):
//   PerBlock, PerChannel with ≤ 16 K elements per group   k_group_fused: persistent, a group per
//             CTA iteration held in registers — amax, scale and codes from ONE read of x
//   PerTensor                         k_tensor_amax → k_scales → k_tensor_codes (two reads: the scale
//                                     needs the global maximum first)
//   PerChannel over the last axis     k_col_amax → k_scales → k_col_codes (column-owned threads)
//   other PerChannel                  generic k_amax → k_scales → k_codes (group cursor per element)
// Maxima are combined with atomicMax on the fp32 bit pattern (order-independent: deterministic).
// quant_error reduces per group in a FIXED order (one CTA per group, or fixed 64 K-element chunks
// for PerTensor + an ordered second pass): bit-identical metrics run to run.
#include <cuda_bf16.h>

#include <algorithm>
#include <climits>
#include <type_traits>

#include "common.hpp"
#include "e4m3.cuh"

namespace {

using vlasim_dev::cvt_e4m3x2;
using vlasim_dev::e4m3_fix;
using vlasim_dev::e4m3_suspect;

constexpr int kElems = 8;  // consecutive elements per thread in the element-wise passes

// Flat index → group, advanced incrementally (no 64-bit division per element).
struct GroupMap {
  int kind;                   // VLASIM_GRAN_*
  int64_t n;                  // elements
  int64_t ch, inner;          // PerChannel: [outer, ch, inner]
  int64_t rows, cols;         // PerBlock:   [batch, rows, cols]
  int64_t nbr, nbc;           //             ⌈rows/128⌉, ⌈cols/128⌉
  int64_t groups;
  int vec;                    // input base 16-byte aligned: 8-element chunks as vector loads
};

// I = int (tensors below 2^31 elements: 32-bit divisions in seek) or int64_t.
template <typename I>
struct GroupCursor {
  I a, b, c;  // PerChannel: (outer, channel, inner); PerBlock: (batch, row, col)
  __device__ void seek(const GroupMap& m, I i) {
    if (m.kind == VLASIM_GRAN_CHANNEL) {
      c = i % I(m.inner);
      const I t = i / I(m.inner);
      b = t % I(m.ch);
      a = t / I(m.ch);
    } else if (m.kind == VLASIM_GRAN_BLOCK) {
      c = i % I(m.cols);
      const I t = i / I(m.cols);
      b = t % I(m.rows);
      a = t / I(m.rows);
    } else {
      a = b = c = 0;
    }
  }
  __device__ int64_t group(const GroupMap& m) const {
    if (m.kind == VLASIM_GRAN_CHANNEL) return b;
    if (m.kind == VLASIM_GRAN_BLOCK) return (int64_t(a) * m.nbr + (b >> 7)) * m.nbc + (c >> 7);
    return 0;
  }
  __device__ void next(const GroupMap& m) {
    if (m.kind == VLASIM_GRAN_CHANNEL) {
      if (++c == I(m.inner)) {
        c = 0;
        if (++b == I(m.ch)) b = 0, ++a;
      }
    } else if (m.kind == VLASIM_GRAN_BLOCK) {
      if (++c == I(m.cols)) {
        c = 0;
        if (++b == I(m.rows)) b = 0, ++a;
      }
    }
  }
};

// 8 consecutive elements → fp32 (vector loads when the chunk lies inside the tensor)
template <typename T>
__device__ __forceinline__ void load8(const T* x, int64_t i0, int64_t n, int vec, float (&v)[8]);
template <>
__device__ __forceinline__ void load8<float>(const float* x, int64_t i0, int64_t n, int vec, float (&v)[8]) {
  if (vec && i0 + 8 <= n) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(x + i0)), b = __ldg(reinterpret_cast<const float4*>(x + i0) + 1);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = i0 + j < n ? __ldg(x + i0 + j) : 0.f;
  }
}
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* x, int64_t i0, int64_t n, int vec,
                                                     float (&v)[8]) {
  if (vec && i0 + 8 <= n) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(x + i0));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      v[2 * j] = f.x, v[2 * j + 1] = f.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = i0 + j < n ? __bfloat162float(x[i0 + j]) : 0.f;
  }
}

constexpr int kChunks = 4;  // 8-element chunks per thread (one cursor seek per 32 elements)

template <typename T>
__device__ __forceinline__ float load_f(const T* p, int64_t i);
template <>
__device__ __forceinline__ float load_f<float>(const float* p, int64_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ float load_f<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
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

// ---- generic pass 1 (PerChannel over a middle axis with groups too large for k_group_fused):
// per-group amax; runs of one group are folded in registers and flushed with one atomicMax on the
// fp32 bit pattern (order-independent, hence deterministic).
template <typename T, typename I>
__global__ void __launch_bounds__(256) k_amax(const T* __restrict__ x, GroupMap m, uint32_t* __restrict__ amax,
                                              int32_t* __restrict__ status) {
  const int64_t nruns = (m.n + 8 * kChunks - 1) / (8 * kChunks);
  for (int64_t rk = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; rk < nruns;
       rk += int64_t(gridDim.x) * blockDim.x) {
    const int64_t base = rk * 8 * kChunks;
    GroupCursor<I> cur;
    cur.seek(m, I(base));
    int64_t g = cur.group(m);
    float run = 0.f;
#pragma unroll
    for (int ck = 0; ck < kChunks; ++ck) {
      const int64_t i0 = base + 8 * ck;
      if (i0 >= m.n) break;
      float v[8];
      load8(x, i0, m.n, m.vec, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (i0 + j >= m.n) break;
        const int64_t gj = cur.group(m);
        if (gj != g) {
          atomicMax(amax + g, __float_as_uint(run));
          g = gj;
          run = 0.f;
        }
        cur.next(m);
        if (!isfinite(v[j])) report_bad(status, i0 + j);
        run = fmaxf(run, fabsf(v[j]));
      }
    }
    atomicMax(amax + g, __float_as_uint(run));
  }
}

__global__ void k_status_init(int32_t* status) {
  status[0] = 0;
  status[1] = INT_MAX;
}

__global__ void k_scales(const uint32_t* __restrict__ amax, int64_t groups, float* __restrict__ scales) {
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (g < groups) {
    const float a = __uint_as_float(amax[g]);
    scales[g] = a == 0.f ? 1.f : __fdiv_rn(a, 448.f);
  }
}

// Per-group reciprocal for code_of: RN(1/amax), or 0 for a degenerate maximum (0, or outside
// 2^±100, where |x|·448 could overflow or 1/amax lose precision as an fp32 subnormal).
__device__ __forceinline__ float group_rcp(float a) {
  const int e = int((__float_as_uint(a) >> 23) & 0xFF) - 127;
  return (a == 0.f || e < -100 || e > 100) ? 0.f : __frcp_rn(a);
}

// Code byte of one element (sign | RNE magnitude) in a group of maximum a, r = group_rcp(a).
// All-zero group: the code of ±0 (scale 1).  Otherwise the RNE code of X = |x|·448/amax from the
// fp32 quotient q (A = fp32(|x|·448), q = A·r corrected once: within ~2 ulps of X), exact unless q
// lies next to a midpoint — then e4m3_fix's fp64 comparisons decide (|x|·448 and midpoint·amax are
// exact there).  Degenerate maxima (r = 0): an fp64 candidate, always re-decided exactly.
__device__ __forceinline__ uint32_t code_of(float x, float a, float r) {
  uint32_t mag = 0;
  if (a != 0.f) {
    const float ax = fabsf(x);
    if (r != 0.f) {
      const float A = ax * 448.f;
      const float q0 = A * r, q = fmaf(fmaf(-q0, a, A), r, q0);
      mag = cvt_e4m3x2(q, 0.f) & 0x7F;
      if (e4m3_suspect(q)) mag = e4m3_fix(mag, ax, a);
    } else {
      mag = e4m3_fix(cvt_e4m3x2(float(double(ax) * 448.0 / double(a)), 0.f) & 0x7F, ax, a);
    }
  }
  return mag | (signbit(x) ? 0x80u : 0u);
}

// Four elements at once, element j in a group of maximum a[j] with r[j] = group_rcp(a[j]) != 0
// (callers route zero / degenerate maxima to code_of).  Branch-free common case: the quotients,
// one packed cvt per pair, the sign bytes by byte permutes; the midpoint test of all four folds into
// one predicate and only a flagged unit re-decides its elements (e4m3_suspect / e4m3_fix).
__device__ __forceinline__ uint32_t encode4(const float (&v)[4], const float (&a)[4], const float (&r)[4]) {
  float q[4];
  bool sus = false;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float A = fabsf(v[j]) * 448.f;
    const float q0 = A * r[j];
    q[j] = fmaf(fmaf(-q0, a[j], A), r[j], q0);
    const float t = fmaf(q[j], 512.f, -0.5f);  // an integer iff q·2^10 is odd (a subnormal-range midpoint)
    const bool near_sub = fabsf(t - rintf(t)) < 0.0001220703125f;
    const bool near_nrm = ((__float_as_uint(q[j]) + (0x40u - 0x80000u)) & 0xFFFFFu) <= 0x80u;
    sus |= q[j] < 0.015625f ? near_sub : near_nrm;
  }
  uint32_t w = uint32_t(cvt_e4m3x2(q[0], q[1])) | (uint32_t(cvt_e4m3x2(q[2], q[3])) << 16);
  if (sus) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (e4m3_suspect(q[j])) {
        const uint32_t c = e4m3_fix((w >> (8 * j)) & 0x7F, fabsf(v[j]), a[j]);
        w = (w & ~(0xFFu << (8 * j))) | (c << (8 * j));
      }
  }
  const uint32_t b0 = __float_as_uint(v[0]), b1 = __float_as_uint(v[1]);
  const uint32_t b2 = __float_as_uint(v[2]), b3 = __float_as_uint(v[3]);
  const uint32_t sg = __byte_perm(__byte_perm(b0, b1, 0x0073), __byte_perm(b2, b3, 0x7300), 0x7610);
  return w | (sg & 0x80808080u);
}

template <typename T, typename I>
__global__ void __launch_bounds__(256) k_codes(const T* __restrict__ x, GroupMap m, const uint32_t* __restrict__ amax,
                                               uint8_t* __restrict__ codes, const int32_t* __restrict__ status) {
  if (status && status[0] != 0) return;  // non-finite input: no codes written
  const int64_t nruns = (m.n + 8 * kChunks - 1) / (8 * kChunks);
  for (int64_t rk = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; rk < nruns;
       rk += int64_t(gridDim.x) * blockDim.x) {
    const int64_t base = rk * 8 * kChunks;
    GroupCursor<I> cur;
    cur.seek(m, I(base));
    int64_t g = -1;
    float a = 0.f, r = 0.f;
#pragma unroll
    for (int ck = 0; ck < kChunks; ++ck) {
      const int64_t i0 = base + 8 * ck;
      if (i0 >= m.n) break;
      float v[8];
      load8(x, i0, m.n, m.vec, v);
      uint32_t w[2] = {0, 0};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (i0 + j >= m.n) break;
        const int64_t gj = cur.group(m);
        if (gj != g) {  // a new group: its amax and reciprocal
          g = gj;
          a = __uint_as_float(__ldg(amax + g));
          r = group_rcp(a);
        }
        w[j >> 2] |= code_of(v[j], a, r) << (8 * (j & 3));
        cur.next(m);
      }
      if (i0 + 8 <= m.n) {
        *reinterpret_cast<uint2*>(codes + i0) = make_uint2(w[0], w[1]);
      } else {
        for (int j = 0; i0 + j < m.n; ++j) codes[i0 + j] = uint8_t(w[j >> 2] >> (8 * (j & 3)));
      }
    }
  }
}

// ---- coalesced specialisations (the generic passes above keep one thread on 32 consecutive
// elements: every warp load then touches 32 lines and the amax/code passes ran at 7-18 % of HBM).
// Here a warp's lanes always read consecutive 4-element units, so each load instruction is one
// contiguous 512-B (fp32) / 256-B (bf16) span.

template <typename T>
__device__ __forceinline__ void load4(const T* x, int64_t i, float (&v)[4]);
template <>
__device__ __forceinline__ void load4<float>(const float* x, int64_t i, float (&v)[4]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(x + i));
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
}
template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* x, int64_t i, float (&v)[4]) {
  const uint2 q = __ldg(reinterpret_cast<const uint2*>(x + i));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.y));
  v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
}

// VEC-element unit u (VEC = 4: vector load; 1: scalar)
template <int VEC, typename T>
__device__ __forceinline__ void load_unit(const T* x, int64_t i, float (&v)[4]) {
  if constexpr (VEC == 4) load4(x, i, v);
  else v[0] = load_f(x, i);
}

template <int VEC>
__device__ __forceinline__ void store_unit(uint8_t* codes, int64_t i, uint32_t w) {
  if constexpr (VEC == 4) *reinterpret_cast<uint32_t*>(codes + i) = w;
  else codes[i] = uint8_t(w);
}

__device__ __forceinline__ bool finite_unit(const float (&v)[4], int cnt, int64_t i, int32_t* status) {
  bool ok = true;
  for (int j = 0; j < cnt; ++j)
    if (!isfinite(v[j])) report_bad(status, i + j), ok = false;
  return ok;
}

// PerTensor pass 1: units grid-strided (4 in flight per thread), block max, one atomic per CTA.
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_tensor_amax(const T* __restrict__ x, int64_t n, uint32_t* __restrict__ amax,
                                                     int32_t* __restrict__ status) {
  __shared__ float s_red[8];
  const int64_t nunits = n / VEC, stride = int64_t(gridDim.x) * blockDim.x;
  float mx = 0.f;
  for (int64_t u0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u0 < nunits; u0 += 4 * stride) {
    float v[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (u0 + k * stride < nunits) load_unit<VEC>(x, (u0 + k * stride) * VEC, v[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (u0 + k * stride < nunits) {
        if (!finite_unit(v[k], VEC, (u0 + k * stride) * VEC, status)) continue;
#pragma unroll
        for (int j = 0; j < VEC; ++j) mx = fmaxf(mx, fabsf(v[k][j]));
      }
  }
  for (int64_t i = nunits * VEC + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const float f = load_f(x, i);  // tail (n % VEC)
    if (!isfinite(f)) report_bad(status, i);
    else mx = fmaxf(mx, fabsf(f));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) b = fmaxf(b, s_red[w]);
    atomicMax(amax, __float_as_uint(b));
  }
}

template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_tensor_codes(const T* __restrict__ x, int64_t n,
                                                      const uint32_t* __restrict__ amax, uint8_t* __restrict__ codes,
                                                      const int32_t* __restrict__ status) {
  if (status && status[0] != 0) return;
  const float a = __uint_as_float(amax[0]), r = group_rcp(a);
  const int64_t nunits = n / VEC, stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t u0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u0 < nunits; u0 += 4 * stride) {
    float v[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (u0 + k * stride < nunits) load_unit<VEC>(x, (u0 + k * stride) * VEC, v[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (u0 + k * stride < nunits) {
        uint32_t w = 0;
        if (VEC == 4 && r != 0.f) {
          const float a4[4] = {a, a, a, a}, r4[4] = {r, r, r, r};
          w = encode4(v[k], a4, r4);
        } else {
#pragma unroll
          for (int j = 0; j < VEC; ++j) w |= code_of(v[k][j], a, r) << (8 * j);
        }
        store_unit<VEC>(codes, (u0 + k * stride) * VEC, w);
      }
  }
  for (int64_t i = nunits * VEC + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    codes[i] = uint8_t(code_of(load_f(x, i), a, r));
}

// Groups whose elements form a 2-D region (nr rows × nc contiguous columns, row pitch ld): PerBlock
// (≤ 128 × 128) and PerChannel with outer·inner ≤ kFusedMax.  Persistent CTAs of NT threads walk
// the groups; each group is held in registers (16 elements per thread), so amax, scale and codes
// come from ONE read of x (5 B/element of HBM traffic for fp32), and the next group's loads are
// issued before the current group is reduced and encoded (two register sets, A/B), so the encode
// arithmetic overlaps the HBM stream instead of alternating with it.  NT = 1024 (one CTA per SM) for
// groups above 8 K elements, else 512 (two per SM): 32 warps per SM either way, ≤ 64 registers.
constexpr int kFusedUnits = 4;                                          // 4-element slots per thread
constexpr int64_t kFusedMax = int64_t(1024) * 4 * kFusedUnits;          // 16384 elements per group

struct Region {
  int64_t base, ld;
  int nr, nc;
  int row0, col0, drow, dcol;  // VEC = 4 unit walk: this thread's first unit, the step of 512 units
};

// (groups < 2^31 and block-grid extents < 2^31: 32-bit divisions, host-checked)
template <int NT>
__device__ __forceinline__ Region group_region(const GroupMap& m, int64_t g64) {
  Region rg;
  const uint32_t g = uint32_t(g64);
  if (m.kind == VLASIM_GRAN_BLOCK) {
    const uint32_t nbc = uint32_t(m.nbc), nbr = uint32_t(m.nbr);
    const uint32_t q = g / nbc, bc = g - q * nbc, b = q / nbr, br = q - b * nbr;
    rg.nr = int(m.rows - br * 128 < 128 ? m.rows - br * 128 : 128);
    rg.nc = int(m.cols - bc * 128 < 128 ? m.cols - bc * 128 : 128);
    rg.ld = m.cols;
    rg.base = (int64_t(b) * m.rows + int64_t(br) * 128) * m.cols + int64_t(bc) * 128;
  } else {  // PerChannel: [outer, ch, inner], channel g
    rg.nr = int(m.n / (m.ch * m.inner));
    rg.nc = int(m.inner);
    rg.ld = m.ch * m.inner;
    rg.base = int64_t(g) * m.inner;
  }
  const uint32_t upr = uint32_t(rg.nc) >> 2, t = threadIdx.x;
  if (upr) {
    rg.row0 = int(t / upr), rg.col0 = int(t - uint32_t(rg.row0) * upr);
    rg.drow = int(uint32_t(NT) / upr), rg.dcol = int(uint32_t(NT) - uint32_t(rg.drow) * upr);
  }
  return rg;
}

// unit k of this thread (VEC = 4): row/column walked incrementally from (row0, col0)
#define FUSED_UNIT_WALK(rg, row, col)                   \
  int row = rg.row0, col = rg.col0;                     \
  const int upr_ = rg.nc >> 2, units_ = rg.nr * upr_;   \
  (void)units_
#define FUSED_UNIT_STEP(rg, row, col) \
  do {                                \
    row += rg.drow;                   \
    col += rg.dcol;                   \
    if (col >= upr_) col -= upr_, ++row; \
  } while (0)

// slot k: one 4-element unit u = tid + NT·k (VEC = 4, nc % 4 == 0, host-checked) or the 4 scalar
// elements (4k + j)·NT + tid (VEC = 1)
template <typename T, int VEC, int NT>
__device__ __forceinline__ void fused_load(const T* __restrict__ x, const Region& rg, float (&v)[kFusedUnits][4]) {
  const int tid = int(threadIdx.x);
  if constexpr (VEC == 4) {
    FUSED_UNIT_WALK(rg, row, col);
#pragma unroll
    for (int k = 0; k < kFusedUnits; ++k) {
      if (row < rg.nr) load4(x, rg.base + row * rg.ld + 4 * col, v[k]);
      FUSED_UNIT_STEP(rg, row, col);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < kFusedUnits; ++k) {
    {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = tid + NT * (4 * k + j);
        if (e < rg.nr * rg.nc) {
          const int row = e / rg.nc, col = e - row * rg.nc;
          v[k][j] = load_f(x, rg.base + row * rg.ld + col);
        }
      }
    }
  }
}

template <int VEC, int NT>
__device__ __forceinline__ void fused_encode(const Region& rg, int64_t g, const float (&v)[kFusedUnits][4],
                                             float* s_red, uint8_t* __restrict__ codes, float* __restrict__ scales,
                                             int32_t* __restrict__ status) {
  const int tid = int(threadIdx.x);
  float mx = 0.f;
  bool ok = true;
  const int total = rg.nr * rg.nc;
#pragma unroll
  for (int k = 0; k < kFusedUnits; ++k) {
    if constexpr (VEC == 4) {
      if (4 * (tid + NT * k) < total) {  // whole unit valid (nc % 4 == 0)
        const float m4 = fmaxf(fmaxf(fabsf(v[k][0]), fabsf(v[k][1])), fmaxf(fabsf(v[k][2]), fabsf(v[k][3])));
        // a non-finite element makes the sum non-finite (an overflowing sum of finite values only
        // sends the unit to the exact per-element test)
        if (!isfinite((v[k][0] + v[k][1]) + (v[k][2] + v[k][3])))
          ok &= isfinite(v[k][0]) && isfinite(v[k][1]) && isfinite(v[k][2]) && isfinite(v[k][3]);
        mx = fmaxf(mx, m4);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (tid + NT * (4 * k + j) < total) {
          ok &= isfinite(v[k][j]);
          mx = fmaxf(mx, fabsf(v[k][j]));
        }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) s_red[tid >> 5] = mx;
  if (__syncthreads_or(!ok)) {  // a non-finite element: name it, leave this group's codes unwritten
    if (!ok) {
#pragma unroll
      for (int k = 0; k < kFusedUnits; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int e = VEC == 4 ? 4 * (tid + NT * k) + j : tid + NT * (4 * k + j);
          if (e < rg.nr * rg.nc && !isfinite(v[k][j])) {
            const int row = e / rg.nc, col = e - row * rg.nc;
            report_bad(status, rg.base + row * rg.ld + col);
          }
        }
    }
    return;
  }
  float a = 0.f;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) a = fmaxf(a, s_red[w]);
  if (tid == 0) scales[g] = a == 0.f ? 1.f : __fdiv_rn(a, 448.f);
  const float r = group_rcp(a);
  if constexpr (VEC == 4) {
    FUSED_UNIT_WALK(rg, row, col);
#pragma unroll
    for (int k = 0; k < kFusedUnits; ++k) {
      if (row < rg.nr) {
        uint32_t w = 0;
        if (r != 0.f) {
          const float a4[4] = {a, a, a, a}, r4[4] = {r, r, r, r};
          w = encode4(v[k], a4, r4);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) w |= code_of(v[k][j], a, r) << (8 * j);
        }
        *reinterpret_cast<uint32_t*>(codes + rg.base + row * rg.ld + 4 * col) = w;
      }
      FUSED_UNIT_STEP(rg, row, col);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < kFusedUnits; ++k) {
    {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = tid + NT * (4 * k + j);
        if (e < rg.nr * rg.nc) {
          const int row = e / rg.nc, col = e - row * rg.nc;
          codes[rg.base + row * rg.ld + col] = uint8_t(code_of(v[k][j], a, r));
        }
      }
    }
  }
}

template <typename T, int VEC, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_group_fused(const T* __restrict__ x, GroupMap m,
                                                               uint8_t* __restrict__ codes, float* __restrict__ scales,
                                                               int32_t* __restrict__ status) {
  __shared__ float s_red[2][NT / 32];  // by group parity: one barrier per group suffices
  float va[kFusedUnits][4], vb[kFusedUnits][4];
  int64_t g = blockIdx.x;
  if (g >= m.groups) return;
  Region ra = group_region<NT>(m, g), rb;
  fused_load<T, VEC, NT>(x, ra, va);
  for (;;) {
    const int64_t g1 = g + gridDim.x, g2 = g1 + gridDim.x;
    if (g1 < m.groups) {
      rb = group_region<NT>(m, g1);
      fused_load<T, VEC, NT>(x, rb, vb);  // in flight while group g is encoded
    }
    fused_encode<VEC, NT>(ra, g, va, s_red[0], codes, scales, status);
    if (g1 >= m.groups) break;
    if (g2 < m.groups) {
      ra = group_region<NT>(m, g2);
      fused_load<T, VEC, NT>(x, ra, va);
    }
    fused_encode<VEC, NT>(rb, g1, vb, s_red[1], codes, scales, status);
    if (g2 >= m.groups) break;
    g = g2;
  }
}

// PerChannel over the LAST axis (inner == 1): the tensor is [R rows, C channels] and a group is a
// column.  Each thread owns VEC adjacent columns of a row slab (blockIdx.y): loads stay coalesced
// along the row, the column maxima live in registers, one atomicMax per column per slab.
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_col_amax(const T* __restrict__ x, int64_t R, int64_t C, int64_t slab,
                                                  uint32_t* __restrict__ amax, int32_t* __restrict__ status) {
  const int64_t c0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * VEC;
  if (c0 >= C) return;
  const int64_t r0 = blockIdx.y * slab, r1 = R < r0 + slab ? R : r0 + slab;
  float mx[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t r = r0; r < r1; r += 4) {
    float v[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (r + k < r1) load_unit<VEC>(x, (r + k) * C + c0, v[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (r + k < r1 && finite_unit(v[k], VEC, (r + k) * C + c0, status)) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) mx[j] = fmaxf(mx[j], fabsf(v[k][j]));
      }
  }
#pragma unroll
  for (int j = 0; j < VEC; ++j) atomicMax(amax + c0 + j, __float_as_uint(mx[j]));
}

template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_col_codes(const T* __restrict__ x, int64_t R, int64_t C, int64_t slab,
                                                   const uint32_t* __restrict__ amax, uint8_t* __restrict__ codes,
                                                   const int32_t* __restrict__ status) {
  if (status && status[0] != 0) return;
  const int64_t c0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * VEC;
  if (c0 >= C) return;
  const int64_t r0 = blockIdx.y * slab, r1 = R < r0 + slab ? R : r0 + slab;
  float a[4] = {0.f, 0.f, 0.f, 0.f}, rc[4] = {0.f, 0.f, 0.f, 0.f};
  bool fast = true;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    a[j] = __uint_as_float(amax[c0 + j]);
    rc[j] = group_rcp(a[j]);
    fast &= rc[j] != 0.f;
  }
  for (int64_t r = r0; r < r1; r += 4) {
    float v[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (r + k < r1) load_unit<VEC>(x, (r + k) * C + c0, v[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (r + k < r1) {
        uint32_t w = 0;
        if (VEC == 4 && fast) {
          w = encode4(v[k], a, rc);
        } else {
#pragma unroll
          for (int j = 0; j < VEC; ++j) w |= code_of(v[k][j], a[j], rc[j]) << (8 * j);
        }
        store_unit<VEC>(codes, (r + k) * C + c0, w);
      }
  }
}

__global__ void __launch_bounds__(256) k_dequant(const uint8_t* __restrict__ codes, const float* __restrict__ scales,
                                                 GroupMap m, float* __restrict__ out) {
  const int64_t nchunks = (m.n + kElems - 1) / kElems;
  for (int64_t ck = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ck < nchunks;
       ck += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i0 = ck * kElems;
    GroupCursor<int64_t> cur;
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
  if (reinterpret_cast<uintptr_t>(d_codes) & 7) return set_error(VLASIM_ECONFIG, "quantize: codes must be 8-byte aligned");
  if ((flags & VLASIM_SYNC_CHECK) && !d_status) return set_error(VLASIM_ECONFIG, "quantize: sync check needs d_status");
  if (!d_workspace || workspace_bytes < size_t(m.groups) * 4)
    return set_error(VLASIM_ECONFIG, "quantize: workspace too small (%zu < %zu)", workspace_bytes,
                     size_t(m.groups) * 4);
  cudaStream_t st = as_stream(stream);
  uint32_t* amax = static_cast<uint32_t*>(d_workspace);
  VLASIM_CUDA_TRY(cudaMemsetAsync(amax, 0, size_t(m.groups) * 4, st));
  if (d_status) k_status_init<<<1, 1, 0, st>>>(d_status);  // {0, INT_MAX} (no pageable copy)
  const int esz = dtype == VLASIM_DTYPE_F32 ? 4 : 2;
  m.vec = (reinterpret_cast<uintptr_t>(d_x) & 15) == 0;
  const bool al4 = (reinterpret_cast<uintptr_t>(d_x) % (4 * esz)) == 0;  // a 4-element unit is one load
  const int nsm = num_sms();
  // routing: PerTensor → coalesced two-pass; PerBlock and small-region PerChannel → fused one-pass;
  // last-axis PerChannel → column-owned two-pass; any other PerChannel → the generic passes
  const int64_t outer = m.kind == VLASIM_GRAN_CHANNEL ? m.n / (m.ch * m.inner) : 0;
  const bool fused = (m.kind == VLASIM_GRAN_BLOCK ||
                      (m.kind == VLASIM_GRAN_CHANNEL && m.inner > 1 && outer * m.inner <= kFusedMax)) &&
                     m.groups <= INT_MAX;  // (32-bit group arithmetic in group_region)
  const bool colwise = m.kind == VLASIM_GRAN_CHANNEL && m.inner == 1;
  const bool i32 = m.n < (int64_t(1) << 31);
  auto run = [&](auto* x) -> int {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(x)>>;
    if (m.kind == VLASIM_GRAN_TENSOR) {
      const int64_t units = al4 ? m.n / 4 : m.n;
      const int grid = int(std::max<int64_t>(1, std::min<int64_t>((units + 1023) / 1024, int64_t(nsm) * 8)));
      if (al4) {
        k_tensor_amax<T, 4><<<grid, 256, 0, st>>>(x, m.n, amax, d_status);
        k_scales<<<1, 256, 0, st>>>(amax, 1, d_scales);
        k_tensor_codes<T, 4><<<grid, 256, 0, st>>>(x, m.n, amax, d_codes, d_status);
      } else {
        k_tensor_amax<T, 1><<<grid, 256, 0, st>>>(x, m.n, amax, d_status);
        k_scales<<<1, 256, 0, st>>>(amax, 1, d_scales);
        k_tensor_codes<T, 1><<<grid, 256, 0, st>>>(x, m.n, amax, d_codes, d_status);
      }
      return VLASIM_OK;
    }
    if (fused) {
      const int64_t nc = m.kind == VLASIM_GRAN_BLOCK ? m.cols : m.inner;
      const int64_t ld = m.kind == VLASIM_GRAN_BLOCK ? m.cols : m.ch * m.inner;
      const bool v4 = al4 && nc % 4 == 0 && ld % 4 == 0;
      const int64_t gelems = m.kind == VLASIM_GRAN_BLOCK ? std::min<int64_t>(m.rows, 128) * std::min<int64_t>(m.cols, 128)
                                                         : outer * m.inner;
      if (gelems > 8192) {
        const int grid = int(std::min<int64_t>(m.groups, nsm));
        if (v4) k_group_fused<T, 4, 1024><<<grid, 1024, 0, st>>>(x, m, d_codes, d_scales, d_status);
        else k_group_fused<T, 1, 1024><<<grid, 1024, 0, st>>>(x, m, d_codes, d_scales, d_status);
      } else {
        const int grid = int(std::min<int64_t>(m.groups, 2 * int64_t(nsm)));
        if (v4) k_group_fused<T, 4, 512><<<grid, 512, 0, st>>>(x, m, d_codes, d_scales, d_status);
        else k_group_fused<T, 1, 512><<<grid, 512, 0, st>>>(x, m, d_codes, d_scales, d_status);
      }
      return VLASIM_OK;
    }
    if (colwise) {
      const int64_t R = m.n / m.ch, Cc = m.ch;
      const bool v4 = al4 && Cc % 4 == 0;
      const int64_t gx = (Cc + (v4 ? 1024 : 256) - 1) / (v4 ? 1024 : 256);
      int64_t gy = std::max<int64_t>(1, std::min<int64_t>(R, (int64_t(nsm) * 8 + gx - 1) / gx));
      int64_t slab = (R + gy - 1) / gy;
      slab = std::max<int64_t>(slab, (R + 65534) / 65535);
      gy = (R + slab - 1) / slab;
      if (gx > INT_MAX) return set_error(VLASIM_ECONFIG, "quantize: too many channels");
      const dim3 grid{unsigned(gx), unsigned(gy), 1u};
      if (v4) k_col_amax<T, 4><<<grid, 256, 0, st>>>(x, R, Cc, slab, amax, d_status);
      else k_col_amax<T, 1><<<grid, 256, 0, st>>>(x, R, Cc, slab, amax, d_status);
      k_scales<<<int((m.groups + 255) / 256), 256, 0, st>>>(amax, m.groups, d_scales);
      if (v4) k_col_codes<T, 4><<<grid, 256, 0, st>>>(x, R, Cc, slab, amax, d_codes, d_status);
      else k_col_codes<T, 1><<<grid, 256, 0, st>>>(x, R, Cc, slab, amax, d_codes, d_status);
      return VLASIM_OK;
    }
    const int64_t nruns = (m.n + 8 * kChunks - 1) / (8 * kChunks);
    const int grid = int(std::min<int64_t>((nruns + 255) / 256, int64_t(nsm) * 8));
    auto ka = i32 ? k_amax<T, int> : k_amax<T, int64_t>;
    auto kc = i32 ? k_codes<T, int> : k_codes<T, int64_t>;
    ka<<<std::max(grid, 1), 256, 0, st>>>(x, m, amax, d_status);
    k_scales<<<int((m.groups + 255) / 256), 256, 0, st>>>(amax, m.groups, d_scales);
    kc<<<std::max(grid, 1), 256, 0, st>>>(x, m, amax, d_codes, d_status);
    return VLASIM_OK;
  };
  if (dtype == VLASIM_DTYPE_F32) {
    if (int rc = run(static_cast<const float*>(d_x))) return rc;
  } else {
    if (int rc = run(static_cast<const __nv_bfloat16*>(d_x))) return rc;
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
