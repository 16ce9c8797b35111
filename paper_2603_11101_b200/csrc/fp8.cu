// fp8.cu — E4M3 per-block quantisation for the FP8 Q/K attention path.
//
// x [T, heads, d] bf16, quantised per head in 128-token × 128-d blocks (the SPEC's "last two
// dimensions" blocks, applied per head — DESIGN.md §2):
//   scale = amax(block) / 448 (1 if the block is all zero)
//   code  = RNE(x / scale) onto E4M3, saturating to ±448
// scale = RN_fp32(amax / 448); codes = the RNE code of the REAL quotient x·448/amax (e4m3_fix below),
// bit-exact with the oracle's exact mode; non-finite input → status VLASIM_ECONFIG.
#include <cuda_bf16.h>

#include "common.hpp"
#include "e4m3.cuh"
#include "sm100.cuh"

using vlasim_dev::cvt_e4m3x2;
using vlasim_dev::e4m3_fix;
using vlasim_dev::e4m3_suspect;
using vlasim_dev::f2_fma;
using vlasim_dev::f2_mul;

namespace {


__device__ __forceinline__ float e4m3_to_float(uint8_t c) {
  const int e = (c >> 3) & 0xF, m = c & 7;
  float v;
  if (e == 0) v = ldexpf(float(m) / 8.f, -6);
  else if (e == 15 && m == 7) v = __int_as_float(0x7fc00000);
  else v = ldexpf(1.f + float(m) / 8.f, e - 7);
  return (c & 0x80) ? -v : v;
}

// The same decision in fp32, exact once both sides are scaled by p2 = 2^-E(amax): A = |x|·p2·448
// (≤ 11 significant bits, ≤ 896) and B = amax·p2 ∈ [1, 2) (8 bits); midpoint · B has ≤ 13 bits.
// Valid for normal amax below 2^127 (p2 normal); e4m3_fix (fp64) covers the two degenerate cases.
__device__ __forceinline__ uint32_t e4m3_fix_f32(uint32_t c, float A, float B) {
  const int e = int(c >> 3), m = int(c & 7), ee = e == 0 ? 1 : e;
  const int mant = e == 0 ? m : 8 + m;
  const float u = __int_as_float((ee - 11 + 127) << 23);  // 2^(ee−11)
  const float mu = float(2 * mant + 1) * u * B;
  const float md = (m == 0 && e >= 2) ? float(4 * mant - 1) * (0.5f * u) * B : float(2 * mant - 1) * u * B;
  if (c < 0x7E && (A > mu || (A == mu && (c & 1)))) return c + 1;
  if (c > 0 && (A < md || (A == md && (c & 1)))) return c - 1;
  return c;
}

// Per-block constants of the fp32 decision: p2 = 2^-E(amax) (0 → use the fp64 path).
__device__ __forceinline__ float e4m3_fix_scale(float amax) {
  const int ef = int((__float_as_uint(amax) >> 23) & 0xFF);
  return (ef == 0 || ef >= 254) ? 0.f : __int_as_float((254 - ef) << 23);
}

__device__ __forceinline__ uint32_t e4m3_decide(uint32_t c, float ax, float amax, float p2) {
  return p2 != 0.f ? e4m3_fix_f32(c, ax * p2 * 448.f, amax * p2) : e4m3_fix(c, ax, amax);
}

// Non-finite bf16 in either half of a 32-bit word (exponent all ones).
__device__ __forceinline__ bool bf16x2_nonfinite(uint32_t w) {
  return ((w & 0x7F80u) == 0x7F80u) || ((w & 0x7F800000u) == 0x7F800000u);
}

__device__ __forceinline__ int first_nonfinite(uint4 q) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  int k = 7;
#pragma unroll
  for (int j = 7; j >= 0; --j)
    if (((w[j >> 1] >> (16 * (j & 1))) & 0x7F80u) == 0x7F80u) k = j;
  return k;
}

__device__ __forceinline__ void report_nonfinite(int32_t* status, int64_t idx) {
  if (status && atomicCAS(status, 0, VLASIM_ECONFIG) == 0) status[1] = int32_t(idx < INT32_MAX ? idx : INT32_MAX);
}

// One CTA (256 threads) per (head, 128-token block, 128-d block).
__global__ void __launch_bounds__(256) k_quant_block(const __nv_bfloat16* __restrict__ x, int T, int heads, int d,
                                                     uint8_t* __restrict__ codes, float* __restrict__ scales,
                                                     int32_t* __restrict__ status) {
  const int nbd = (d + 127) / 128, nbt = (T + 127) / 128;
  const int bd = blockIdx.x % nbd, bt = (blockIdx.x / nbd) % nbt, h = blockIdx.x / (nbd * nbt);
  const int t0 = bt * 128, c0 = bd * 128;
  const int rows = min(128, T - t0), cols = min(128, d - c0);
  __shared__ float red[8];
  // pass 1: amax (each thread: 2-element chunks of the block)
  float amax = 0.f;
  int64_t bad = -1;
  for (int e = threadIdx.x * 2; e < rows * 128; e += 512) {
    const int r = e / 128, c = e % 128;
    if (c < cols) {
      const __nv_bfloat16* p = x + (int64_t(t0 + r) * heads + h) * d + c0 + c;
      const float a0 = __bfloat162float(p[0]);
      if (!isfinite(a0)) bad = p - x;
      amax = fmaxf(amax, fabsf(a0));
      if (c + 1 < cols) {
        const float a1 = __bfloat162float(p[1]);
        if (!isfinite(a1)) bad = p + 1 - x;
        amax = fmaxf(amax, fabsf(a1));
      }
    }
  }
  if (__syncthreads_or(bad >= 0)) {
    if (bad >= 0) report_nonfinite(status, bad);
    return;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < 8 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  amax = red[0];
  const float scale = amax == 0.f ? 1.f : __fdiv_rn(amax, 448.f);
  const float p2 = e4m3_fix_scale(amax);
  if (threadIdx.x == 0) scales[(int64_t(h) * nbt + bt) * nbd + bd] = scale;
  // pass 2: codes
  for (int e = threadIdx.x * 2; e < rows * 128; e += 512) {
    const int r = e / 128, c = e % 128;
    if (c < cols) {
      const int64_t off = (int64_t(t0 + r) * heads + h) * d + c0 + c;
      const float xa = __bfloat162float(x[off]);
      const float a = __fdiv_rn(xa, scale);
      uint32_t ca = cvt_e4m3x2(a, 0.f) & 0xFF;
      if (amax != 0.f && e4m3_suspect(a)) ca = (ca & 0x80) | e4m3_decide(ca & 0x7F, fabsf(xa), amax, p2);
      codes[off] = uint8_t(ca);
      if (c + 1 < cols) {
        const float xb = __bfloat162float(x[off + 1]);
        const float b = __fdiv_rn(xb, scale);
        uint32_t cb = cvt_e4m3x2(b, 0.f) & 0xFF;
        if (amax != 0.f && e4m3_suspect(b)) cb = (cb & 0x80) | e4m3_decide(cb & 0x7F, fabsf(xb), amax, p2);
        codes[off + 1] = uint8_t(cb);
      }
    }
  }
}

// Vectorised variant for d % 8 == 0 (every head_dim the attention path takes): one CTA per
// (128-token block, 128-d block, head) with the head fastest, so co-resident CTAs read whole
// token rows; the block (≤ 32 KB bf16) is read ONCE into registers — 8 × 16-B loads per thread,
// 16 threads per 256-B row segment — reduced to amax, then written as 8-B code chunks.  One HBM
// read of x and one write of the codes: the HBM roofline of the operation.
__global__ void __launch_bounds__(256) k_quant_block_v(const __nv_bfloat16* __restrict__ x, int T, int heads, int d,
                                                       uint8_t* __restrict__ codes, float* __restrict__ scales,
                                                       int32_t* __restrict__ status) {
  const int nbd = (d + 127) / 128, nbt = (T + 127) / 128;
  const int h = blockIdx.x % heads, rest = blockIdx.x / heads;
  const int bd = rest % nbd, bt = rest / nbd;
  const int t0 = bt * 128, c0 = bd * 128;
  const int ch = threadIdx.x & 15, r0 = threadIdx.x >> 4;
  const bool cv = ch * 8 < min(128, d - c0);
  __shared__ float red[8];
  uint4 v[8];
  // |x| as bf16 bit patterns orders like the values (non-negative), and every non-finite bf16 has the
  // exponent all ones (≥ 0x7F80): one unsigned 16-bit-pair max per word gives both the block
  // maximum and the finiteness test
  uint32_t mb = 0;
  const size_t rstride = size_t(16) * heads * d;  // 16 token rows
  const __nv_bfloat16* xp = x + (int64_t(t0 + r0) * heads + h) * d + c0 + ch * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int t = t0 + r0 + 16 * i;
    v[i] = make_uint4(0, 0, 0, 0);
    if (cv && t < T) v[i] = __ldcs(reinterpret_cast<const uint4*>(xp + i * rstride));
    mb = __vmaxu2(mb, v[i].x & 0x7FFF7FFFu);
    mb = __vmaxu2(mb, v[i].y & 0x7FFF7FFFu);
    mb = __vmaxu2(mb, v[i].z & 0x7FFF7FFFu);
    mb = __vmaxu2(mb, v[i].w & 0x7FFF7FFFu);
  }
  const uint32_t top = max(mb & 0xFFFFu, mb >> 16);
  if (__syncthreads_or(top >= 0x7F80u)) {  // non-finite input → error (no codes written)
    if (top >= 0x7F80u) {
      int bad = 0;
#pragma unroll
      for (int i = 7; i >= 0; --i)
        if (bf16x2_nonfinite(v[i].x) | bf16x2_nonfinite(v[i].y) | bf16x2_nonfinite(v[i].z) | bf16x2_nonfinite(v[i].w))
          bad = 8 * i + first_nonfinite(v[i]);
      report_nonfinite(status, (int64_t(t0 + r0 + 16 * (bad >> 3)) * heads + h) * d + c0 + ch * 8 + (bad & 7));
    }
    return;
  }
  float amax = __uint_as_float(top << 16);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = fmaxf(fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3])), fmaxf(fmaxf(red[4], red[5]), fmaxf(red[6], red[7])));
  const float scale = amax == 0.f ? 1.f : __fdiv_rn(amax, 448.f);
  const float p2 = e4m3_fix_scale(amax);
  if (threadIdx.x == 0) scales[(int64_t(h) * nbt + bt) * nbd + bd] = scale;
  // Codes = RNE of the REAL quotient X = |x|·448/amax, computed as A / B with both operands
  // scaled by p2 = 2^-E(amax) so that they are exact in fp32: A = x·(448·p2) (≤ 11 significant
  // bits) and B = amax·p2 ∈ [1, 2) (8 bits).  A midpoint M between two E4M3 codes has ≤ 5
  // significant bits, so when X ≠ M, |A − M·B| is a nonzero multiple of a grid ≥ 2^-13·M·B: X sits
  // at relative distance ≥ 2^-14 from every midpoint, far beyond the few fp32 ulps of error of the
  // quotient below — cvt.rn of the fp32 quotient is then the RNE code of X, and when X = M exactly
  // the quotient is exactly M and cvt's ties-to-even decides as the SPEC does.  No per-element
  // re-decision: the kernel stays a single HBM pass.  The quotient avoids a division per element
  // (IEEE div.rn is ~10 dependent instructions and made this kernel ALU-bound): q0 = RN(A·r) with
  // r = RN(1/B), corrected once, q = RN(q0 + RN(A − q0·B)·r) (the residual is exact by FMA).
  // Degenerate block maxima (bf16 subnormal or ≥ 2^127, p2 = 0) take the fp64 decision instead.
  const bool fast = p2 != 0.f;
  const float Bs = fast ? amax * p2 : scale, As = fast ? 448.f * p2 : 1.f;
  const float rs = __frcp_rn(Bs);
  const float2 r2 = make_float2(rs, rs), ns2 = make_float2(-Bs, -Bs), a2 = make_float2(As, As);
  auto quot = [&](float2 f) {  // (the correction turns −0 into +0: the sign bytes are OR-ed in below)
    const float2 fa = f2_mul(f, a2);
    const float2 q0 = f2_mul(fa, r2);
    return f2_fma(f2_fma(q0, ns2, fa), r2, q0);
  };
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int t = t0 + r0 + 16 * i;
    if (!cv || t >= T) continue;
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v[i]);
    uint32_t w[2];
    float qv[8];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float2 q0 = quot(__bfloat1622float2(b[2 * j])), q1 = quot(__bfloat1622float2(b[2 * j + 1]));
      qv[4 * j] = q0.x, qv[4 * j + 1] = q0.y, qv[4 * j + 2] = q1.x, qv[4 * j + 3] = q1.y;
      const uint32_t lo = cvt_e4m3x2(q0.x, q0.y);
      const uint32_t hi = cvt_e4m3x2(q1.x, q1.y);
      // the four inputs' sign bits (bf16 high bytes) onto the four codes: −0 keeps its sign
      const uint32_t wa = j ? v[i].z : v[i].x, wb = j ? v[i].w : v[i].y;
      w[j] = (lo | (hi << 16)) | (__byte_perm(wa, wb, 0x7531) & 0x80808080u);
    }
    if (!fast && amax != 0.f) {  // degenerate block maximum (block-uniform): fp64 re-decision
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (!e4m3_suspect(qv[k])) continue;
        const uint32_t sh = 8 * (k & 3), c = (w[k >> 2] >> sh) & 0xFF;
        const float ax = fabsf(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(&v[i])[k]));
        const uint32_t f = (c & 0x80) | e4m3_fix(c & 0x7F, ax, amax);
        w[k >> 2] = (w[k >> 2] & ~(0xFFu << sh)) | (f << sh);
      }
    }
    __stcs(reinterpret_cast<uint2*>(codes + (int64_t(t0 + r0) * heads + h) * d + c0 + ch * 8 + i * rstride),
           make_uint2(w[0], w[1]));
  }
}

__global__ void k_dequant_block(const uint8_t* __restrict__ codes, const float* __restrict__ scales, int64_t T,
                                int heads, int d, float* __restrict__ out) {
  const int64_t n = T * heads * d;
  const int nbd = (d + 127) / 128, nbt = int((T + 127) / 128);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(i % d);
    const int64_t th = i / d;
    const int h = int(th % heads);
    const int64_t t = th / heads;
    out[i] = e4m3_to_float(codes[i]) * scales[(int64_t(h) * nbt + t / 128) * nbd + c / 128];
  }
}

// quant_error per (head, 128-token, 128-d) group: max relative roundtrip
// error over the elements in E4M3's normal range (|x / scale| >= 2^-6, with the quantiser's fp32
// quotient), and the sum of squared errors.  deq = value(code) · scale and every error
// term are fp32 (one rounding each, as the oracle restates them); SSE accumulates in fp64.
__global__ void __launch_bounds__(256) k_quant_error(const __nv_bfloat16* __restrict__ x,
                                                     const uint8_t* __restrict__ codes,
                                                     const float* __restrict__ scales, int T, int heads, int d,
                                                     float* __restrict__ gmax, double* __restrict__ gsse,
                                                     int* __restrict__ gcnt) {
  const int nbd = (d + 127) / 128, nbt = (T + 127) / 128;
  const int bd = blockIdx.x % nbd, bt = (blockIdx.x / nbd) % nbt, h = blockIdx.x / (nbd * nbt);
  const int t0 = bt * 128, c0 = bd * 128;
  const int rows = min(128, T - t0), cols = min(128, d - c0);
  const float scale = scales[(int64_t(h) * nbt + bt) * nbd + bd];
  float mx = 0.f;
  double sse = 0.0;
  for (int e = threadIdx.x; e < rows * 128; e += 256) {
    const int r = e / 128, c = e % 128;
    if (c >= cols) continue;
    const int64_t off = (int64_t(t0 + r) * heads + h) * d + c0 + c;
    const float xv = __bfloat162float(x[off]);
    const uint8_t code = codes[off];
    const float diff = __fsub_rn(__fmul_rn(e4m3_to_float(code), scale), xv);
    sse += double(diff) * double(diff);
    if (fabsf(__fdiv_rn(xv, scale)) >= 0.015625f) mx = fmaxf(mx, __fdiv_rn(fabsf(diff), fabsf(xv)));
  }
  __shared__ float smx[8];
  __shared__ double ssse[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
  }
  if ((threadIdx.x & 31) == 0) {
    smx[threadIdx.x >> 5] = mx;
    ssse[threadIdx.x >> 5] = sse;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    double t = 0.0;
    for (int w = 0; w < 8; ++w) {
      m = fmaxf(m, smx[w]);
      t += ssse[w];
    }
    gmax[blockIdx.x] = m;
    gsse[blockIdx.x] = t;
    gcnt[blockIdx.x] = rows * cols;
  }
}

// codes → bf16(value(code) · scale) (fp32 product, one rounding): the Q/K operands of the FP8
// path's backward.  A thread converts 8 codes of one (token, head) row (8-B load, 16-B store) with
// the hardware E4M3 → f16 conversion (exact: every E4M3 value is an f16), indexing rows with 32-bit
// arithmetic (T · heads · d / 8 < 2^31, host-checked); d % 8 == 0.
__device__ __forceinline__ float2 e4m3x2_to_float2(uint16_t w) {
  uint32_t h;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(w));
  return __half22float2(*reinterpret_cast<const __half2*>(&h));
}

__global__ void k_dequant_bf16(const uint8_t* __restrict__ codes, const float* __restrict__ scales, uint32_t rows,
                               int heads, int d, int nbt, __nv_bfloat16* __restrict__ out) {
  const uint32_t cpr = uint32_t(d) >> 3, n8 = rows * cpr;
  const int nbd = (d + 127) / 128;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += gridDim.x * blockDim.x) {
    const uint32_t r = i / cpr, c8 = i - r * cpr;
    const uint32_t h = r % uint32_t(heads), t = r / uint32_t(heads);
    const float sc = __ldg(scales + (int64_t(h) * nbt + (t >> 7)) * nbd + (c8 >> 4));
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(codes) + i);
    uint4 o;
    uint32_t* oo = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t word = j < 2 ? w.x : w.y;
      const float2 f = e4m3x2_to_float2(uint16_t(word >> (16 * (j & 1))));
      const __nv_bfloat162 v = __floats2bfloat162_rn(f.x * sc, f.y * sc);
      oo[j] = *reinterpret_cast<const uint32_t*>(&v);
    }
    reinterpret_cast<uint4*>(out)[i] = o;
  }
}

}  // namespace

namespace vlasim_host {
int launch_fp8_dequant_bf16(const uint8_t* codes, const float* scales, int64_t T, int heads, int d, void* out,
                            cudaStream_t st) {
  if (d % 8) return set_error(VLASIM_ECONFIG, "fp8 dequant: head_dim %d not a multiple of 8", d);
  const int64_t n8 = T * heads * d / 8;
  if (n8 >= (int64_t(1) << 31)) return set_error(VLASIM_ECONFIG, "fp8 dequant: tensor too large");
  const int64_t blocks = std::min<int64_t>((n8 + 255) / 256, int64_t(num_sms()) * 16);
  k_dequant_bf16<<<blocks, 256, 0, st>>>(codes, scales, uint32_t(T * heads), heads, d, int((T + 127) / 128),
                                          static_cast<__nv_bfloat16*>(out));
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}
}  // namespace vlasim_host

extern "C" int vlasim_fp8_quant_error_cuda(const void* d_x, const uint8_t* d_codes, const float* d_scales, int64_t T,
                                           int32_t heads, int32_t d, float* d_group_maxrel, double* d_group_sse,
                                           int32_t* d_group_count, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (!d_x || !d_codes || !d_scales || !d_group_maxrel || !d_group_sse || !d_group_count)
    return set_error(VLASIM_ECONFIG, "fp8_quant_error: null buffer");
  if (T < 1 || heads < 1 || d < 1 || T >= (int64_t(1) << 31))
    return set_error(VLASIM_ECONFIG, "fp8_quant_error: bad shape T=%lld heads=%d d=%d", (long long)T, heads, d);
  const int64_t groups = int64_t(heads) * ((T + 127) / 128) * ((d + 127) / 128);
  k_quant_error<<<groups, 256, 0, as_stream(stream)>>>(static_cast<const __nv_bfloat16*>(d_x), d_codes, d_scales,
                                                       int(T), heads, d, d_group_maxrel, d_group_sse, d_group_count);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

extern "C" int vlasim_fp8_quant_block_cuda(const void* d_x, int64_t T, int32_t heads, int32_t d, uint8_t* d_codes,
                                           float* d_scales, int32_t* d_status, uint32_t flags,
                                           vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (!d_x || !d_codes || !d_scales) return set_error(VLASIM_ECONFIG, "fp8_quant_block: null buffer");
  if (T < 1 || heads < 1 || d < 1 || T >= (int64_t(1) << 31))
    return set_error(VLASIM_ECONFIG, "fp8_quant_block: bad shape T=%lld heads=%d d=%d", (long long)T, heads, d);
  if ((flags & VLASIM_SYNC_CHECK) && !d_status)
    return set_error(VLASIM_ECONFIG, "fp8_quant_block: VLASIM_SYNC_CHECK needs a status buffer");
  cudaStream_t st = as_stream(stream);
  if (d_status) VLASIM_CUDA_TRY(cudaMemsetAsync(d_status, 0, 2 * sizeof(int32_t), st));
  const int64_t blocks = int64_t(heads) * ((T + 127) / 128) * ((d + 127) / 128);
  if (d % 8 == 0 && (reinterpret_cast<uintptr_t>(d_x) & 15) == 0 && (reinterpret_cast<uintptr_t>(d_codes) & 7) == 0)
    k_quant_block_v<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(d_x), int(T), heads, d, d_codes,
                                            d_scales, d_status);
  else
    k_quant_block<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(d_x), int(T), heads, d, d_codes, d_scales,
                                          d_status);
  VLASIM_LAUNCH_CHECK();
  if (flags & VLASIM_SYNC_CHECK) {
    int32_t h[2];
    VLASIM_CUDA_TRY(cudaMemcpyAsync(h, d_status, sizeof(h), cudaMemcpyDeviceToHost, st));
    VLASIM_CUDA_TRY(cudaStreamSynchronize(st));
    if (h[0]) return set_error(VLASIM_ECONFIG, "quantize: non-finite input at element %d (SPEC.md:585)", h[1]);
  }
  return VLASIM_OK;
}

extern "C" int vlasim_fp8_dequant_block_cuda(const uint8_t* d_codes, const float* d_scales, int64_t T, int32_t heads,
                                             int32_t d, float* d_out, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (!d_codes || !d_scales || !d_out) return set_error(VLASIM_ECONFIG, "fp8_dequant_block: null buffer");
  if (T < 1 || heads < 1 || d < 1) return set_error(VLASIM_ECONFIG, "fp8_dequant_block: bad shape");
  const int64_t n = T * heads * d;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16);
  k_dequant_block<<<blocks, 256, 0, as_stream(stream)>>>(d_codes, d_scales, T, heads, d, d_out);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}
