// e4m3.cuh — shared pieces of the E4M3 quantisers (fp8.cu, quant.cu): the packed RNE conversion and
// the exact re-decision of a code whose fp32 quotient lies next to a midpoint.
#pragma once
#include <cstdint>

namespace vlasim_dev {

__device__ __forceinline__ uint16_t cvt_e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

// Exact RNE (the code of the REAL quotient x / scale, scale = amax / 448).  The fp32
// quotient q = RN(x / RN(amax / 448)) is within a few fp32 ulps of the real quotient X = |x|·448/amax,
// so cvt(q) is the right code unless X lies within those ulps of a midpoint between two E4M3 values
// (or in the subnormal range, where the midpoint grid is finer): only then is the candidate code
// re-decided, by exact fp64 comparisons of |x|·448 against midpoint · amax (both products exact:
// ≤ 11 and ≤ 13 significant bits for bf16 inputs).  Midpoints have the fp32 pattern 1.xxx1 000…0,
// i.e. low 20 mantissa bits 0x80000.
// Below 2^-6 (E4M3's subnormal range) the midpoints are the odd multiples of 2^-10: suspect when
// q·2^10 lies within 2^-12 of an odd integer (the quotient's error there is below 2^-17 on that
// scale), not for the whole range — small elements of a wide-range group must not all take the
// fp64 path (they made the PerTensor code pass 4x slower on logspace data).
__device__ __forceinline__ bool e4m3_suspect(float q) {
  const float a = fabsf(q);
  if (a < 0.015625f) {
    const float t = fmaf(a, 512.f, -0.5f);  // an integer iff a·2^10 is odd
    return fabsf(t - rintf(t)) < 0.0001220703125f;
  }
  const int low = int(__float_as_uint(a) & 0xFFFFFu);
  return abs(low - 0x80000) <= 64;
}

static __device__ __noinline__ uint32_t e4m3_fix(uint32_t c, float ax, float amax) {
  const double A = double(ax) * 448.0, B = double(amax);
  const int e = int(c >> 3), m = int(c & 7), ee = e == 0 ? 1 : e;
  const int mant = e == 0 ? m : 8 + m;
  if (c < 0x7E) {  // midpoint to the next code up: (2·mant + 1) · 2^(ee−11)
    const double mu = ldexp(double(2 * mant + 1), ee - 11) * B;
    if (A > mu || (A == mu && (c & 1))) return c + 1;
  }
  if (c > 0) {  // midpoint to the next code down (half the spacing across a binade edge)
    const double md = (m == 0 && e >= 2) ? ldexp(double(4 * mant - 1), ee - 12) * B
                                         : ldexp(double(2 * mant - 1), ee - 11) * B;
    if (A < md || (A == md && (c & 1))) return c - 1;
  }
  return c;
}

}  // namespace vlasim_dev
