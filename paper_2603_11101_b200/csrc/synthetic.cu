// synthetic.cu — seeded synthetic inputs shared bit-for-bit with the CPU oracle
// (SURVEY.md §8(d)): sample lengths from the reference's seeding API (rng.hpp) and
// counter-based tensor values that are exactly representable in bf16.
#include <cuda_bf16.h>

#include <cmath>
#include <string_view>

#include "common.hpp"
#include "vlasim/util/rng.hpp"

namespace {

__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// value(i) = (top8(splitmix64(seed ^ i)) - 128) / 128  ∈ [-1, 1), exact in bf16.
__global__ void k_fill(__nv_bfloat16* __restrict__ x, int64_t count, uint64_t seed) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
  for (int64_t base = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * 8; base < count; base += stride) {
    if (base + 8 <= count) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float a = float(int(splitmix64_dev(seed ^ uint64_t(base + 2 * j)) >> 56) - 128) * (1.0f / 128.0f);
        const float b = float(int(splitmix64_dev(seed ^ uint64_t(base + 2 * j + 1)) >> 56) - 128) * (1.0f / 128.0f);
        __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
        w[j] = *reinterpret_cast<uint32_t*>(&v);
      }
      *reinterpret_cast<uint4*>(x + base) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (int64_t i = base; i < count; ++i)
        x[i] = __float2bfloat16_rn(float(int(splitmix64_dev(seed ^ uint64_t(i)) >> 56) - 128) * (1.0f / 128.0f));
    }
  }
}

}  // namespace

extern "C" int vlasim_fill_synthetic_bf16(void* d_x, int64_t count, uint64_t seed, vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (count <= 0) return VLASIM_OK;
  if (reinterpret_cast<uintptr_t>(d_x) & 15) return set_error(VLASIM_ECONFIG, "fill_synthetic: 16-byte alignment");
  const int64_t blocks = std::min<int64_t>((count / 8 + 255) / 256 + 1, int64_t(num_sms()) * 8);
  k_fill<<<blocks, 256, 0, as_stream(stream)>>>(static_cast<__nv_bfloat16*>(d_x), count, seed);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}

// Host-side length generators (the data-loader side of the path; not timed).
//  dist 0: uniform_int(lo=p1, hi=p2)                                (configs 1, 2)
//  dist 1: truncated geometric(p=p1, max=p2), inverse CDF on uniform01 (config 5;
//          the reference's long-tailed episode model)
//  dist 2: GR00T-like  64·uniform_int(1,2) + uniform_int(16,64)     (config 2, secondary)
//  dist 3: π0.5  2 views × 256 + uniform_int(p1, p2) text + p3 action tokens (config 3;
//          prefix = length - p3)
extern "C" int vlasim_gen_lengths(uint64_t root_seed, const char* label, int dist, int64_t n, double p1, double p2,
                                  double p3, int32_t* out) {
  using namespace vlasim_host;
  if (n < 0 || !out || !label) return set_error(VLASIM_ECONFIG, "gen_lengths: bad arguments");
  auto rng = vlasim::make_rng(root_seed, std::string_view(label), 0);
  switch (dist) {
    case 0:
      for (int64_t i = 0; i < n; ++i) out[i] = int32_t(vlasim::uniform_int(rng, int64_t(p1), int64_t(p2)));
      return VLASIM_OK;
    case 1: {
      const double p = p1;
      const int64_t mx = int64_t(p2);
      if (!(p > 0 && p < 1) || mx < 1) return set_error(VLASIM_ECONFIG, "gen_lengths: geometric needs 0<p<1, max>=1");
      const double tail = 1.0 - std::pow(1.0 - p, double(mx));
      for (int64_t i = 0; i < n; ++i) {
        const double u = vlasim::uniform01(rng);
        double k = std::ceil(std::log1p(-u * tail) / std::log1p(-p));
        if (!(k >= 1)) k = 1;
        if (k > double(mx)) k = double(mx);
        out[i] = int32_t(k);
      }
      return VLASIM_OK;
    }
    case 2:
      for (int64_t i = 0; i < n; ++i) {
        const int64_t views = vlasim::uniform_int(rng, 1, 2);
        out[i] = int32_t(64 * views + vlasim::uniform_int(rng, 16, 64));
      }
      return VLASIM_OK;
    case 3:
      for (int64_t i = 0; i < n; ++i)
        out[i] = int32_t(512 + vlasim::uniform_int(rng, int64_t(p1), int64_t(p2)) + int64_t(p3));
      return VLASIM_OK;
    default:
      return set_error(VLASIM_ECONFIG, "gen_lengths: unknown distribution %d", dist);
  }
}
