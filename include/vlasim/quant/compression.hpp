// vlasim/quant/compression.hpp — model-compression calculator (reconstructed drop-in header for
// proj/CMakeLists.txt:21 src/quant/compression.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "vlasim/quant/quantize.hpp"

namespace vlasim {

struct ModelComponent {
  std::string name;
  std::int64_t params = 0;
  bool quantize = false;
  Granularity granularity = Granularity::per_block();
};

struct ModelSizeSpec {
  std::vector<ModelComponent> components;
  double bytes_hi = 2.0;
  double bytes_lo = 1.0;
  double scale_bytes = 4.0;  // per scale; amortised per element by the granularity's group size
};

// 1 − (Σ unquantized·bytes_hi + Σ quantized·(bytes_lo + scale bytes per element)) / (Σ all·bytes_hi).
// Scale bytes per element: PerBlock scale_bytes / (128·128); PerChannel / PerTensor are negligible
// without layer shapes (SPEC.md:625's amortised accounting).
double compression_ratio(const ModelSizeSpec& spec);

}  // namespace vlasim
