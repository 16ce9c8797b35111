// vlasim/quant/quantize.hpp — E4M3 quantization at PerTensor / PerChannel(axis) / PerBlock(128×128)
// granularity (reconstructed drop-in header for proj/CMakeLists.txt:20 src/quant/quantize.cpp;
// contract SPEC.md:550-606).  quantize / dequantize / quant_error run on the GPU through the C-ABI
// (vlasim_fp8_quantize_cuda & co., include/vlasim_cuda.h).  The device holds the tensor at fp32: the
// codes are the exact RNE E4M3 codes of |x|·448/amax for fp32-representable values.
//
// QuantizedTensor binary form (little endian): "VLQ1", uint8 granularity (0 tensor, 1 channel,
// 2 block), int32 axis, uint32 ndim, int64 dims[ndim], uint64 nscales, float32 scales[nscales],
// uint8 codes[Π dims].
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "vlasim/quant/fp8.hpp"
#include "vlasim/quant/tensor.hpp"

namespace vlasim {

enum class GranularityKind : std::uint8_t { PerTensor = 0, PerChannel = 1, PerBlock = 2 };

struct Granularity {
  GranularityKind kind = GranularityKind::PerBlock;
  int axis = 0;  // PerChannel only
  static Granularity per_tensor() { return {GranularityKind::PerTensor, 0}; }
  static Granularity per_channel(int axis) { return {GranularityKind::PerChannel, axis}; }
  static Granularity per_block() { return {GranularityKind::PerBlock, 0}; }
  std::string name() const;  // "tensor", "channel:<axis>", "block"
  static Granularity parse(const std::string& s);  // the same spellings; else ConfigError
};

struct QuantizedTensor {
  std::vector<std::uint8_t> codes;          // E4M3 bytes, row-major like the input
  std::vector<float> scales;                // per group (scales_shape)
  std::vector<std::int64_t> shape;          // original shape
  std::vector<std::int64_t> scales_shape;
  Granularity granularity;
};

// blocks tiling the last two dims, edge blocks truncated.
struct BlockExtent {
  std::int64_t row0, rows, col0, cols;
};
std::vector<BlockExtent> block_partition(const std::vector<std::int64_t>& shape, std::int64_t block_rows = 128,
                                         std::int64_t block_cols = 128);

QuantizedTensor quantize(const Tensor& t, const Granularity& g, const Fp8Format& fmt = {});
Tensor dequantize(const QuantizedTensor& qt);

struct QuantErrorMetrics {
  double max_rel = 0;  // over elements in E4M3's normal range
  double mse = 0;
  std::vector<float> group_max_rel;  // per group (scales_shape)
  std::vector<double> group_mse;
};
QuantErrorMetrics quant_error(const Tensor& original, const QuantizedTensor& qt);

void write_quantized(const std::string& path, const QuantizedTensor& qt);
QuantizedTensor read_quantized(const std::string& path);

}  // namespace vlasim
