// vlasim/quant/tensor.hpp — dense high-precision tensors and their file forms (reconstructed drop-in
// header for proj/CMakeLists.txt:19 src/quant/tensor.cpp; "Tensor I/O: flat binary
// (shape header + row-major high-precision values) and a text form for small fixtures").
//
// Binary form (little endian): "VLT1", uint32 ndim, int64 dims[ndim], float64 values[Π dims].
// Text form: first non-comment line = the dims, then the values in row-major order ('#' comments).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace vlasim {

struct Tensor {
  std::vector<std::int64_t> shape;
  std::vector<double> data;  // row-major
  std::int64_t numel() const;
};

Tensor read_tensor(const std::string& path);  // binary or text form (by magic)
void write_tensor(const std::string& path, const Tensor& t);
Tensor read_tensor_text(const std::string& path);

}  // namespace vlasim
