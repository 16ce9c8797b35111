// vlasim/quant/fp8.hpp — FP8 E4M3 format (reconstructed drop-in header for proj/CMakeLists.txt:18
// src/quant/fp8.cpp; the E4M3 choice SPEC.md:624).
#pragma once

#include <cstdint>

namespace vlasim {

struct Fp8Format {
  int exponent_bits = 4;
  int mantissa_bits = 3;
  int bias = 7;
  double max_normal = 448.0;  // subnormals supported, no infinities, 0x7F / 0xFF are NaN
};

// Value of an E4M3 code byte.
double fp8_decode(std::uint8_t code);

}  // namespace vlasim
