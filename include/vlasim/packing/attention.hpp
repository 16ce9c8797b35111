// vlasim/packing/attention.hpp — packed (block-diagonal) attention (reconstructed drop-in header).
//
// Reconstructed from proj/CMakeLists.txt:24 (src/packing/attention.cpp) and SPEC.md:431-434,
// 493-509.  The reference defines the op on high-precision host tensors; the
// drop-in runs the hand-written sm_100a kernels in bf16 (north_star tolerance: max-abs 2e-2 vs
// the fp32/fp64 reference), multi-head as the reference's looped single-head op.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "vlasim_cuda.h"

namespace vlasim {

// dense (sequence, model_dim) real tensor, row-major.
struct SmallTensor {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> data;
  double& at(std::int64_t r, std::int64_t c) { return data[r * cols + c]; }
  double at(std::int64_t r, std::int64_t c) const { return data[r * cols + c]; }
};

// softmax(q·kᵀ/√d)·v, one head (= packed_attention with one segment).
// model_dim (cols) 1..256: columns are zero-padded to the kernels' head_dim on the device.
SmallTensor reference_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v);

// per-segment attention over a packed stream; no cross-segment interaction.
SmallTensor packed_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v,
                             std::span<const std::int64_t> cu_seqlens);

// Device-level multi-head varlen attention over caller-owned device buffers (the hot path).
// Layout as in vlasim_cuda.h: q/o [T,H,d], k/v [T,Hkv,d] bf16, lse [H,T] fp32.
class VarlenAttention {
 public:
  VarlenAttention() = default;
  ~VarlenAttention();
  VarlenAttention(const VarlenAttention&) = delete;
  VarlenAttention& operator=(const VarlenAttention&) = delete;

  void forward(const vlasim_attn_args& args, vlasim_stream_t stream);
  void backward(const vlasim_attn_args& args, const vlasim_attn_grads& grads, vlasim_stream_t stream);

 private:
  void* ws_ = nullptr;
  std::size_t ws_bytes_ = 0;
  void reserve(std::size_t bytes);
};

}  // namespace vlasim
