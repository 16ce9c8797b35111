// vlasim/packing/pack.hpp — padding-free sequence packing (reconstructed drop-in header).
//
// Reconstructed from proj/CMakeLists.txt:23 (src/packing/pack.cpp) and SPEC.md:419-454,
// 511-522.  pack_ffd / pack_greedy run on the GPU through the C-ABI
// (include/vlasim_cuda.h: vlasim_pack_ffd_cuda); results are bit-identical to the sequential
// reference semantics with the pinned order (length desc, id asc) — DESIGN.md §2.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "vlasim_cuda.h"

namespace vlasim {

// cu_seqlens(pack)[0] = 0, strictly increasing, last = fill <= capacity.
struct PackedSequence {
  std::int64_t capacity = 0;
  std::vector<std::int64_t> member_ids;
  std::vector<std::int64_t> member_lens;
  std::int64_t fill() const;
};

// SPEC.md:425-429.
struct PackingStats {
  std::int64_t bins_used = 0;
  double fill_rate = 0;
  double padding_rate_before = 0;
  double padding_rate_after = 0;
  double attention_flops_fixed = 0;
  double attention_flops_packed = 0;
};

// first-fit decreasing.  Oversize sample → ConfigError naming the id.
std::vector<PackedSequence> pack_ffd(std::span<const std::int64_t> lengths, std::int64_t capacity);

// streaming first fit in arrival order.
std::vector<PackedSequence> pack_greedy(std::span<const std::int64_t> lengths, std::int64_t capacity);

// prefix sums with a leading 0.
std::vector<std::int64_t> cu_seqlens(const PackedSequence& pack);

// SPEC.md:425-429 / 456-472 for a packing of `lengths` (pad_to: the fixed-length baseline).
PackingStats packing_stats(std::span<const std::int64_t> lengths, const std::vector<PackedSequence>& bins,
                           std::int64_t pad_to, std::int64_t head_dim);

// Device-resident packer for the hot path: owns the device outputs and workspace for batches of
// up to max_n samples; pack() is stream-ordered and allocation-free.
class GpuPacker {
 public:
  GpuPacker(std::int64_t max_n, std::int32_t capacity);
  ~GpuPacker();
  GpuPacker(const GpuPacker&) = delete;
  GpuPacker& operator=(const GpuPacker&) = delete;

  // d_lengths: device int32[n].  sync_check → synchronise and throw ConfigError on bad input.
  void pack(const std::int32_t* d_lengths, std::int64_t n, vlasim_stream_t stream, bool sync_check = true);
  // greedy arrival-order first fit; same outputs.
  void pack_greedy(const std::int32_t* d_lengths, std::int64_t n, vlasim_stream_t stream, bool sync_check = true);
  const vlasim_pack_out& out() const { return out_; }
  std::int32_t capacity() const { return capacity_; }

 private:
  std::int64_t max_n_;
  std::int32_t capacity_;
  vlasim_pack_out out_{};
  void* ws_ = nullptr;
  std::size_t ws_bytes_ = 0;
  void* block_ = nullptr;
};

}  // namespace vlasim
