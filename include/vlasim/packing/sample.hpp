// vlasim/packing/sample.hpp — per-sample token accounting (reconstructed drop-in header).
//
// The reference names src/packing/sample.cpp (proj/CMakeLists.txt:22) but ships no header;
// this interface is reconstructed from SPEC.md:413-417 and 456-491 in the
// reference's namespace and error convention (errors.hpp).  These are host-side scalar
// helpers; the hot path (pack.hpp, attention.hpp) runs on the GPU.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <string>
#include <string_view>

namespace vlasim {

// total_len = Σ view_lens + text_len; all >= 0; total_len >= 1.
struct SampleLen {
  std::int64_t id = 0;
  std::int64_t total_len = 0;
  std::map<std::string, std::int64_t> view_lens;
  std::int64_t text_len = 0;
};

// Validating constructor (ConfigError on a negative count or an empty sample).
SampleLen make_sample(std::int64_t id, const std::map<std::string, std::int64_t>& view_lens, std::int64_t text_len);

// SPEC.md:483-491 (π0.5 view pruning): view removed, total reduced; unknown view → ConfigError.
SampleLen prune_view(const SampleLen& sample, std::string_view view);

// 1 − Σl / (count · pad_to); pad_to >= max(lengths) else ConfigError.
double padding_rate(std::span<const std::int64_t> lengths, std::int64_t pad_to);

// max(lengths) of a non-empty batch (π0.5 dynamic padding).
std::int64_t dynamic_pad_length(std::span<const std::int64_t> lengths);

// fixed(pad_to) = count·c·pad_to²·d ; packed (no pad_to) = c·Σl²·d, c = 4 (one head, fwd).
double attention_flops(std::span<const std::int64_t> lengths, std::int64_t head_dim,
                       std::optional<std::int64_t> pad_to = std::nullopt, double c = 4.0);

}  // namespace vlasim
