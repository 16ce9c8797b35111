// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product path.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this code, and only as the checker / the timed CPU
// baseline.  The product (paper_2603_11101_b200/) never links or calls it.
//
// CPU restatement (C++20) of the reference's packing + attention semantics.
// The reference ships no implementation: its behavioural contract
// is /root/reference/SPEC.md, and every function below cites the SPEC lines it
// follows.  Pinning: every SPEC example is a known-answer
// test in tests/test_oracle.py; rng is pinned against the reference's own
// rng.hpp compiled under oracle/_ref/.
// ============================================================================
#pragma once

#include <cstdint>
#include <map>
#include <span>
#include <string>
#include <vector>

namespace vlasim::oracle {

// ---------------------------------------------------------------- sample
struct SampleLen {
  std::int64_t id = 0;
  std::int64_t total_len = 0;
  std::map<std::string, std::int64_t> view_lens;
  std::int64_t text_len = 0;
};
SampleLen make_sample(std::int64_t id, const std::map<std::string, std::int64_t>& views, std::int64_t text_len);
SampleLen prune_view(const SampleLen& s, const std::string& view);
double padding_rate(std::span<const std::int64_t> lengths, std::int64_t pad_to);
std::int64_t dynamic_pad_length(std::span<const std::int64_t> lengths);
// fixed = count·c·pad_to²·d ; packed = c·Σl²·d   (c = 4 per head, fwd)
double attention_flops_fixed(std::span<const std::int64_t> lengths, std::int64_t pad_to, std::int64_t d, double c = 4);
double attention_flops_packed(std::span<const std::int64_t> lengths, std::int64_t d, double c = 4);

// ---------------------------------------------------------------- pack
struct PackedSequence {
  std::int64_t capacity = 0;
  std::vector<std::int64_t> member_ids;
  std::vector<std::int64_t> member_lens;
  std::int64_t fill() const;
};
// First-fit decreasing, order (len desc, id asc), first fit by lowest bin index.
// naive=true scans bins linearly (the literal restatement); false uses a max
// segment tree over bin remainders (same first-fit choice, O(log B)).
std::vector<PackedSequence> pack_ffd(std::span<const std::int64_t> lengths, std::int64_t capacity, bool naive = true);
// Greedy first-fit in arrival order.
std::vector<PackedSequence> pack_greedy(std::span<const std::int64_t> lengths, std::int64_t capacity);
std::vector<std::int64_t> cu_seqlens(const PackedSequence& p);

struct PackingStats {
  std::int64_t bins_used = 0;
  double fill_rate = 0, padding_rate_before = 0, padding_rate_after = 0;
  double attention_flops_fixed = 0, attention_flops_packed = 0;
};
PackingStats packing_stats(std::span<const std::int64_t> lengths, const std::vector<PackedSequence>& bins,
                           std::int64_t pad_to, std::int64_t d);

// ---------------------------------------------------------------- attention
struct SmallTensor {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> data;
  double& at(std::int64_t r, std::int64_t c) { return data[r * cols + c]; }
  double at(std::int64_t r, std::int64_t c) const { return data[r * cols + c]; }
};
SmallTensor reference_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v);
SmallTensor packed_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v,
                             std::span<const std::int64_t> cu_seqlens);
// Explicit block-diagonal masked full attention (the mask-based oracle).
SmallTensor masked_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v,
                             std::span<const std::int64_t> cu_seqlens);

// ---------------------------------------------------------------- E4M3
std::vector<double> e4m3_values();                // all finite non-negative representable values, ascending
double e4m3_rne(double x);                        // RNE projection onto the set, saturating to ±448
std::uint8_t e4m3_encode(double x);               // code byte of e4m3_rne(x)
std::uint8_t e4m3_encode_ratio(double num, double den);  // code of RNE(num / den), exact (den > 0)
double e4m3_decode(std::uint8_t code);

}  // namespace vlasim::oracle
