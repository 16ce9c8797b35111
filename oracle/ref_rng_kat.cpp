// ORACLE — TEST INFRASTRUCTURE ONLY.
// Known-answer generator for the seeding API (rng.hpp).  Compiled twice by
// oracle/Makefile: once against the reference's own header
// (/root/reference/proj/include/vlasim/util/rng.hpp → oracle/_ref/ref_rng_kat) and once
// against this repo's restatement (include/vlasim/util/rng.hpp → oracle/rng_kat).
// tests/test_rng.py compares both outputs and the committed tests/golden/rng_kat.json.
#include <cstdio>
#include <cstdint>

#include "vlasim/util/rng.hpp"

int main() {
  using namespace vlasim;
  std::printf("{\n");
  std::printf("  \"splitmix64_0\": \"%016llx\",\n", (unsigned long long)splitmix64(0));
  std::printf("  \"splitmix64_1\": \"%016llx\",\n", (unsigned long long)splitmix64(1));
  std::printf("  \"derive_42_lengths_0\": \"%016llx\",\n", (unsigned long long)derive_seed(42, "lengths", 0));
  std::printf("  \"derive_42_lengths_1\": \"%016llx\",\n", (unsigned long long)derive_seed(42, "lengths", 1));
  std::printf("  \"derive_42_empty_0\": \"%016llx\",\n", (unsigned long long)derive_seed(42, "", 0));
  std::printf("  \"derive_7_q_3\": \"%016llx\",\n", (unsigned long long)derive_seed(7, "q", 3));
  {
    auto r = make_rng(42, "lengths", 0);
    std::printf("  \"uniform_int_42_lengths_16_512\": [");
    for (int i = 0; i < 64; ++i) std::printf("%s%lld", i ? ", " : "", (long long)uniform_int(r, 16, 512));
    std::printf("],\n");
  }
  {
    auto r = make_rng(7, "lengths", 0);
    std::printf("  \"uniform_int_7_lengths_16_512\": [");
    for (int i = 0; i < 16; ++i) std::printf("%s%lld", i ? ", " : "", (long long)uniform_int(r, 16, 512));
    std::printf("],\n");
  }
  {
    auto r = make_rng(42, "q", 0);
    std::printf("  \"uniform01_42_q_0\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", uniform01(r));
    std::printf("],\n");
  }
  {
    auto r = make_rng(42, "range", 5);
    std::printf("  \"uniform_range_42_range_5\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", uniform_range(r, -3.5, 11.25));
    std::printf("],\n");
  }
  {
    auto r = make_rng(123, "edge", 0);
    std::printf("  \"uniform_int_123_edge_0_0\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%lld", i ? ", " : "", (long long)uniform_int(r, 0, 0));
    std::printf("],\n");
  }
  {
    auto r = make_rng(42, "raw", 9);
    std::printf("  \"mt_raw_42_raw_9\": [");
    for (int i = 0; i < 4; ++i) std::printf("%s\"%016llx\"", i ? ", " : "", (unsigned long long)r());
    std::printf("]\n");
  }
  std::printf("}\n");
  return 0;
}
