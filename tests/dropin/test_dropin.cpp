// test_dropin.cpp — the reconstructed vlasim:: C++ API (libvlasim.so) exercised the way the
// reference's own tests would call it, on the SPEC's known-answer examples:
//   reference_attention  SPEC.md:498-500   (seq 1 → v row; q = 0 → column mean of v; random 8×4)
//   packed_attention     SPEC.md:507-509   (one segment ≡ reference; two segments ≡ concatenation;
//                                           masked-full-attention equivalence)
//   acceptance 8         SPEC.md:722       (200 random instances, lengths ≤ 64, dim ≤ 16)
//   pack_ffd / cu_seqlens / errors
// The fp64 scalar loops below are this test's own checker.  The GPU computes in bf16, so every
// attention comparison uses north_star's bf16 tolerance: max |gpu − ref| ≤ 2e-2 · max(1, max|ref|).
// Exit code 0 = all checks passed; the failing check is printed otherwise.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "vlasim/packing/attention.hpp"
#include "vlasim/packing/pack.hpp"
#include "vlasim/util/errors.hpp"

using vlasim::SmallTensor;

static int failures = 0;
#define CHECK(cond, ...)                         \
  do {                                           \
    if (!(cond)) {                               \
      std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      std::fprintf(stderr, __VA_ARGS__);         \
      std::fprintf(stderr, "\n");                \
      ++failures;                                \
    }                                            \
  } while (0)

static SmallTensor rand_tensor(std::mt19937_64& g, std::int64_t r, std::int64_t c, double scale = 1.0) {
  std::normal_distribution<double> n(0.0, scale);
  SmallTensor t{r, c, std::vector<double>(std::size_t(r * c))};
  for (auto& x : t.data) x = n(g);
  return t;
}

// fp64 scalar loop: softmax(q kᵀ/√d) v over rows [s, e), with an optional block-diagonal mask
// given by cu (masked full attention over all rows when cu has the segments).
static SmallTensor loop_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v,
                                  const std::vector<std::int64_t>& cu) {
  const std::int64_t T = q.rows, d = q.cols;
  SmallTensor o{T, d, std::vector<double>(std::size_t(T * d), 0.0)};
  std::vector<double> p(static_cast<std::size_t>(T));
  for (std::int64_t i = 0; i < T; ++i) {
    std::size_t seg = 0;
    while (cu[seg + 1] <= i) ++seg;
    double mx = -INFINITY;
    for (std::int64_t j = 0; j < T; ++j) {
      const bool vis = j >= cu[seg] && j < cu[seg + 1];  // explicit block-diagonal mask
      if (!vis) {
        p[j] = -INFINITY;
        continue;
      }
      double s = 0;
      for (std::int64_t c = 0; c < d; ++c) s += q.at(i, c) * k.at(j, c);
      p[j] = s / std::sqrt(double(d));
      mx = std::max(mx, p[j]);
    }
    double den = 0;
    for (std::int64_t j = 0; j < T; ++j) den += p[j] == -INFINITY ? 0.0 : std::exp(p[j] - mx);
    for (std::int64_t j = 0; j < T; ++j) {
      if (p[j] == -INFINITY) continue;
      const double w = std::exp(p[j] - mx) / den;
      for (std::int64_t c = 0; c < d; ++c) o.at(i, c) += w * v.at(j, c);
    }
  }
  return o;
}

static double rel_err(const SmallTensor& a, const SmallTensor& ref) {
  double mx = 0, mref = 0;
  for (std::size_t i = 0; i < ref.data.size(); ++i) {
    mx = std::max(mx, std::fabs(a.data[i] - ref.data[i]));
    mref = std::max(mref, std::fabs(ref.data[i]));
  }
  return mx / std::max(1.0, mref);
}

static SmallTensor rows(const SmallTensor& t, std::int64_t s, std::int64_t e) {
  SmallTensor r{e - s, t.cols, std::vector<double>(t.data.begin() + s * t.cols, t.data.begin() + e * t.cols)};
  return r;
}

int main() {
  constexpr double TOL = 2e-2;
  std::mt19937_64 g(42);

  // ---- reference_attention
  {
    SmallTensor q = rand_tensor(g, 1, 8), k = rand_tensor(g, 1, 8), v = rand_tensor(g, 1, 8);
    SmallTensor o = vlasim::reference_attention(q, k, v);
    CHECK(rel_err(o, v) < 4e-3, "seq length 1 must return the v row (err %g)", rel_err(o, v));
  }
  {
    SmallTensor q{6, 5, std::vector<double>(30, 0.0)}, k = rand_tensor(g, 6, 5), v = rand_tensor(g, 6, 5);
    SmallTensor mean{6, 5, std::vector<double>(30, 0.0)};
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 5; ++c)
        for (int j = 0; j < 6; ++j) mean.at(r, c) += v.at(j, c) / 6.0;
    SmallTensor o = vlasim::reference_attention(q, k, v);
    CHECK(rel_err(o, mean) < TOL, "q = 0 must give the column mean of v (err %g)", rel_err(o, mean));
  }
  {
    SmallTensor q = rand_tensor(g, 8, 4), k = rand_tensor(g, 8, 4), v = rand_tensor(g, 8, 4);
    SmallTensor o = vlasim::reference_attention(q, k, v);
    const double e = rel_err(o, loop_attention(q, k, v, {0, 8}));
    CHECK(e < TOL, "random 8x4 vs the scalar loop (err %g)", e);
  }

  // ---- packed_attention
  {
    SmallTensor q = rand_tensor(g, 37, 16), k = rand_tensor(g, 37, 16), v = rand_tensor(g, 37, 16);
    const std::int64_t cu1[2] = {0, 37};
    SmallTensor a = vlasim::packed_attention(q, k, v, cu1), b = vlasim::reference_attention(q, k, v);
    CHECK(a.data == b.data, "one segment must equal reference_attention");
  }
  {
    SmallTensor q = rand_tensor(g, 50, 12), k = rand_tensor(g, 50, 12), v = rand_tensor(g, 50, 12);
    const std::int64_t cu2[3] = {0, 21, 50};
    SmallTensor p = vlasim::packed_attention(q, k, v, cu2);
    SmallTensor r0 = vlasim::reference_attention(rows(q, 0, 21), rows(k, 0, 21), rows(v, 0, 21));
    SmallTensor r1 = vlasim::reference_attention(rows(q, 21, 50), rows(k, 21, 50), rows(v, 21, 50));
    std::vector<double> cat = r0.data;
    cat.insert(cat.end(), r1.data.begin(), r1.data.end());
    CHECK(p.data == cat, "two segments must equal the concatenation of the per-segment outputs (bit for bit)");
    const double e = rel_err(p, loop_attention(q, k, v, {0, 21, 50}));
    CHECK(e < TOL, "two segments vs the masked full attention (err %g)", e);
  }
  // model_dim coverage: every width 1..256 class boundary (zero-padded to 64 / 128 / 256 on the device)
  for (std::int64_t d : {1, 3, 16, 63, 64, 65, 100, 128, 129, 200, 255, 256}) {
    SmallTensor q = rand_tensor(g, 40, d), k = rand_tensor(g, 40, d), v = rand_tensor(g, 40, d);
    const std::int64_t cu[3] = {0, 15, 40};
    const double e = rel_err(vlasim::packed_attention(q, k, v, cu), loop_attention(q, k, v, {0, 15, 40}));
    CHECK(e < TOL, "model_dim %lld (err %g)", (long long)d, e);
  }
  // acceptance 8: 200 random instances, lengths <= 64, dim <= 16
  {
    std::uniform_int_distribution<int> nseg(1, 6), len(1, 64), dim(1, 16);
    double worst = 0;
    for (int inst = 0; inst < 200; ++inst) {
      const int m = nseg(g), d = dim(g);
      std::vector<std::int64_t> cu{0};
      for (int s = 0; s < m; ++s) cu.push_back(cu.back() + len(g));
      SmallTensor q = rand_tensor(g, cu.back(), d), k = rand_tensor(g, cu.back(), d), v = rand_tensor(g, cu.back(), d);
      worst = std::max(worst, rel_err(vlasim::packed_attention(q, k, v, cu), loop_attention(q, k, v, cu)));
    }
    CHECK(worst < TOL, "acceptance 8: worst error over 200 instances %g", worst);
    std::printf("acceptance 8: 200 instances, worst bf16 error %.3g (tolerance %.0e)\n", worst, TOL);
  }
  // errors: inconsistent cu_seqlens and model_dim beyond one head are ConfigError (errors.hpp:8)
  {
    SmallTensor q = rand_tensor(g, 10, 8);
    const std::int64_t bad[2] = {0, 9};
    bool thrown = false;
    try {
      vlasim::packed_attention(q, q, q, bad);
    } catch (const vlasim::ConfigError&) {
      thrown = true;
    }
    CHECK(thrown, "cu_seqlens inconsistent with the tensors must throw ConfigError");
    SmallTensor w = rand_tensor(g, 4, 300);
    thrown = false;
    try {
      vlasim::reference_attention(w, w, w);
    } catch (const vlasim::ConfigError&) {
      thrown = true;
    }
    CHECK(thrown, "model_dim 300 must throw ConfigError");
  }

  // ---- pack_ffd / cu_seqlens
  {
    const std::int64_t L[5] = {6, 5, 4, 3, 2};
    auto bins = vlasim::pack_ffd(L, 8);
    CHECK(bins.size() == 3, "FFD [6,5,4,3,2] cap 8 must use 3 bins");
    if (bins.size() == 3) {
      CHECK((bins[0].member_lens == std::vector<std::int64_t>{6, 2}), "bin 0 = {6,2}");
      CHECK((bins[1].member_lens == std::vector<std::int64_t>{5, 3}), "bin 1 = {5,3}");
      CHECK((bins[2].member_lens == std::vector<std::int64_t>{4}), "bin 2 = {4}");
      CHECK((vlasim::cu_seqlens(bins[0]) == std::vector<std::int64_t>{0, 6, 8}), "cu_seqlens of {6,2}");
    }
    const std::int64_t over[3] = {3, 9, 2};
    bool thrown = false;
    try {
      vlasim::pack_ffd(over, 8);
    } catch (const vlasim::ConfigError& e) {
      thrown = std::string(e.what()).find("id 1") != std::string::npos;
    }
    CHECK(thrown, "oversize sample must throw ConfigError naming id 1 (SPEC.md:441)");
  }

  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("drop-in C++ API: all SPEC known-answer checks passed\n");
  return 0;
}
