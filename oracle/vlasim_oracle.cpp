// ORACLE — TEST INFRASTRUCTURE ONLY (see vlasim_oracle.hpp header).
// CPU restatement of /root/reference/SPEC.md:408-537 (seq-packing) and the E4M3
// part of SPEC.md:539-627 (quantizer), plus multi-head / masked / backward
// extensions used as the numerics checker for the GPU kernels.
#include "vlasim_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <thread>

#include "vlasim/util/errors.hpp"
#include "vlasim/util/rng.hpp"

namespace vlasim::oracle {

// ============================================================ sample
SampleLen make_sample(std::int64_t id, const std::map<std::string, std::int64_t>& views, std::int64_t text_len) {
  // SPEC.md:416 invariants: all >= 0, total = Σviews + text >= 1
  if (text_len < 0) throw ConfigError("negative text length for sample " + std::to_string(id));
  SampleLen s;
  s.id = id;
  s.view_lens = views;
  s.text_len = text_len;
  s.total_len = text_len;
  for (const auto& [name, n] : views) {
    if (n < 0) throw ConfigError("negative view length '" + name + "' for sample " + std::to_string(id));
    s.total_len += n;
  }
  if (s.total_len < 1) throw ConfigError("sample " + std::to_string(id) + " has no tokens");
  return s;
}

SampleLen prune_view(const SampleLen& s, const std::string& view) {
  // view removed, total reduced by its count; unknown view → error
  auto it = s.view_lens.find(view);
  if (it == s.view_lens.end())
    throw ConfigError("prune_view: sample " + std::to_string(s.id) + " has no view '" + view + "'");
  SampleLen r = s;
  r.total_len -= it->second;
  r.view_lens.erase(view);
  return r;
}

double padding_rate(std::span<const std::int64_t> lengths, std::int64_t pad_to) {
  // pre pad_to >= max(lengths); 1 - Σl / (count·pad_to)
  if (lengths.empty()) throw ConfigError("padding_rate: empty batch");
  std::int64_t sum = 0, mx = 0;
  for (auto l : lengths) {
    sum += l;
    mx = std::max(mx, l);
  }
  if (pad_to < mx) throw ConfigError("padding_rate: pad_to below the longest sample");
  return 1.0 - static_cast<double>(sum) / (static_cast<double>(lengths.size()) * static_cast<double>(pad_to));
}

std::int64_t dynamic_pad_length(std::span<const std::int64_t> lengths) {
  // max of the batch
  if (lengths.empty()) throw ConfigError("dynamic_pad_length: empty batch");
  return *std::max_element(lengths.begin(), lengths.end());
}

double attention_flops_fixed(std::span<const std::int64_t> lengths, std::int64_t pad_to, std::int64_t d, double c) {
  // SPEC.md:468 fixed: count·c·pad_to²·d
  for (auto l : lengths)
    if (l > pad_to) throw ConfigError("attention_flops: length above pad_to");
  return static_cast<double>(lengths.size()) * c * static_cast<double>(pad_to) * static_cast<double>(pad_to) *
         static_cast<double>(d);
}

double attention_flops_packed(std::span<const std::int64_t> lengths, std::int64_t d, double c) {
  // SPEC.md:468 packed: c·Σl²·d
  double s = 0;
  for (auto l : lengths) s += static_cast<double>(l) * static_cast<double>(l);
  return c * s * static_cast<double>(d);
}

// ============================================================ pack
std::int64_t PackedSequence::fill() const {
  return std::accumulate(member_lens.begin(), member_lens.end(), std::int64_t{0});
}

static void validate_lengths(std::span<const std::int64_t> lengths, std::int64_t capacity) {
  // every length <= capacity, else oversize error naming the id
  if (capacity < 1) throw ConfigError("capacity must be >= 1");
  for (std::size_t i = 0; i < lengths.size(); ++i) {
    if (lengths[i] > capacity)
      throw ConfigError("oversize sample id " + std::to_string(i) + ": length " + std::to_string(lengths[i]) +
                        " > capacity " + std::to_string(capacity));
    if (lengths[i] < 1) throw ConfigError("empty sample id " + std::to_string(i));
  }
}

namespace {
// Max segment tree over bin remainders; first_fit returns the lowest index with rem >= L.
struct FirstFitTree {
  std::int64_t size = 1;
  std::vector<std::int64_t> t;
  explicit FirstFitTree(std::int64_t n) {
    while (size < n) size <<= 1;
    t.assign(2 * size, -1);
  }
  void set(std::int64_t i, std::int64_t v) {
    i += size;
    t[i] = v;
    for (i >>= 1; i; i >>= 1) t[i] = std::max(t[2 * i], t[2 * i + 1]);
  }
  std::int64_t first_fit(std::int64_t L) const {
    if (t[1] < L) return -1;
    std::int64_t i = 1;
    while (i < size) i = (t[2 * i] >= L) ? 2 * i : 2 * i + 1;
    return i - size;
  }
};

std::vector<PackedSequence> first_fit(std::span<const std::int64_t> lengths, std::int64_t capacity,
                                      const std::vector<std::int64_t>& order, bool naive) {
  std::vector<PackedSequence> bins;
  std::vector<std::int64_t> rem;
  FirstFitTree tree(naive ? 1 : static_cast<std::int64_t>(std::max<std::size_t>(1, lengths.size())));
  for (std::int64_t id : order) {
    const std::int64_t L = lengths[id];
    std::int64_t b = -1;
    if (naive) {
      for (std::size_t j = 0; j < rem.size(); ++j)
        if (rem[j] >= L) {
          b = static_cast<std::int64_t>(j);
          break;
        }
    } else {
      b = tree.first_fit(L);
    }
    if (b < 0) {
      b = static_cast<std::int64_t>(bins.size());
      bins.push_back(PackedSequence{capacity, {}, {}});
      rem.push_back(capacity);
    }
    bins[b].member_ids.push_back(id);
    bins[b].member_lens.push_back(L);
    rem[b] -= L;
    if (!naive) tree.set(b, rem[b]);
  }
  return bins;
}
}  // namespace

std::vector<PackedSequence> pack_ffd(std::span<const std::int64_t> lengths, std::int64_t capacity, bool naive) {
  // SPEC.md:437-445 + design decision SPEC.md:519; tiebreak pinned to (len desc, id asc)
  validate_lengths(lengths, capacity);
  std::vector<std::int64_t> order(lengths.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](std::int64_t a, std::int64_t b) { return lengths[a] > lengths[b]; });
  return first_fit(lengths, capacity, order, naive);
}

std::vector<PackedSequence> pack_greedy(std::span<const std::int64_t> lengths, std::int64_t capacity) {
  // SPEC.md:519 "greedy in-arrival-order variant for streaming use": first fit, no sort
  validate_lengths(lengths, capacity);
  std::vector<std::int64_t> order(lengths.size());
  std::iota(order.begin(), order.end(), 0);
  return first_fit(lengths, capacity, order, lengths.size() <= 4096);
}

std::vector<std::int64_t> cu_seqlens(const PackedSequence& p) {
  // pack nonempty; prefix sums with leading 0
  if (p.member_lens.empty()) throw ConfigError("cu_seqlens: empty pack");
  std::vector<std::int64_t> cu(p.member_lens.size() + 1, 0);
  for (std::size_t i = 0; i < p.member_lens.size(); ++i) cu[i + 1] = cu[i] + p.member_lens[i];
  return cu;
}

PackingStats packing_stats(std::span<const std::int64_t> lengths, const std::vector<PackedSequence>& bins,
                           std::int64_t pad_to, std::int64_t d) {
  // SPEC.md:425-429; "after" padding = unused capacity of the bins
  PackingStats s;
  s.bins_used = static_cast<std::int64_t>(bins.size());
  std::int64_t sum = std::accumulate(lengths.begin(), lengths.end(), std::int64_t{0});
  const std::int64_t cap = bins.empty() ? 1 : bins[0].capacity;
  s.fill_rate = static_cast<double>(sum) / (static_cast<double>(s.bins_used) * static_cast<double>(cap));
  s.padding_rate_before = padding_rate(lengths, pad_to);
  s.padding_rate_after = 1.0 - s.fill_rate;
  s.attention_flops_fixed = attention_flops_fixed(lengths, pad_to, d);
  s.attention_flops_packed = attention_flops_packed(lengths, d);
  return s;
}

// ============================================================ attention (fp64, SPEC semantics)
SmallTensor reference_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v) {
  // single head, softmax(q·kᵀ/√d)·v in high precision
  if (q.cols != k.cols || k.rows != v.rows || q.rows < 0)
    throw ConfigError("reference_attention: shape mismatch");
  const std::int64_t n = q.rows, m = k.rows, d = q.cols, dv = v.cols;
  const double scale = 1.0 / std::sqrt(static_cast<double>(d));
  SmallTensor o{n, dv, std::vector<double>(static_cast<std::size_t>(n * dv), 0.0)};
  std::vector<double> s(static_cast<std::size_t>(m));
  for (std::int64_t i = 0; i < n; ++i) {
    double mx = -std::numeric_limits<double>::infinity();
    for (std::int64_t j = 0; j < m; ++j) {
      double acc = 0;
      for (std::int64_t c = 0; c < d; ++c) acc += q.at(i, c) * k.at(j, c);
      s[j] = acc * scale;
      mx = std::max(mx, s[j]);
    }
    double den = 0;
    for (std::int64_t j = 0; j < m; ++j) den += (s[j] = std::exp(s[j] - mx));
    for (std::int64_t j = 0; j < m; ++j) {
      const double p = s[j] / den;
      for (std::int64_t c = 0; c < dv; ++c) o.at(i, c) += p * v.at(j, c);
    }
  }
  return o;
}

static SmallTensor slice_rows(const SmallTensor& t, std::int64_t r0, std::int64_t r1) {
  SmallTensor s{r1 - r0, t.cols, {}};
  s.data.assign(t.data.begin() + r0 * t.cols, t.data.begin() + r1 * t.cols);
  return s;
}

static void check_cu(std::span<const std::int64_t> cu, std::int64_t rows) {
  // SPEC.md:422 / 504: cu[0] = 0, strictly increasing, last = rows
  if (cu.size() < 2 || cu.front() != 0 || cu.back() != rows)
    throw ConfigError("packed_attention: cu_seqlens inconsistent with tensors");
  for (std::size_t i = 1; i < cu.size(); ++i)
    if (cu[i] <= cu[i - 1]) throw ConfigError("packed_attention: cu_seqlens not strictly increasing");
}

SmallTensor packed_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v,
                             std::span<const std::int64_t> cu) {
  // per-segment reference_attention, concatenated; no cross-segment terms
  if (q.rows != k.rows || k.rows != v.rows) throw ConfigError("packed_attention: row mismatch");
  check_cu(cu, q.rows);
  SmallTensor o{q.rows, v.cols, std::vector<double>(static_cast<std::size_t>(q.rows * v.cols))};
  for (std::size_t s = 0; s + 1 < cu.size(); ++s) {
    SmallTensor os = reference_attention(slice_rows(q, cu[s], cu[s + 1]), slice_rows(k, cu[s], cu[s + 1]),
                                         slice_rows(v, cu[s], cu[s + 1]));
    std::copy(os.data.begin(), os.data.end(), o.data.begin() + cu[s] * v.cols);
  }
  return o;
}

SmallTensor masked_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v,
                             std::span<const std::int64_t> cu) {
  // full attention with an explicit block-diagonal mask (−inf off-block)
  check_cu(cu, q.rows);
  const std::int64_t n = q.rows, d = q.cols, dv = v.cols;
  std::vector<std::int64_t> seg(static_cast<std::size_t>(n));
  for (std::size_t s = 0; s + 1 < cu.size(); ++s)
    for (std::int64_t t = cu[s]; t < cu[s + 1]; ++t) seg[t] = static_cast<std::int64_t>(s);
  const double scale = 1.0 / std::sqrt(static_cast<double>(d));
  SmallTensor o{n, dv, std::vector<double>(static_cast<std::size_t>(n * dv), 0.0)};
  std::vector<double> s(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) {
    double mx = -std::numeric_limits<double>::infinity();
    for (std::int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (std::int64_t c = 0; c < d; ++c) acc += q.at(i, c) * k.at(j, c);
      s[j] = (seg[i] == seg[j]) ? acc * scale : -std::numeric_limits<double>::infinity();
      mx = std::max(mx, s[j]);
    }
    double den = 0;
    for (std::int64_t j = 0; j < n; ++j) den += (s[j] = std::exp(s[j] - mx));
    for (std::int64_t j = 0; j < n; ++j)
      for (std::int64_t c = 0; c < dv; ++c) o.at(i, c) += (s[j] / den) * v.at(j, c);
  }
  return o;
}

// ============================================================ E4M3
std::vector<double> e4m3_values() {
  // 4 exponent bits, 3 mantissa bits, bias 7, subnormals, max 448, no inf;
  // exponent 15 / mantissa 7 is NaN and excluded.
  std::vector<double> v;
  for (int e = 0; e < 16; ++e)
    for (int m = 0; m < 8; ++m) {
      if (e == 15 && m == 7) continue;
      v.push_back(e == 0 ? std::ldexp(m / 8.0, -6) : std::ldexp(1.0 + m / 8.0, e - 7));
    }
  return v;  // ascending by construction
}

std::uint8_t e4m3_encode(double x) {
  // round-to-nearest-even onto the representable set, saturating.
  if (std::isnan(x)) throw ConfigError("e4m3: non-finite input");
  static const std::vector<double> vals = e4m3_values();  // index i ↔ code i (e = i>>3, m = i&7)
  const std::uint8_t sign = std::signbit(x) ? 0x80 : 0x00;
  const double a = std::fabs(x);
  if (a >= 448.0) return sign | 0x7E;
  auto it = std::lower_bound(vals.begin(), vals.end(), a);  // first >= a
  std::size_t hi = static_cast<std::size_t>(it - vals.begin());
  if (vals[hi] == a) return sign | static_cast<std::uint8_t>(hi);
  const std::size_t lo = hi - 1;
  const double dlo = a - vals[lo], dhi = vals[hi] - a;
  std::size_t pick;
  if (dlo < dhi) pick = lo;
  else if (dhi < dlo) pick = hi;
  else pick = (lo % 2 == 0) ? lo : hi;  // tie → even mantissa (code LSB 0)
  return sign | static_cast<std::uint8_t>(pick);
}

double e4m3_rne(double x) { return e4m3_decode(e4m3_encode(x)); }

// SPEC.md:583 with the REAL quotient: code of RNE(num / den) for den > 0 without forming the quotient.
// The exhaustive nearest-value search over the representable set ("oracle is exhaustive
// nearest-value search") decided by exact comparisons: |num| against mid_i · den for the midpoints
// mid_i = (v_i + v_{i+1}) / 2 of consecutive representable values.  Callers pass num = x · 448 and
// den = amax with x, amax fp32: both products are exact in double (≤ 27 and ≤ 29 significant bits).
std::uint8_t e4m3_encode_ratio(double num, double den) {
  if (!std::isfinite(num) || !std::isfinite(den) || !(den > 0)) throw ConfigError("e4m3: non-finite input");
  static const std::vector<double> vals = e4m3_values();
  const std::uint8_t sign = std::signbit(num) ? 0x80 : 0x00;
  const double a = std::fabs(num);
  for (std::size_t i = 0; i + 1 < vals.size(); ++i) {
    const double m = 0.5 * (vals[i] + vals[i + 1]);  // exact (≤ 5 significant bits)
    const double b = m * den;                         // exact
    if (a < b) return sign | static_cast<std::uint8_t>(i);
    if (a == b) return sign | static_cast<std::uint8_t>(i % 2 == 0 ? i : i + 1);  // tie → even mantissa
  }
  return sign | 0x7E;  // above the last midpoint: 448 (saturating)
}

double e4m3_decode(std::uint8_t code) {
  static const std::vector<double> vals = e4m3_values();
  const std::uint8_t mag = code & 0x7F;
  if (mag == 0x7F) return std::numeric_limits<double>::quiet_NaN();
  const double v = vals[mag];
  return (code & 0x80) ? -v : v;
}

}  // namespace vlasim::oracle

// ============================================================================
// Multi-head varlen attention (fwd + closed-form bwd), templated on the compute
// type: double = the numerics checker; float = the timed CPU baseline.
// Layout mirrors the GPU path: q/o/dq [T,H,d], k/v/dk/dv [T,Hkv,d], lse [H,T].
// Mask (SPEC.md:496 is bidirectional; causal/prefix pinned in DESIGN.md §2):
//   key j of segment [s,e) visible to query t  iff  j - s < P  or  j <= t,
//   P = e - s (bidirectional), 0 (causal), prefix_len[seg] (prefix).
// ============================================================================
namespace {

struct MhaShape {
  std::int64_t T, H, Hkv, d;
  int mask;
  double scale;
};

inline std::int64_t seg_prefix(int mask, const std::int32_t* prefix, std::int64_t s, std::int64_t len) {
  if (mask == 0) return len;
  if (mask == 1) return 0;
  return std::min<std::int64_t>(len, std::max<std::int64_t>(0, prefix[s]));
}

template <typename T>
void run_parallel(std::int64_t items, int threads, const T& fn) {
  if (threads <= 1 || items <= 1) {
    for (std::int64_t i = 0; i < items; ++i) fn(i);
    return;
  }
  std::atomic<std::int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (std::int64_t i = next++; i < items; i = next++) fn(i);
    });
  for (auto& th : pool) th.join();
}

template <typename F>
inline F dot(const F* a, const F* b, std::int64_t n) {
  F acc = 0;
#pragma omp simd reduction(+ : acc)
  for (std::int64_t c = 0; c < n; ++c) acc += a[c] * b[c];
  return acc;
}

template <typename F>
void mha_fwd(const F* q, const F* k, const F* v, F* o, F* lse, const std::int32_t* cu, std::int64_t nseq,
             const std::int32_t* prefix, const MhaShape& sh, int threads) {
  const std::int64_t H = sh.H, Hkv = sh.Hkv, d = sh.d, grp = H / Hkv;
  run_parallel(nseq * H, threads, [&](std::int64_t item) {
    const std::int64_t s = item / H, h = item % H, kh = h / grp;
    const std::int64_t b = cu[s], e = cu[s + 1], len = e - b;
    const std::int64_t P = seg_prefix(sh.mask, prefix, s, len);
    std::vector<F> sc(static_cast<std::size_t>(len));
    std::vector<F> acc(static_cast<std::size_t>(d));
    for (std::int64_t t = b; t < e; ++t) {
      const F* qr = q + (t * H + h) * d;
      const std::int64_t hi = std::max<std::int64_t>(b + P, t + 1);  // visible keys [b, min(hi,e))
      const std::int64_t ke = std::min(hi, e);
      F mx = -std::numeric_limits<F>::infinity();
      for (std::int64_t j = b; j < ke; ++j) {
        sc[j - b] = dot(qr, k + (j * Hkv + kh) * d, d) * static_cast<F>(sh.scale);
        mx = std::max(mx, sc[j - b]);
      }
      F den = 0;
      for (std::int64_t j = b; j < ke; ++j) den += (sc[j - b] = std::exp(sc[j - b] - mx));
      std::fill(acc.begin(), acc.end(), F(0));
      for (std::int64_t j = b; j < ke; ++j) {
        const F p = sc[j - b] / den;
        const F* vr = v + (j * Hkv + kh) * d;
#pragma omp simd
        for (std::int64_t c = 0; c < d; ++c) acc[c] += p * vr[c];
      }
      std::copy(acc.begin(), acc.end(), o + (t * H + h) * d);
      if (lse) lse[h * sh.T + t] = mx + std::log(den);
    }
  });
}

template <typename F>
void mha_bwd(const F* q, const F* k, const F* v, const F* o, const F* dout, F* dq, F* dk, F* dv,
             const std::int32_t* cu, std::int64_t nseq, const std::int32_t* prefix, const MhaShape& sh, int threads) {
  // dV = Pᵀ dO ; dP = dO Vᵀ ; dS = P ∘ (dP − rowsum(dO ∘ O)) ; dQ = scale·dS K ; dK = scale·dSᵀ Q
  const std::int64_t H = sh.H, Hkv = sh.Hkv, d = sh.d, grp = H / Hkv;
  const F scale = static_cast<F>(sh.scale);
  run_parallel(nseq * Hkv, threads, [&](std::int64_t item) {
    const std::int64_t s = item / Hkv, kh = item % Hkv;
    const std::int64_t b = cu[s], e = cu[s + 1], len = e - b;
    const std::int64_t P = seg_prefix(sh.mask, prefix, s, len);
    std::vector<F> p(static_cast<std::size_t>(len)), dp(static_cast<std::size_t>(len));
    for (std::int64_t t = b; t < e; ++t)
      for (std::int64_t c = 0; c < d; ++c) {
        dk[(t * Hkv + kh) * d + c] = 0;
        dv[(t * Hkv + kh) * d + c] = 0;
      }
    for (std::int64_t h = kh * grp; h < (kh + 1) * grp; ++h) {
      for (std::int64_t t = b; t < e; ++t) {
        const F* qr = q + (t * H + h) * d;
        const F* dor = dout + (t * H + h) * d;
        const F* orow = o + (t * H + h) * d;
        const std::int64_t ke = std::min(std::max<std::int64_t>(b + P, t + 1), e);
        F mx = -std::numeric_limits<F>::infinity();
        for (std::int64_t j = b; j < ke; ++j) {
          p[j - b] = dot(qr, k + (j * Hkv + kh) * d, d) * scale;
          mx = std::max(mx, p[j - b]);
        }
        F den = 0;
        for (std::int64_t j = b; j < ke; ++j) den += (p[j - b] = std::exp(p[j - b] - mx));
        for (std::int64_t j = b; j < ke; ++j) p[j - b] /= den;
        const F D = dot(dor, orow, d);
        F* dqr = dq + (t * H + h) * d;
        for (std::int64_t c = 0; c < d; ++c) dqr[c] = 0;
        for (std::int64_t j = b; j < ke; ++j) {
          const F* kr = k + (j * Hkv + kh) * d;
          const F* vr = v + (j * Hkv + kh) * d;
          const F dpj = dot(dor, vr, d);
          const F ds = p[j - b] * (dpj - D);
          F* dvr = dv + (j * Hkv + kh) * d;
          F* dkr = dk + (j * Hkv + kh) * d;
#pragma omp simd
          for (std::int64_t c = 0; c < d; ++c) {
            dvr[c] += p[j - b] * dor[c];
            dkr[c] += scale * ds * qr[c];
            dqr[c] += scale * ds * kr[c];
          }
        }
      }
    }
  });
}

MhaShape make_shape(std::int64_t T, std::int64_t H, std::int64_t Hkv, std::int64_t d, int mask, double scale) {
  if (H < 1 || Hkv < 1 || H % Hkv || d < 1 || mask < 0 || mask > 2) throw vlasim::ConfigError("bad attention shape");
  return MhaShape{T, H, Hkv, d, mask, scale};
}

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const vlasim::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

void bins_to_arrays(const std::vector<vlasim::oracle::PackedSequence>& bins, std::int32_t* bin_of,
                    std::int32_t* slot, std::int32_t* tok_off, std::int32_t* num_bins) {
  for (std::size_t b = 0; b < bins.size(); ++b) {
    std::int64_t off = 0;
    for (std::size_t m = 0; m < bins[b].member_ids.size(); ++m) {
      const auto id = bins[b].member_ids[m];
      bin_of[id] = static_cast<std::int32_t>(b);
      slot[id] = static_cast<std::int32_t>(m);
      tok_off[id] = static_cast<std::int32_t>(off);
      off += bins[b].member_lens[m];
    }
  }
  *num_bins = static_cast<std::int32_t>(bins.size());
}

}  // namespace

// ============================================================ C exports (ctypes)
extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

// mode 0: FFD naive scan, 1: FFD segment tree, 2: greedy arrival-order first fit.
int oracle_pack(const std::int64_t* len, std::int64_t n, std::int64_t cap, int mode, std::int32_t* bin_of,
                std::int32_t* slot, std::int32_t* tok_off, std::int32_t* num_bins) {
  return guarded([&] {
    std::span<const std::int64_t> L(len, static_cast<std::size_t>(n));
    auto bins = mode == 2 ? vlasim::oracle::pack_greedy(L, cap) : vlasim::oracle::pack_ffd(L, cap, mode == 0);
    bins_to_arrays(bins, bin_of, slot, tok_off, num_bins);
  });
}

int oracle_cu_seqlens(const std::int64_t* member_lens, std::int64_t m, std::int64_t* out) {
  return guarded([&] {
    vlasim::oracle::PackedSequence p;
    p.member_lens.assign(member_lens, member_lens + m);
    auto cu = vlasim::oracle::cu_seqlens(p);
    std::copy(cu.begin(), cu.end(), out);
  });
}

int oracle_padding_rate(const std::int64_t* len, std::int64_t n, std::int64_t pad_to, double* out) {
  return guarded([&] { *out = vlasim::oracle::padding_rate({len, static_cast<std::size_t>(n)}, pad_to); });
}
int oracle_dynamic_pad_length(const std::int64_t* len, std::int64_t n, std::int64_t* out) {
  return guarded([&] { *out = vlasim::oracle::dynamic_pad_length({len, static_cast<std::size_t>(n)}); });
}
int oracle_attention_flops(const std::int64_t* len, std::int64_t n, std::int64_t pad_to /* <=0: packed */,
                           std::int64_t d, double* out) {
  return guarded([&] {
    std::span<const std::int64_t> L(len, static_cast<std::size_t>(n));
    *out = pad_to > 0 ? vlasim::oracle::attention_flops_fixed(L, pad_to, d)
                      : vlasim::oracle::attention_flops_packed(L, d);
  });
}
// prune: views given as parallel arrays; returns the new total.
int oracle_prune_view(const char** names, const std::int64_t* counts, std::int64_t nviews, std::int64_t text,
                      const char* prune1, const char* prune2, std::int64_t* total_out) {
  return guarded([&] {
    std::map<std::string, std::int64_t> views;
    for (std::int64_t i = 0; i < nviews; ++i) views[names[i]] = counts[i];
    auto s = vlasim::oracle::make_sample(0, views, text);
    if (prune1) s = vlasim::oracle::prune_view(s, prune1);
    if (prune2) s = vlasim::oracle::prune_view(s, prune2);
    *total_out = s.total_len;
  });
}

// single-head SPEC ops on row-major double buffers
int oracle_reference_attention(const double* q, const double* k, const double* v, std::int64_t n, std::int64_t d,
                               double* out) {
  return guarded([&] {
    using vlasim::oracle::SmallTensor;
    SmallTensor Q{n, d, {q, q + n * d}}, K{n, d, {k, k + n * d}}, V{n, d, {v, v + n * d}};
    auto o = vlasim::oracle::reference_attention(Q, K, V);
    std::copy(o.data.begin(), o.data.end(), out);
  });
}
int oracle_packed_attention(const double* q, const double* k, const double* v, std::int64_t n, std::int64_t d,
                            const std::int64_t* cu, std::int64_t ncu, int masked, double* out) {
  return guarded([&] {
    using vlasim::oracle::SmallTensor;
    SmallTensor Q{n, d, {q, q + n * d}}, K{n, d, {k, k + n * d}}, V{n, d, {v, v + n * d}};
    std::span<const std::int64_t> c(cu, static_cast<std::size_t>(ncu));
    auto o = masked ? vlasim::oracle::masked_attention(Q, K, V, c) : vlasim::oracle::packed_attention(Q, K, V, c);
    std::copy(o.data.begin(), o.data.end(), out);
  });
}

int oracle_mha_fwd_f64(const double* q, const double* k, const double* v, double* o, double* lse,
                       const std::int32_t* cu, std::int64_t nseq, const std::int32_t* prefix, std::int64_t T,
                       std::int64_t H, std::int64_t Hkv, std::int64_t d, int mask, double scale, int threads) {
  return guarded([&] { mha_fwd<double>(q, k, v, o, lse, cu, nseq, prefix, make_shape(T, H, Hkv, d, mask, scale), threads); });
}
int oracle_mha_fwd_f32(const float* q, const float* k, const float* v, float* o, float* lse, const std::int32_t* cu,
                       std::int64_t nseq, const std::int32_t* prefix, std::int64_t T, std::int64_t H, std::int64_t Hkv,
                       std::int64_t d, int mask, double scale, int threads) {
  return guarded([&] { mha_fwd<float>(q, k, v, o, lse, cu, nseq, prefix, make_shape(T, H, Hkv, d, mask, scale), threads); });
}
int oracle_mha_bwd_f64(const double* q, const double* k, const double* v, const double* o, const double* dout,
                       double* dq, double* dk, double* dv, const std::int32_t* cu, std::int64_t nseq,
                       const std::int32_t* prefix, std::int64_t T, std::int64_t H, std::int64_t Hkv, std::int64_t d,
                       int mask, double scale, int threads) {
  return guarded([&] {
    mha_bwd<double>(q, k, v, o, dout, dq, dk, dv, cu, nseq, prefix, make_shape(T, H, Hkv, d, mask, scale), threads);
  });
}
int oracle_mha_bwd_f32(const float* q, const float* k, const float* v, const float* o, const float* dout, float* dq,
                       float* dk, float* dv, const std::int32_t* cu, std::int64_t nseq, const std::int32_t* prefix,
                       std::int64_t T, std::int64_t H, std::int64_t Hkv, std::int64_t d, int mask, double scale,
                       int threads) {
  return guarded([&] {
    mha_bwd<float>(q, k, v, o, dout, dq, dk, dv, cu, nseq, prefix, make_shape(T, H, Hkv, d, mask, scale), threads);
  });
}

// E4M3 per-block quantisation of x [T, heads, d] (per head: [T, d] tiled 128×128).
// quotient_fp32 = 1 mirrors the GPU arithmetic (fp32 scale and fp32 quotient, then RNE);
// 0 is the SPEC's high-precision real quotient.
int oracle_fp8_quant_block(const float* x, std::int64_t T, std::int64_t heads, std::int64_t d, int quotient_fp32,
                           std::uint8_t* codes, float* scales) {
  return guarded([&] {
    const std::int64_t nbt = (T + 127) / 128, nbd = (d + 127) / 128;
    for (std::int64_t h = 0; h < heads; ++h)
      for (std::int64_t bt = 0; bt < nbt; ++bt)
        for (std::int64_t bd = 0; bd < nbd; ++bd) {
          const std::int64_t t1 = std::min(T, (bt + 1) * 128), d1 = std::min(d, (bd + 1) * 128);
          double amax = 0;
          for (std::int64_t t = bt * 128; t < t1; ++t)
            for (std::int64_t c = bd * 128; c < d1; ++c) {
              const double a = std::fabs(static_cast<double>(x[(t * heads + h) * d + c]));
              if (!std::isfinite(a)) throw vlasim::ConfigError("quantize: non-finite input");
              amax = std::max(amax, a);
            }
          const float scale_f = amax == 0 ? 1.0f : static_cast<float>(amax) / 448.0f;
          // the stored scale is the fp32 rounding of amax / 448 in both modes (scale storage is
          // 4-byte); the codes differ only in the quotient they round
          scales[(h * nbt + bt) * nbd + bd] = scale_f;
          for (std::int64_t t = bt * 128; t < t1; ++t)
            for (std::int64_t c = bd * 128; c < d1; ++c) {
              const std::int64_t i = (t * heads + h) * d + c;
              if (quotient_fp32)
                codes[i] = vlasim::oracle::e4m3_encode(static_cast<double>(x[i] / scale_f));
              else if (amax == 0)
                codes[i] = vlasim::oracle::e4m3_encode(static_cast<double>(x[i]));  // ±0 at scale 1
              else
                codes[i] = vlasim::oracle::e4m3_encode_ratio(static_cast<double>(x[i]) * 448.0, amax);
            }
        }
  });
}
// The SPEC's quantize for every Granularity: groups are
// PerTensor (one), PerChannel(axis) (index along `axis`), PerBlock (128×128 tiles of the last two
// dims, per leading index; block_partition SPEC.md:566-572).  scale_g = fp32(amax_g / 448) (1 if
// the group is all zero); codes by the exhaustive midpoint search on the REAL quotient
// x·448 / amax_g (e4m3_encode_ratio).  Non-finite input → ConfigError.
// gran: 0 tensor, 1 channel, 2 block.  Scales laid out like vlasim_fp8_quantize_cuda's.
int oracle_fp8_quantize(const float* x, const std::int64_t* shape, int ndim, int gran, int axis,
                        std::uint8_t* codes, float* scales) {
  return guarded([&] {
    std::int64_t n = 1;
    for (int i = 0; i < ndim; ++i) n *= shape[i];
    std::vector<std::int64_t> grp(static_cast<std::size_t>(n));
    std::int64_t groups = 1;
    if (gran == 1) {
      if (axis < 0) axis += ndim;
      std::int64_t inner = 1;
      for (int i = axis + 1; i < ndim; ++i) inner *= shape[i];
      groups = shape[axis];
      for (std::int64_t i = 0; i < n; ++i) grp[i] = (i / inner) % groups;
    } else if (gran == 2) {
      if (ndim < 2) throw vlasim::ConfigError("block_partition: shape needs >= 2 dims");
      const std::int64_t rows = shape[ndim - 2], cols = shape[ndim - 1];
      const std::int64_t nbr = (rows + 127) / 128, nbc = (cols + 127) / 128;
      groups = (n / (rows * cols)) * nbr * nbc;
      for (std::int64_t i = 0; i < n; ++i) {
        const std::int64_t c = i % cols, r = (i / cols) % rows, b = i / (rows * cols);
        grp[i] = (b * nbr + r / 128) * nbc + c / 128;
      }
    } else {
      std::fill(grp.begin(), grp.end(), 0);
    }
    std::vector<double> amax(static_cast<std::size_t>(groups), 0.0);
    for (std::int64_t i = 0; i < n; ++i) {
      const double a = std::fabs(static_cast<double>(x[i]));
      if (!std::isfinite(a)) throw vlasim::ConfigError("quantize: non-finite input");
      amax[grp[i]] = std::max(amax[grp[i]], a);
    }
    for (std::int64_t g = 0; g < groups; ++g)
      scales[g] = amax[g] == 0 ? 1.0f : static_cast<float>(amax[g]) / 448.0f;
    for (std::int64_t i = 0; i < n; ++i) {
      const double a = amax[grp[i]];
      codes[i] = a == 0 ? vlasim::oracle::e4m3_encode(static_cast<double>(x[i]))
                        : vlasim::oracle::e4m3_encode_ratio(static_cast<double>(x[i]) * 448.0, a);
    }
  });
}
int oracle_e4m3_encode(const double* x, std::int64_t n, std::uint8_t* codes) {
  return guarded([&] {
    for (std::int64_t i = 0; i < n; ++i) codes[i] = vlasim::oracle::e4m3_encode(x[i]);
  });
}
// Sample lengths on the reference's seeding API (rng.hpp:28-49), the same conventions as the bench
// inputs: dist 0 uniform_int(p1, p2); 1 truncated geometric(p1, max p2) by inverse
// CDF on uniform01; 2 GR00T-like 64·uniform_int(1,2) + uniform_int(16,64); 3 π0.5 512 +
// uniform_int(p1, p2) + p3.  Lets the CPU arms generate their inputs without the product library.
int oracle_gen_lengths(std::uint64_t root_seed, const char* label, int dist, std::int64_t n, double p1, double p2,
                       double p3, std::int32_t* out) {
  return guarded([&] {
    auto rng = vlasim::make_rng(root_seed, std::string_view(label), 0);
    for (std::int64_t i = 0; i < n; ++i) {
      std::int64_t l = 0;
      if (dist == 0) {
        l = vlasim::uniform_int(rng, std::int64_t(p1), std::int64_t(p2));
      } else if (dist == 1) {
        const double tail = 1.0 - std::pow(1.0 - p1, p2);
        double k = std::ceil(std::log1p(-vlasim::uniform01(rng) * tail) / std::log1p(-p1));
        l = std::int64_t(std::min(std::max(k, 1.0), p2));
      } else if (dist == 2) {
        const std::int64_t views = vlasim::uniform_int(rng, 1, 2);
        l = 64 * views + vlasim::uniform_int(rng, 16, 64);
      } else if (dist == 3) {
        l = 512 + vlasim::uniform_int(rng, std::int64_t(p1), std::int64_t(p2)) + std::int64_t(p3);
      } else {
        throw vlasim::ConfigError("gen_lengths: unknown distribution");
      }
      out[i] = std::int32_t(l);
    }
  });
}

int oracle_e4m3_values(double* out /* [127] */) {
  return guarded([&] {
    auto v = vlasim::oracle::e4m3_values();
    std::copy(v.begin(), v.end(), out);
  });
}

}  // extern "C"
