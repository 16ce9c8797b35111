// vlasim_host.cpp — the reconstructed vlasim:: C++ API (include/vlasim/packing/*.hpp) implemented
// over the C-ABI (include/vlasim_cuda.h).  Host-side scalar helpers restate SPEC.md directly; the
// packing and attention entry points copy to the device, call the sm_100a kernels and map the
// C-ABI status codes onto the reference's exceptions (errors.hpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include "vlasim/packing/attention.hpp"
#include "vlasim/packing/pack.hpp"
#include "vlasim/packing/sample.hpp"
#include "vlasim/util/errors.hpp"

namespace vlasim {
namespace {

void check(int rc, const char* what) {
  if (rc != 0) detail::throw_status(rc, std::string(what) + ": " + vlasim_last_error_message());
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw SimError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(std::size_t n) { cuda_check(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

// ------------------------------------------------------------------ sample.hpp
SampleLen make_sample(std::int64_t id, const std::map<std::string, std::int64_t>& view_lens, std::int64_t text_len) {
  if (text_len < 0) throw ConfigError("sample " + std::to_string(id) + ": negative text length");
  SampleLen s{id, text_len, view_lens, text_len};
  for (const auto& [name, n] : view_lens) {
    if (n < 0) throw ConfigError("sample " + std::to_string(id) + ": negative view '" + name + "'");
    s.total_len += n;
  }
  if (s.total_len < 1) throw ConfigError("sample " + std::to_string(id) + " has no tokens");
  return s;
}

SampleLen prune_view(const SampleLen& sample, std::string_view view) {
  auto it = sample.view_lens.find(std::string(view));
  if (it == sample.view_lens.end())
    throw ConfigError("prune_view: sample " + std::to_string(sample.id) + " has no view '" + std::string(view) + "'");
  SampleLen r = sample;
  r.total_len -= it->second;
  r.view_lens.erase(std::string(view));
  return r;
}

double padding_rate(std::span<const std::int64_t> lengths, std::int64_t pad_to) {
  if (lengths.empty()) throw ConfigError("padding_rate: empty batch");
  const std::int64_t mx = *std::max_element(lengths.begin(), lengths.end());
  if (pad_to < mx) throw ConfigError("padding_rate: pad_to below the longest sample");
  const double sum = std::accumulate(lengths.begin(), lengths.end(), 0.0);
  return 1.0 - sum / (double(lengths.size()) * double(pad_to));
}

std::int64_t dynamic_pad_length(std::span<const std::int64_t> lengths) {
  if (lengths.empty()) throw ConfigError("dynamic_pad_length: empty batch");
  return *std::max_element(lengths.begin(), lengths.end());
}

double attention_flops(std::span<const std::int64_t> lengths, std::int64_t head_dim, std::optional<std::int64_t> pad_to,
                       double c) {
  if (pad_to) {
    for (auto l : lengths)
      if (l > *pad_to) throw ConfigError("attention_flops: length above pad_to");
    return double(lengths.size()) * c * double(*pad_to) * double(*pad_to) * double(head_dim);
  }
  double s = 0;
  for (auto l : lengths) s += double(l) * double(l);
  return c * s * double(head_dim);
}

// ------------------------------------------------------------------ pack.hpp
std::int64_t PackedSequence::fill() const {
  return std::accumulate(member_lens.begin(), member_lens.end(), std::int64_t{0});
}

GpuPacker::GpuPacker(std::int64_t max_n, std::int32_t capacity) : max_n_(max_n), capacity_(capacity) {
  if (max_n < 1) throw ConfigError("GpuPacker: max_n must be >= 1");
  const std::size_t n = std::size_t(max_n);
  // one device block for every output array (sizes from vlasim_cuda.h)
  const std::size_t ints = 5 * n + 2 * (n + 1) + n + (n + 1) + 2 * n + (n + 1) + 1 + 2;
  cuda_check(cudaMalloc(&block_, ints * 4 + 16), "cudaMalloc");
  auto* p = static_cast<std::int32_t*>(block_);
  auto take = [&](std::size_t k) {
    std::int32_t* r = p;
    p += k;
    return r;
  };
  out_.bin_of = take(n);
  out_.slot = take(n);
  out_.tok_off = take(n);
  out_.bin_count = take(n);
  out_.bin_fill = take(n);
  out_.bin_member_off = take(n + 1);
  out_.bin_token_off = take(n + 1);
  out_.member_ids = take(n);
  out_.cu_seqlens = take(n + 1);
  out_.cu_seqlens_bins = take(2 * n);
  out_.src_off = take(n + 1);
  out_.num_bins = take(1);
  out_.status = take(2);
  p += (reinterpret_cast<std::uintptr_t>(p) & 7) ? 1 : 0;
  out_.total_tokens = reinterpret_cast<std::int64_t*>(p);
  ws_bytes_ = vlasim_pack_workspace_size(max_n, capacity);
  cuda_check(cudaMalloc(&ws_, ws_bytes_), "cudaMalloc");
}

GpuPacker::~GpuPacker() {
  cudaFree(ws_);
  cudaFree(block_);
}

void GpuPacker::pack(const std::int32_t* d_lengths, std::int64_t n, vlasim_stream_t stream, bool sync_check) {
  if (n > max_n_) throw ConfigError("GpuPacker: batch larger than max_n");
  check(vlasim_pack_ffd_cuda(d_lengths, n, capacity_, &out_, ws_, ws_bytes_, sync_check ? VLASIM_PACK_SYNC_CHECK : 0u,
                             stream),
        "pack_ffd");
}

void GpuPacker::pack_greedy(const std::int32_t* d_lengths, std::int64_t n, vlasim_stream_t stream, bool sync_check) {
  if (n > max_n_) throw ConfigError("GpuPacker: batch larger than max_n");
  check(vlasim_pack_greedy_cuda(d_lengths, n, capacity_, &out_, ws_, ws_bytes_,
                                sync_check ? VLASIM_PACK_SYNC_CHECK : 0u, stream),
        "pack_greedy");
}

static std::vector<PackedSequence> run_pack(std::span<const std::int64_t> lengths, std::int64_t capacity, bool greedy) {
  const std::int64_t n = std::int64_t(lengths.size());
  if (n < 1) throw ConfigError("pack: need at least one sample");
  if (capacity < 1 || capacity > VLASIM_PACK_MAX_CAPACITY) throw ConfigError("pack: capacity out of range");
  std::vector<std::int32_t> h(lengths.size());
  for (std::size_t i = 0; i < lengths.size(); ++i) {
    if (lengths[i] > capacity)
      throw ConfigError("oversize sample id " + std::to_string(i) + ": length " + std::to_string(lengths[i]) +
                        " > capacity " + std::to_string(capacity));
    if (lengths[i] < 1) throw ConfigError("empty sample id " + std::to_string(i));
    h[i] = std::int32_t(lengths[i]);
  }
  GpuPacker packer(n, std::int32_t(capacity));
  DevBuf<std::int32_t> d_len{std::size_t(n)};
  cuda_check(cudaMemcpy(d_len.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  const vlasim_pack_out& o = packer.out();
  if (greedy)
    packer.pack_greedy(d_len.p, n, nullptr, true);
  else
    packer.pack(d_len.p, n, nullptr, true);
  std::int32_t nb = 0;
  cuda_check(cudaMemcpy(&nb, o.num_bins, 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  std::vector<std::int32_t> member_off(std::size_t(nb) + 1), member_ids(static_cast<std::size_t>(n));
  cuda_check(cudaMemcpy(member_off.data(), o.bin_member_off, member_off.size() * 4, cudaMemcpyDeviceToHost),
             "cudaMemcpy");
  cuda_check(cudaMemcpy(member_ids.data(), o.member_ids, member_ids.size() * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  std::vector<PackedSequence> bins(static_cast<std::size_t>(nb));
  for (std::int32_t b = 0; b < nb; ++b) {
    bins[b].capacity = capacity;
    for (std::int32_t m = member_off[b]; m < member_off[b + 1]; ++m) {
      bins[b].member_ids.push_back(member_ids[m]);
      bins[b].member_lens.push_back(lengths[member_ids[m]]);
    }
  }
  return bins;
}

std::vector<PackedSequence> pack_ffd(std::span<const std::int64_t> lengths, std::int64_t capacity) {
  return run_pack(lengths, capacity, false);
}
std::vector<PackedSequence> pack_greedy(std::span<const std::int64_t> lengths, std::int64_t capacity) {
  return run_pack(lengths, capacity, true);
}

std::vector<std::int64_t> cu_seqlens(const PackedSequence& pack) {
  if (pack.member_lens.empty()) throw ConfigError("cu_seqlens: empty pack");
  std::vector<std::int64_t> cu(pack.member_lens.size() + 1, 0);
  for (std::size_t i = 0; i < pack.member_lens.size(); ++i) cu[i + 1] = cu[i] + pack.member_lens[i];
  return cu;
}

PackingStats packing_stats(std::span<const std::int64_t> lengths, const std::vector<PackedSequence>& bins,
                           std::int64_t pad_to, std::int64_t head_dim) {
  PackingStats s;
  s.bins_used = std::int64_t(bins.size());
  const double sum = std::accumulate(lengths.begin(), lengths.end(), 0.0);
  const double cap = bins.empty() ? 1.0 : double(bins[0].capacity);
  s.fill_rate = bins.empty() ? 0.0 : sum / (double(s.bins_used) * cap);
  s.padding_rate_before = padding_rate(lengths, pad_to);
  s.padding_rate_after = 1.0 - s.fill_rate;
  s.attention_flops_fixed = attention_flops(lengths, head_dim, pad_to);
  s.attention_flops_packed = attention_flops(lengths, head_dim);
  return s;
}

// ------------------------------------------------------------------ attention.hpp
VarlenAttention::~VarlenAttention() { cudaFree(ws_); }

void VarlenAttention::reserve(std::size_t bytes) {
  if (bytes <= ws_bytes_) return;
  cudaFree(ws_);
  ws_ = nullptr;
  cuda_check(cudaMalloc(&ws_, bytes), "cudaMalloc");
  ws_bytes_ = bytes;
}

void VarlenAttention::forward(const vlasim_attn_args& a, vlasim_stream_t stream) {
  reserve(vlasim_varlen_attn_workspace_size(&a, 0));
  check(vlasim_varlen_attn_fwd_cuda(&a, ws_, ws_bytes_, stream), "varlen_attn_fwd");
}

void VarlenAttention::backward(const vlasim_attn_args& a, const vlasim_attn_grads& g, vlasim_stream_t stream) {
  reserve(vlasim_varlen_attn_workspace_size(&a, 1));
  check(vlasim_varlen_attn_bwd_cuda(&a, &g, ws_, ws_bytes_, stream), "varlen_attn_bwd");
}

namespace {
std::uint16_t to_bf16(double x) {  // round-to-nearest-even on the fp32 value
  float f = float(x);
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return std::uint16_t(u >> 16);
}
double from_bf16(std::uint16_t b) {
  std::uint32_t u = std::uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
}  // namespace

SmallTensor packed_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v,
                             std::span<const std::int64_t> cu) {
  if (q.rows != k.rows || k.rows != v.rows || q.cols != k.cols || v.cols != q.cols)
    throw ConfigError("packed_attention: shape mismatch");
  if (cu.size() < 2 || cu.front() != 0 || cu.back() != q.rows)
    throw ConfigError("packed_attention: cu_seqlens inconsistent with tensors");
  for (std::size_t i = 1; i < cu.size(); ++i)
    if (cu[i] <= cu[i - 1]) throw ConfigError("packed_attention: cu_seqlens not strictly increasing");
  const std::int64_t T = q.rows, d = q.cols;
  if (d < 1 || T < 1) throw ConfigError("packed_attention: empty tensors");
  if (std::int64_t(q.data.size()) != T * d || std::int64_t(k.data.size()) != T * d ||
      std::int64_t(v.data.size()) != T * d)
    throw ConfigError("packed_attention: data size does not match rows x cols");
  // Any model_dim up to 256: the columns are zero-padded to the kernels' head_dim (64 / 128 / 256),
  // which leaves q·kᵀ unchanged and adds zero columns to p·v that are sliced off; the softmax
  // scale stays 1/sqrt(model_dim).
  if (d > 256) throw ConfigError("packed_attention: model_dim " + std::to_string(d) + " > 256 (one head of the "
                                 "sm_100a kernels; split heads instead)");
  const std::int64_t D = d <= 64 ? 64 : (d <= 128 ? 128 : 256);
  std::vector<std::uint16_t> hq(T * D, 0), hk(T * D, 0), hv(T * D, 0), ho(T * D);
  for (std::int64_t r = 0; r < T; ++r)
    for (std::int64_t c = 0; c < d; ++c) {
      hq[r * D + c] = to_bf16(q.data[r * d + c]);
      hk[r * D + c] = to_bf16(k.data[r * d + c]);
      hv[r * D + c] = to_bf16(v.data[r * d + c]);
    }
  std::vector<std::int32_t> hcu(cu.begin(), cu.end());
  DevBuf<std::uint16_t> dq(T * D), dk(T * D), dv(T * D), dout(T * D);
  DevBuf<float> dlse(T);
  DevBuf<std::int32_t> dcu(hcu.size());
  cuda_check(cudaMemcpy(dq.p, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMemcpy(dk.p, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMemcpy(dv.p, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMemcpy(dcu.p, hcu.data(), hcu.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  vlasim_attn_args a{};
  a.q = dq.p;
  a.k = dk.p;
  a.v = dv.p;
  a.o = dout.p;
  a.lse = dlse.p;
  a.cu_seqlens = dcu.p;
  a.num_seqs = std::int32_t(cu.size() - 1);
  a.total_tokens = T;
  a.num_heads = 1;
  a.num_kv_heads = 1;
  a.head_dim = std::int32_t(D);
  a.mask_mode = VLASIM_MASK_BIDIR;
  a.softmax_scale = float(1.0 / std::sqrt(double(d)));
  VarlenAttention attn;
  attn.forward(a, nullptr);
  cuda_check(cudaMemcpy(ho.data(), dout.p, ho.size() * 2, cudaMemcpyDeviceToHost), "cudaMemcpy");
  SmallTensor o{T, d, std::vector<double>(std::size_t(T * d))};
  for (std::int64_t r = 0; r < T; ++r)
    for (std::int64_t c = 0; c < d; ++c) o.data[r * d + c] = from_bf16(ho[r * D + c]);
  return o;
}

SmallTensor reference_attention(const SmallTensor& q, const SmallTensor& k, const SmallTensor& v) {
  const std::int64_t cu[2] = {0, q.rows};
  return packed_attention(q, k, v, cu);
}

}  // namespace vlasim
