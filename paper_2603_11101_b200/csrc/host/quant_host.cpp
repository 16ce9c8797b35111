// quant_host.cpp — the reconstructed vlasim:: quantizer API (include/vlasim/quant/*.hpp) over the
// C-ABI: quantize / dequantize / quant_error copy the tensor to the device (fp32), run the sm_100a
// kernels (quant.cu) and copy the results back; file forms and the compression calculator are host
// code restating SPEC.md:564-615, 631-634.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>

#include "vlasim/quant/compression.hpp"
#include "vlasim/quant/quantize.hpp"
#include "vlasim/util/errors.hpp"
#include "vlasim_cuda.h"

namespace vlasim {
namespace {

void check(int rc, const char* what) {
  if (rc != 0) detail::throw_status(rc, std::string(what) + ": " + vlasim_last_error_message());
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw SimError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Dev {
  void* p = nullptr;
  explicit Dev(std::size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

std::vector<float> to_f32(const Tensor& t) {
  std::vector<float> x(t.data.size());
  for (std::size_t i = 0; i < x.size(); ++i) x[i] = static_cast<float>(t.data[i]);
  return x;
}

void validate_shape(const std::vector<std::int64_t>& shape, std::size_t n) {
  if (shape.empty() || shape.size() > 8) throw ConfigError("tensor: 1-8 dimensions required");
  std::int64_t p = 1;
  for (auto s : shape) {
    if (s < 1) throw ConfigError("tensor: dimensions must be >= 1");
    p *= s;
  }
  if (std::size_t(p) != n) throw ConfigError("tensor: shape does not match the data size");
}

std::vector<std::int64_t> scales_shape_of(const std::vector<std::int64_t>& shape, const Granularity& g) {
  if (g.kind == GranularityKind::PerTensor) return {1};
  if (g.kind == GranularityKind::PerChannel) {
    const int nd = int(shape.size());
    const int ax = g.axis < 0 ? g.axis + nd : g.axis;
    if (ax < 0 || ax >= nd) throw ConfigError("quantize: channel axis out of range");
    return {shape[ax]};
  }
  if (shape.size() < 2) throw ConfigError("block_partition: shape needs >= 2 dims");
  std::vector<std::int64_t> s(shape.begin(), shape.end() - 2);
  s.push_back((shape[shape.size() - 2] + 127) / 128);
  s.push_back((shape.back() + 127) / 128);
  return s;
}

template <typename T>
void put(std::ostream& o, const T& v) {
  o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get(std::istream& in, const std::string& path) {
  T v{};
  if (!in.read(reinterpret_cast<char*>(&v), sizeof(T))) throw ConfigError(path + ": truncated file");
  return v;
}

}  // namespace

// ------------------------------------------------------------------ fp8.hpp
double fp8_decode(std::uint8_t code) {
  const int e = (code >> 3) & 0xF, m = code & 7;
  if (e == 15 && m == 7) return std::nan("");
  const double v = e == 0 ? std::ldexp(m / 8.0, -6) : std::ldexp(1.0 + m / 8.0, e - 7);
  return (code & 0x80) ? -v : v;
}

// ------------------------------------------------------------------ tensor.hpp
std::int64_t Tensor::numel() const {
  std::int64_t p = 1;
  for (auto s : shape) p *= s;
  return shape.empty() ? 0 : p;
}

Tensor read_tensor_text(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open tensor file " + path);
  Tensor t;
  std::string line;
  bool have_shape = false;
  while (std::getline(in, line)) {
    if (auto h = line.find('#'); h != std::string::npos) line.resize(h);
    std::istringstream ss(line);
    if (!have_shape) {
      long long d;
      while (ss >> d) t.shape.push_back(d);
      have_shape = !t.shape.empty();
      continue;
    }
    std::string tok;
    while (ss >> tok) {
      char* end = nullptr;
      const double v = std::strtod(tok.c_str(), &end);
      if (end == tok.c_str() || *end) throw ConfigError(path + ": bad value '" + tok + "'");
      t.data.push_back(v);
    }
  }
  if (!have_shape) throw ConfigError(path + ": missing shape line");
  validate_shape(t.shape, t.data.size());
  return t;
}

Tensor read_tensor(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ConfigError("cannot open tensor file " + path);
  char magic[4] = {0, 0, 0, 0};
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "VLT1", 4) != 0) return read_tensor_text(path);
  Tensor t;
  const auto nd = get<std::uint32_t>(in, path);
  if (nd < 1 || nd > 8) throw ConfigError(path + ": 1-8 dimensions required");
  for (std::uint32_t i = 0; i < nd; ++i) t.shape.push_back(get<std::int64_t>(in, path));
  std::int64_t n = 1;
  for (auto s : t.shape) {
    if (s < 1) throw ConfigError(path + ": dimensions must be >= 1");
    n *= s;
  }
  t.data.resize(std::size_t(n));
  if (!in.read(reinterpret_cast<char*>(t.data.data()), std::streamsize(n * 8))) throw ConfigError(path + ": truncated");
  return t;
}

void write_tensor(const std::string& path, const Tensor& t) {
  validate_shape(t.shape, t.data.size());
  std::ofstream o(path, std::ios::binary);
  if (!o) throw SimError("cannot write " + path);
  o.write("VLT1", 4);
  put(o, std::uint32_t(t.shape.size()));
  for (auto s : t.shape) put(o, std::int64_t(s));
  o.write(reinterpret_cast<const char*>(t.data.data()), std::streamsize(t.data.size() * 8));
}

// ------------------------------------------------------------------ quantize.hpp
std::string Granularity::name() const {
  if (kind == GranularityKind::PerTensor) return "tensor";
  if (kind == GranularityKind::PerChannel) return "channel:" + std::to_string(axis);
  return "block";
}

Granularity Granularity::parse(const std::string& s) {
  if (s == "tensor") return per_tensor();
  if (s == "block") return per_block();
  if (s == "channel") return per_channel(0);
  if (s.rfind("channel:", 0) == 0) {
    std::size_t used = 0;
    int ax = 0;
    try {
      ax = std::stoi(s.substr(8), &used);
    } catch (const std::exception&) {
      used = 0;
    }
    if (used == 0 || used != s.size() - 8) throw ConfigError("bad granularity '" + s + "'");
    return per_channel(ax);
  }
  throw ConfigError("unknown granularity '" + s + "' (tensor | channel[:axis] | block)");
}

std::vector<BlockExtent> block_partition(const std::vector<std::int64_t>& shape, std::int64_t br, std::int64_t bc) {
  if (shape.size() < 2) throw ConfigError("block_partition: shape needs >= 2 dims");
  if (br < 1 || bc < 1) throw ConfigError("block_partition: block dims must be >= 1");
  const std::int64_t R = shape[shape.size() - 2], C = shape.back();
  std::vector<BlockExtent> out;
  for (std::int64_t r = 0; r < R; r += br)
    for (std::int64_t c = 0; c < C; c += bc) out.push_back({r, std::min(br, R - r), c, std::min(bc, C - c)});
  return out;
}

QuantizedTensor quantize(const Tensor& t, const Granularity& g, const Fp8Format& fmt) {
  if (fmt.exponent_bits != 4 || fmt.mantissa_bits != 3 || fmt.bias != 7 || fmt.max_normal != 448.0)
    throw ConfigError("quantize: only FP8 E4M3 is supported (SPEC.md:624)");
  validate_shape(t.shape, t.data.size());
  for (std::size_t i = 0; i < t.data.size(); ++i)
    if (!std::isfinite(t.data[i])) throw ConfigError("quantize: non-finite input at flat index " + std::to_string(i));
  QuantizedTensor qt;
  qt.shape = t.shape;
  qt.granularity = g;
  qt.scales_shape = scales_shape_of(t.shape, g);
  const int gk = int(g.kind);
  const int nd = int(t.shape.size());
  const std::int64_t groups = vlasim_fp8_groups(t.shape.data(), nd, gk, g.axis);
  if (groups < 1) check(VLASIM_ECONFIG, "quantize");
  const std::vector<float> x = to_f32(t);
  const std::size_t n = x.size();
  Dev dx(n * 4), dcodes(n), dscales(std::size_t(groups) * 4), dstatus(8);
  const std::size_t wsb = vlasim_fp8_quantize_workspace_size(t.shape.data(), nd, gk, g.axis);
  Dev dws(wsb);
  cuda_check(cudaMemcpy(dx.p, x.data(), n * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  check(vlasim_fp8_quantize_cuda(dx.p, VLASIM_DTYPE_F32, t.shape.data(), nd, gk, g.axis, dcodes.as<std::uint8_t>(),
                                 dscales.as<float>(), dstatus.as<std::int32_t>(), dws.p, wsb, VLASIM_SYNC_CHECK,
                                 nullptr),
        "quantize");
  qt.codes.resize(n);
  qt.scales.resize(std::size_t(groups));
  cuda_check(cudaMemcpy(qt.codes.data(), dcodes.p, n, cudaMemcpyDeviceToHost), "cudaMemcpy");
  cuda_check(cudaMemcpy(qt.scales.data(), dscales.p, std::size_t(groups) * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  return qt;
}

Tensor dequantize(const QuantizedTensor& qt) {
  validate_shape(qt.shape, qt.codes.size());
  const int nd = int(qt.shape.size()), gk = int(qt.granularity.kind);
  const std::size_t n = qt.codes.size();
  Dev dcodes(n), dscales(qt.scales.size() * 4), dout(n * 4);
  cuda_check(cudaMemcpy(dcodes.p, qt.codes.data(), n, cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMemcpy(dscales.p, qt.scales.data(), qt.scales.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  check(vlasim_fp8_dequantize_cuda(dcodes.as<std::uint8_t>(), dscales.as<float>(), qt.shape.data(), nd, gk,
                                   qt.granularity.axis, dout.as<float>(), nullptr),
        "dequantize");
  std::vector<float> out(n);
  cuda_check(cudaMemcpy(out.data(), dout.p, n * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  Tensor t;
  t.shape = qt.shape;
  t.data.assign(out.begin(), out.end());
  return t;
}

QuantErrorMetrics quant_error(const Tensor& original, const QuantizedTensor& qt) {
  if (original.shape != qt.shape) throw ConfigError("quant_error: shapes differ");
  validate_shape(qt.shape, qt.codes.size());
  const int nd = int(qt.shape.size()), gk = int(qt.granularity.kind);
  const std::int64_t ng = vlasim_fp8_error_groups(qt.shape.data(), nd, gk, qt.granularity.axis);
  const std::vector<float> x = to_f32(original);
  const std::size_t n = x.size();
  Dev dx(n * 4), dcodes(n), dscales(qt.scales.size() * 4), dmax(std::size_t(ng) * 4), dsse(std::size_t(ng) * 8),
      dcnt(std::size_t(ng) * 8);
  cuda_check(cudaMemcpy(dx.p, x.data(), n * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMemcpy(dcodes.p, qt.codes.data(), n, cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMemcpy(dscales.p, qt.scales.data(), qt.scales.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  check(vlasim_fp8_quant_error_general_cuda(dx.p, VLASIM_DTYPE_F32, dcodes.as<std::uint8_t>(), dscales.as<float>(),
                                            qt.shape.data(), nd, gk, qt.granularity.axis, dmax.as<float>(),
                                            dsse.as<double>(), dcnt.as<std::int64_t>(), nullptr),
        "quant_error");
  const std::size_t groups = qt.granularity.kind == GranularityKind::PerTensor ? 1 : std::size_t(ng);
  std::vector<float> gmax(groups);
  std::vector<double> gsse(groups);
  std::vector<std::int64_t> gcnt(groups);
  cuda_check(cudaMemcpy(gmax.data(), dmax.p, groups * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  cuda_check(cudaMemcpy(gsse.data(), dsse.p, groups * 8, cudaMemcpyDeviceToHost), "cudaMemcpy");
  cuda_check(cudaMemcpy(gcnt.data(), dcnt.p, groups * 8, cudaMemcpyDeviceToHost), "cudaMemcpy");
  QuantErrorMetrics m;
  double sse = 0;
  std::int64_t cnt = 0;
  for (std::size_t g = 0; g < groups; ++g) {  // fixed (group) order
    m.max_rel = std::max(m.max_rel, double(gmax[g]));
    sse += gsse[g];
    cnt += gcnt[g];
    m.group_max_rel.push_back(gmax[g]);
    m.group_mse.push_back(gsse[g] / double(gcnt[g]));
  }
  m.mse = sse / double(cnt);
  return m;
}

void write_quantized(const std::string& path, const QuantizedTensor& qt) {
  std::ofstream o(path, std::ios::binary);
  if (!o) throw SimError("cannot write " + path);
  o.write("VLQ1", 4);
  put(o, std::uint8_t(qt.granularity.kind));
  put(o, std::int32_t(qt.granularity.axis));
  put(o, std::uint32_t(qt.shape.size()));
  for (auto s : qt.shape) put(o, std::int64_t(s));
  put(o, std::uint64_t(qt.scales.size()));
  o.write(reinterpret_cast<const char*>(qt.scales.data()), std::streamsize(qt.scales.size() * 4));
  o.write(reinterpret_cast<const char*>(qt.codes.data()), std::streamsize(qt.codes.size()));
}

QuantizedTensor read_quantized(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ConfigError("cannot open " + path);
  char magic[4] = {0, 0, 0, 0};
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "VLQ1", 4) != 0) throw ConfigError(path + ": not a quantized tensor file");
  QuantizedTensor qt;
  const auto kind = get<std::uint8_t>(in, path);
  if (kind > 2) throw ConfigError(path + ": bad granularity tag");
  qt.granularity.kind = GranularityKind(kind);
  qt.granularity.axis = get<std::int32_t>(in, path);
  const auto nd = get<std::uint32_t>(in, path);
  if (nd < 1 || nd > 8) throw ConfigError(path + ": 1-8 dimensions required");
  std::int64_t n = 1;
  for (std::uint32_t i = 0; i < nd; ++i) {
    qt.shape.push_back(get<std::int64_t>(in, path));
    if (qt.shape.back() < 1) throw ConfigError(path + ": dimensions must be >= 1");
    n *= qt.shape.back();
  }
  qt.scales_shape = scales_shape_of(qt.shape, qt.granularity);
  const auto ns = get<std::uint64_t>(in, path);
  std::uint64_t want = 1;
  for (auto s : qt.scales_shape) want *= std::uint64_t(s);
  if (ns != want) throw ConfigError(path + ": scale count does not match the granularity");
  qt.scales.resize(ns);
  qt.codes.resize(std::size_t(n));
  if (!in.read(reinterpret_cast<char*>(qt.scales.data()), std::streamsize(ns * 4)) ||
      !in.read(reinterpret_cast<char*>(qt.codes.data()), std::streamsize(n)))
    throw ConfigError(path + ": truncated");
  for (float s : qt.scales)
    if (!(s > 0)) throw ConfigError(path + ": scales must be > 0");
  return qt;
}

// ------------------------------------------------------------------ compression.hpp
double compression_ratio(const ModelSizeSpec& spec) {
  if (spec.components.empty()) throw ConfigError("compression_ratio: empty spec");
  double total = 0, bytes = 0;
  for (const auto& c : spec.components) {
    if (c.params <= 0) throw ConfigError("compression_ratio: component '" + c.name + "' has no parameters");
    total += double(c.params);
    if (!c.quantize) {
      bytes += double(c.params) * spec.bytes_hi;
    } else {
      const double per_elem = c.granularity.kind == GranularityKind::PerBlock ? spec.scale_bytes / (128.0 * 128.0) : 0.0;
      bytes += double(c.params) * (spec.bytes_lo + per_elem);
    }
  }
  return 1.0 - bytes / (total * spec.bytes_hi);
}

}  // namespace vlasim
