// cli_quantbench.cpp — `vlasim_quantbench`: the reference's `quantbench` subcommand
// on the GPU quantizer: a granularity sweep over tensor fixtures emitting error / compression tables,
// plus the model-compression calculator.
//
//   vlasim_quantbench [--config FILE] [--fixture PATH]... [--synthetic ROWSxCOLS] [--seed N]
//                     [--granularity LIST] [--model-spec FILE] [--out DIR]
//
// Config (strict schema, vlasim/util/kv_file.hpp):
//   seed = 42                          out = DIR
//   [quantization]  fixtures = a.vlt, b.txt   granularities = tensor, channel:0, block
//                   synthetic = 512x1024
//   [model]         bytes_hi = 2   bytes_lo = 1   scale_bytes = 4
//                   component.<name> = <params> <quantize|keep> [granularity]
// Tables are flat tab-separated text on stdout and, with --out, in
// DIR/quantbench.tsv and DIR/compression.tsv.  Exit codes SPEC.md:703: 0 ok, 2 ConfigError (unknown
// key, non-finite fixture value, ...), 3 runtime error.
#include <sys/stat.h>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "vlasim/quant/compression.hpp"
#include "vlasim/quant/quantize.hpp"
#include "vlasim/util/errors.hpp"
#include "vlasim/util/kv_file.hpp"
#include "vlasim/util/rng.hpp"

namespace {

std::vector<std::string> split_list(const std::string& s) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s + ",") {
    if (c == ',') {
      const auto b = cur.find_first_not_of(" \t"), e = cur.find_last_not_of(" \t");
      if (b != std::string::npos) out.push_back(cur.substr(b, e - b + 1));
      cur.clear();
    } else {
      cur += c;
    }
  }
  return out;
}

// Heterogeneous synthetic weight-like tensor from the reference's seeding API (rng.hpp:28-49): row r
// has magnitude 10^(4·u_r − 2), elements uniform in (−1, 1) times it.
vlasim::Tensor synthetic(std::int64_t rows, std::int64_t cols, std::uint64_t seed) {
  vlasim::Tensor t;
  t.shape = {rows, cols};
  t.data.resize(std::size_t(rows * cols));
  auto rr = vlasim::make_rng(seed, "quant_rows", 0);
  auto re = vlasim::make_rng(seed, "quant_vals", 0);
  for (std::int64_t r = 0; r < rows; ++r) {
    const double mag = std::pow(10.0, 4.0 * vlasim::uniform01(rr) - 2.0);
    for (std::int64_t c = 0; c < cols; ++c)
      t.data[std::size_t(r * cols + c)] = double(float((2.0 * vlasim::uniform01(re) - 1.0) * mag));
  }
  return t;
}

int usage() {
  std::fprintf(stderr,
               "usage: vlasim_quantbench [--config FILE] [--fixture PATH]... [--synthetic RxC] [--seed N]\n"
               "                         [--granularity LIST] [--model-spec FILE] [--out DIR]\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    std::vector<std::string> fixtures;
    std::vector<std::string> grans;
    std::string synth, model_spec, out_dir, config;
    long long seed = 42;
    bool seed_set = false;
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) throw vlasim::ConfigError("missing value for " + a);
        return argv[++i];
      };
      if (a == "--config") config = val();
      else if (a == "--fixture") fixtures.push_back(val());
      else if (a == "--synthetic") synth = val();
      else if (a == "--seed") { seed = std::stoll(val()); seed_set = true; }
      else if (a == "--granularity") grans = split_list(val());
      else if (a == "--model-spec") model_spec = val();
      else if (a == "--out") out_dir = val();
      else if (a == "-h" || a == "--help") return usage();
      else throw vlasim::ConfigError("unknown option " + a);
    }
    vlasim::ModelSizeSpec spec;
    bool have_spec = false;
    auto load_model = [&](const vlasim::KvFile& kv, const std::string& pre) {
      spec.bytes_hi = kv.get_double(pre + "bytes_hi", spec.bytes_hi);
      spec.bytes_lo = kv.get_double(pre + "bytes_lo", spec.bytes_lo);
      spec.scale_bytes = kv.get_double(pre + "scale_bytes", spec.scale_bytes);
      const std::string cp = pre + "component.";
      for (const auto& [key, e] : kv.entries()) {
        if (key.rfind(cp, 0) != 0) continue;
        std::istringstream ss(e.value);
        vlasim::ModelComponent c;
        c.name = key.substr(cp.size());
        std::string q, g;
        if (!(ss >> c.params >> q)) throw vlasim::ConfigError(kv.name() + ":" + std::to_string(e.line) +
                                                              ": expected `<params> <quantize|keep> [granularity]`");
        if (q != "quantize" && q != "keep")
          throw vlasim::ConfigError(kv.name() + ":" + std::to_string(e.line) + ": expected quantize or keep, got " + q);
        c.quantize = q == "quantize";
        if (ss >> g) c.granularity = vlasim::Granularity::parse(g);
        spec.components.push_back(c);
        have_spec = true;
      }
    };
    if (!config.empty()) {
      const auto kv = vlasim::KvFile::parse_file(config);
      kv.require_known({"seed", "out", "quantization.fixtures", "quantization.granularities", "quantization.synthetic",
                        "model.bytes_hi", "model.bytes_lo", "model.scale_bytes", "model.component.*"});
      if (!seed_set) seed = kv.get_int("seed", seed);
      if (out_dir.empty()) out_dir = kv.get("out");
      if (fixtures.empty()) fixtures = split_list(kv.get("quantization.fixtures"));
      if (grans.empty()) grans = split_list(kv.get("quantization.granularities"));
      if (synth.empty()) synth = kv.get("quantization.synthetic");
      load_model(kv, "model.");
    }
    if (!model_spec.empty()) {
      const auto kv = vlasim::KvFile::parse_file(model_spec);
      kv.require_known({"bytes_hi", "bytes_lo", "scale_bytes", "component.*"});
      load_model(kv, "");
    }
    if (grans.empty()) grans = {"tensor", "channel:0", "block"};
    std::vector<std::pair<std::string, vlasim::Tensor>> tensors;
    for (const auto& f : fixtures) tensors.emplace_back(f, vlasim::read_tensor(f));
    if (!synth.empty()) {
      const auto x = synth.find('x');
      if (x == std::string::npos) throw vlasim::ConfigError("synthetic shape must be ROWSxCOLS, got " + synth);
      tensors.emplace_back("synthetic:" + synth,
                           synthetic(std::stoll(synth.substr(0, x)), std::stoll(synth.substr(x + 1)), std::uint64_t(seed)));
    }
    if (tensors.empty() && !have_spec) return usage();

    std::ostringstream table;
    table << "fixture\tgranularity\tgroups\tmax_rel\tmse\tfp8_bytes\tcompression\n";
    for (const auto& [name, t] : tensors) {
      for (const auto& gs : grans) {
        const auto g = vlasim::Granularity::parse(gs);
        const auto qt = vlasim::quantize(t, g);
        const auto m = vlasim::quant_error(t, qt);
        const double bytes = double(qt.codes.size()) + 4.0 * double(qt.scales.size());
        const double comp = 1.0 - bytes / (2.0 * double(qt.codes.size()));  // vs 2-byte (bf16) storage
        char line[512];
        std::snprintf(line, sizeof(line), "%s\t%s\t%zu\t%.9g\t%.9g\t%.0f\t%.6f\n", name.c_str(), g.name().c_str(),
                      qt.scales.size(), m.max_rel, m.mse, bytes, comp);
        table << line;
      }
    }
    std::ostringstream ctab;
    if (have_spec) {
      ctab << "component\tparams\tquantized\tgranularity\n";
      for (const auto& c : spec.components)
        ctab << c.name << "\t" << c.params << "\t" << (c.quantize ? "yes" : "no") << "\t" << c.granularity.name()
             << "\n";
      char line[128];
      std::snprintf(line, sizeof(line), "compression_ratio\t%.6f\n", vlasim::compression_ratio(spec));
      ctab << line;
    }
    std::fputs(table.str().c_str(), stdout);
    std::fputs(ctab.str().c_str(), stdout);
    if (!out_dir.empty()) {
      ::mkdir(out_dir.c_str(), 0755);
      std::ofstream(out_dir + "/quantbench.tsv") << table.str();
      if (have_spec) std::ofstream(out_dir + "/compression.tsv") << ctab.str();
    }
    return 0;
  } catch (const vlasim::ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
