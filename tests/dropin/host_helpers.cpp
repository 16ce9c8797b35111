// host_helpers.cpp — evaluates the reconstructed C++ host helpers of libvlasim.so (no GPU needed) on a
// list of cases read from stdin and prints one JSON object per case, so tests/test_host_helpers.py can
// hold the C++ copy, the Python copy (paper_2603_11101_b200.packing / quant) and the oracle to the same
// values (padding_rate, dynamic_pad_length, attention_flops, PackingStats; plus
// prune_view, block_partition, compression_ratio and the kv config parser).
//
// stdin: one case per line:
//   lengths <pad_to> <head_dim> <l0> <l1> ...      → padding_rate, dynamic_pad_length, attention_flops
//   stats <capacity> <pad_to> <head_dim> <nbins> <m0> <l..>... → packing_stats over the given bins
//   blocks <rows> <cols>                           → block_partition count and Σ area
//   compression <bytes_hi> <bytes_lo> <scale_bytes> <params> <q|k> ...  → compression_ratio
//   prune <text> <view>=<n>... -- <view_to_prune> → total_len after prune_view (or "error")
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "vlasim/packing/pack.hpp"
#include "vlasim/packing/sample.hpp"
#include "vlasim/quant/compression.hpp"
#include "vlasim/util/errors.hpp"

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    std::istringstream ss(line);
    std::string kind;
    if (!(ss >> kind)) continue;
    try {
      if (kind == "lengths") {
        std::int64_t pad_to, d, x;
        ss >> pad_to >> d;
        std::vector<std::int64_t> L;
        while (ss >> x) L.push_back(x);
        std::printf("{\"padding_rate\": %.17g, \"dynamic_pad_length\": %lld, \"flops_fixed\": %.17g, "
                    "\"flops_packed\": %.17g}\n",
                    vlasim::padding_rate(L, pad_to), (long long)vlasim::dynamic_pad_length(L),
                    vlasim::attention_flops(L, d, pad_to), vlasim::attention_flops(L, d));
      } else if (kind == "stats") {
        std::int64_t cap, pad_to, d, nb;
        ss >> cap >> pad_to >> d >> nb;
        std::vector<vlasim::PackedSequence> bins;
        std::vector<std::int64_t> L;
        for (std::int64_t b = 0; b < nb; ++b) {
          std::int64_t m;
          ss >> m;
          vlasim::PackedSequence p;
          p.capacity = cap;
          for (std::int64_t j = 0; j < m; ++j) {
            std::int64_t l;
            ss >> l;
            p.member_ids.push_back(std::int64_t(L.size()));
            p.member_lens.push_back(l);
            L.push_back(l);
          }
          bins.push_back(p);
        }
        const auto st = vlasim::packing_stats(L, bins, pad_to, d);
        std::printf("{\"bins_used\": %lld, \"fill_rate\": %.17g, \"padding_rate_before\": %.17g, "
                    "\"padding_rate_after\": %.17g, \"flops_fixed\": %.17g, \"flops_packed\": %.17g}\n",
                    (long long)st.bins_used, st.fill_rate, st.padding_rate_before, st.padding_rate_after,
                    st.attention_flops_fixed, st.attention_flops_packed);
      } else if (kind == "blocks") {
        std::int64_t r, c;
        ss >> r >> c;
        const auto b = vlasim::block_partition({r, c});
        std::int64_t area = 0;
        for (const auto& e : b) area += e.rows * e.cols;
        std::printf("{\"blocks\": %zu, \"area\": %lld}\n", b.size(), (long long)area);
      } else if (kind == "compression") {
        vlasim::ModelSizeSpec spec;
        ss >> spec.bytes_hi >> spec.bytes_lo >> spec.scale_bytes;
        std::int64_t p;
        std::string q;
        while (ss >> p >> q) {
          vlasim::ModelComponent c;
          c.name = "c" + std::to_string(spec.components.size());
          c.params = p;
          c.quantize = q == "q";
          spec.components.push_back(c);
        }
        std::printf("{\"compression_ratio\": %.17g}\n", vlasim::compression_ratio(spec));
      } else if (kind == "prune") {
        std::int64_t text;
        ss >> text;
        std::map<std::string, std::int64_t> views;
        std::string tok, view;
        while (ss >> tok && tok != "--") {
          const auto eq = tok.find('=');
          views[tok.substr(0, eq)] = std::stoll(tok.substr(eq + 1));
        }
        ss >> view;
        const auto s = vlasim::prune_view(vlasim::make_sample(0, views, text), view);
        std::printf("{\"total_len\": %lld}\n", (long long)s.total_len);
      } else {
        std::printf("{\"error\": \"unknown case\"}\n");
      }
    } catch (const vlasim::ConfigError& e) {
      std::printf("{\"config_error\": \"%s\"}\n", e.what());
    }
  }
  return 0;
}
