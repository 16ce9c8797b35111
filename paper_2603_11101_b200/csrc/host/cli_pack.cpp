// cli_pack.cpp — `vlasim_pack`: the reference's `pack` subcommand on the GPU packer.
//
//   vlasim_pack --capacity N (--corpus FILE | --synthetic N LO HI [SEED]) [--pad-to P] [--head-dim D]
//               [--prune VIEW] [--greedy] [--manifest]
//
// Corpus file (flat tabular text): one sample per line, `id text_len [view=count ...]`,
// '#' starts a comment.  Prints PackingStats and, with --manifest, every bin's
// members and cu_seqlens.  Exit codes follow SPEC.md:703: 0 ok, 2 ConfigError, 3 runtime error.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "vlasim/packing/pack.hpp"
#include "vlasim/packing/sample.hpp"
#include "vlasim/util/errors.hpp"
#include "vlasim/util/rng.hpp"

namespace {

std::vector<vlasim::SampleLen> read_corpus(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw vlasim::ConfigError("cannot open corpus file " + path);
  std::vector<vlasim::SampleLen> out;
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (auto h = line.find('#'); h != std::string::npos) line.resize(h);
    std::istringstream ss(line);
    long long id, text;
    if (!(ss >> id)) continue;
    if (!(ss >> text)) throw vlasim::ConfigError(path + ":" + std::to_string(lineno) + ": expected `id text_len`");
    std::map<std::string, std::int64_t> views;
    std::string tok;
    while (ss >> tok) {
      auto eq = tok.find('=');
      if (eq == std::string::npos) throw vlasim::ConfigError(path + ":" + std::to_string(lineno) + ": bad view " + tok);
      views[tok.substr(0, eq)] = std::stoll(tok.substr(eq + 1));
    }
    out.push_back(vlasim::make_sample(id, views, text));
  }
  return out;
}

int usage() {
  std::fprintf(stderr,
               "usage: vlasim_pack --capacity N (--corpus FILE | --synthetic N LO HI [SEED]) [--pad-to P]\n"
               "                   [--head-dim D] [--prune VIEW] [--greedy] [--manifest]\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    std::int64_t capacity = 0, pad_to = 0, head_dim = 128;
    std::string corpus, prune;
    long long syn_n = 0, syn_lo = 16, syn_hi = 512, seed = 42;
    bool manifest = false, greedy = false;
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      auto need = [&](int k) {
        if (i + k >= argc) throw vlasim::ConfigError("missing value for " + a);
      };
      if (a == "--capacity") { need(1); capacity = std::stoll(argv[++i]); }
      else if (a == "--corpus") { need(1); corpus = argv[++i]; }
      else if (a == "--synthetic") {
        need(3);
        syn_n = std::stoll(argv[++i]);
        syn_lo = std::stoll(argv[++i]);
        syn_hi = std::stoll(argv[++i]);
        if (i + 1 < argc && argv[i + 1][0] != '-') seed = std::stoll(argv[++i]);
      } else if (a == "--pad-to") { need(1); pad_to = std::stoll(argv[++i]); }
      else if (a == "--head-dim") { need(1); head_dim = std::stoll(argv[++i]); }
      else if (a == "--prune") { need(1); prune = argv[++i]; }
      else if (a == "--manifest") manifest = true;
      else if (a == "--greedy") greedy = true;  // arrival-order first fit
      else throw vlasim::ConfigError("unknown option " + a);
    }
    if (capacity <= 0 || (corpus.empty() == (syn_n == 0))) return usage();
    std::vector<std::int64_t> lengths;
    if (!corpus.empty()) {
      for (auto s : read_corpus(corpus)) {
        if (!prune.empty() && s.view_lens.count(prune)) s = vlasim::prune_view(s, prune);
        lengths.push_back(s.total_len);
      }
    } else {
      auto rng = vlasim::make_rng(std::uint64_t(seed), "lengths", 0);
      for (long long i = 0; i < syn_n; ++i) lengths.push_back(vlasim::uniform_int(rng, syn_lo, syn_hi));
    }
    if (lengths.empty()) throw vlasim::ConfigError("empty corpus");
    if (pad_to <= 0) pad_to = vlasim::dynamic_pad_length(lengths);
    const auto bins = greedy ? vlasim::pack_greedy(lengths, capacity) : vlasim::pack_ffd(lengths, capacity);
    const auto st = vlasim::packing_stats(lengths, bins, pad_to, head_dim);
    std::printf("{\"samples\": %zu, \"capacity\": %lld, \"bins_used\": %lld, \"fill_rate\": %.6f, "
                "\"padding_rate_before\": %.6f, \"padding_rate_after\": %.6f, \"attention_flops_fixed\": %.6e, "
                "\"attention_flops_packed\": %.6e}\n",
                lengths.size(), (long long)capacity, (long long)st.bins_used, st.fill_rate, st.padding_rate_before,
                st.padding_rate_after, st.attention_flops_fixed, st.attention_flops_packed);
    if (manifest) {
      for (std::size_t b = 0; b < bins.size(); ++b) {
        std::printf("bin %zu fill %lld members", b, (long long)bins[b].fill());
        for (auto id : bins[b].member_ids) std::printf(" %lld", (long long)id);
        std::printf(" cu_seqlens");
        for (auto c : vlasim::cu_seqlens(bins[b])) std::printf(" %lld", (long long)c);
        std::printf("\n");
      }
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
