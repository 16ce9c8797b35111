// cli_pack.cpp — `vlasim_pack`: the reference's `pack` subcommand on the GPU packer.
//
//   vlasim_pack [--config FILE] [--capacity N] [--corpus FILE | --synthetic N LO HI] [--seed S]
//               [--pad-to P] [--head-dim D] [--prune VIEW] [--greedy] [--manifest] [--out DIR]
//
// Corpus file (flat tabular text): one sample per line, `id text_len [view=count ...]`,
// '#' starts a comment.  Prints PackingStats and, with --manifest, every bin's
// members and cu_seqlens; --out DIR writes them to DIR/stats.json and DIR/manifest.tsv.  --prune
// applies prune_view to every sample (a sample without the view is an error).
// Config (strict schema — an unknown key is rejected naming it; flags override):
//   seed = 42      out = DIR
//   [packing]   corpus = FILE   capacity = 8192   algorithm = ffd | greedy   pad_to = P
//               head_dim = D    prune_view = VIEW   manifest = yes | no
//   [synthetic] n = 512   lo = 16   hi = 512
// Exit codes follow SPEC.md:703: 0 ok, 2 ConfigError, 3 runtime error.
#include <sys/stat.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "vlasim/packing/pack.hpp"
#include "vlasim/packing/sample.hpp"
#include "vlasim/util/errors.hpp"
#include "vlasim/util/kv_file.hpp"
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
               "usage: vlasim_pack [--config FILE] [--capacity N] [--corpus FILE | --synthetic N LO HI [SEED]]\n"
               "                   [--seed S] [--pad-to P] [--head-dim D] [--prune VIEW] [--greedy] [--manifest]\n"
               "                   [--out DIR]\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    std::int64_t capacity = 0, pad_to = 0, head_dim = 128;
    std::string corpus, prune, out_dir, config;
    long long syn_n = 0, syn_lo = 16, syn_hi = 512, seed = 42;
    bool manifest = false, greedy = false, seed_set = false, greedy_set = false, manifest_set = false;
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      auto need = [&](int k) {
        if (i + k >= argc) throw vlasim::ConfigError("missing value for " + a);
      };
      if (a == "--config") { need(1); config = argv[++i]; }
      else if (a == "--capacity") { need(1); capacity = std::stoll(argv[++i]); }
      else if (a == "--corpus") { need(1); corpus = argv[++i]; }
      else if (a == "--synthetic") {
        need(3);
        syn_n = std::stoll(argv[++i]);
        syn_lo = std::stoll(argv[++i]);
        syn_hi = std::stoll(argv[++i]);
        if (i + 1 < argc && argv[i + 1][0] != '-') { seed = std::stoll(argv[++i]); seed_set = true; }
      } else if (a == "--seed") { need(1); seed = std::stoll(argv[++i]); seed_set = true; }
      else if (a == "--pad-to") { need(1); pad_to = std::stoll(argv[++i]); }
      else if (a == "--head-dim") { need(1); head_dim = std::stoll(argv[++i]); }
      else if (a == "--prune") { need(1); prune = argv[++i]; }
      else if (a == "--out") { need(1); out_dir = argv[++i]; }
      else if (a == "--manifest") { manifest = true; manifest_set = true; }
      else if (a == "--greedy") { greedy = true; greedy_set = true; }  // arrival-order first fit
      else if (a == "-h" || a == "--help") return usage();
      else throw vlasim::ConfigError("unknown option " + a);
    }
    if (!config.empty()) {
      const auto kv = vlasim::KvFile::parse_file(config);
      kv.require_known({"seed", "out", "packing.corpus", "packing.capacity", "packing.algorithm", "packing.pad_to",
                        "packing.head_dim", "packing.prune_view", "packing.manifest", "synthetic.n", "synthetic.lo",
                        "synthetic.hi"});
      if (!seed_set) seed = kv.get_int("seed", seed);
      if (out_dir.empty()) out_dir = kv.get("out");
      if (corpus.empty() && syn_n == 0) {
        corpus = kv.get("packing.corpus");
        syn_n = kv.get_int("synthetic.n", 0);
        syn_lo = kv.get_int("synthetic.lo", syn_lo);
        syn_hi = kv.get_int("synthetic.hi", syn_hi);
      }
      if (capacity == 0) capacity = kv.get_int("packing.capacity", 0);
      if (pad_to == 0) pad_to = kv.get_int("packing.pad_to", 0);
      head_dim = kv.get_int("packing.head_dim", head_dim);
      if (prune.empty()) prune = kv.get("packing.prune_view");
      const std::string algo = kv.get("packing.algorithm", "ffd");
      if (algo != "ffd" && algo != "greedy")
        throw vlasim::ConfigError(config + ":" + std::to_string(kv.entries().at("packing.algorithm").line) +
                                  ": packing.algorithm must be ffd or greedy, got '" + algo + "'");
      if (!greedy_set) greedy = algo == "greedy";
      const std::string mf = kv.get("packing.manifest", "no");
      if (mf != "yes" && mf != "no") throw vlasim::ConfigError(config + ": packing.manifest must be yes or no");
      if (!manifest_set) manifest = mf == "yes";
    }
    if (capacity <= 0 || (corpus.empty() == (syn_n == 0))) return usage();
    std::vector<std::int64_t> lengths;
    if (!corpus.empty()) {
      for (auto s : read_corpus(corpus)) {
        if (!prune.empty()) s = vlasim::prune_view(s, prune);  // unknown view → ConfigError
        lengths.push_back(s.total_len);
      }
    } else {
      if (!prune.empty()) throw vlasim::ConfigError("--prune needs a corpus with per-view token counts");
      auto rng = vlasim::make_rng(std::uint64_t(seed), "lengths", 0);
      for (long long i = 0; i < syn_n; ++i) lengths.push_back(vlasim::uniform_int(rng, syn_lo, syn_hi));
    }
    if (lengths.empty()) throw vlasim::ConfigError("empty corpus");
    if (pad_to <= 0) pad_to = vlasim::dynamic_pad_length(lengths);
    const auto bins = greedy ? vlasim::pack_greedy(lengths, capacity) : vlasim::pack_ffd(lengths, capacity);
    const auto st = vlasim::packing_stats(lengths, bins, pad_to, head_dim);
    char stats[512];
    std::snprintf(stats, sizeof(stats),
                  "{\"samples\": %zu, \"capacity\": %lld, \"bins_used\": %lld, \"fill_rate\": %.6f, "
                  "\"padding_rate_before\": %.6f, \"padding_rate_after\": %.6f, \"attention_flops_fixed\": %.6e, "
                  "\"attention_flops_packed\": %.6e}\n",
                  lengths.size(), (long long)capacity, (long long)st.bins_used, st.fill_rate, st.padding_rate_before,
                  st.padding_rate_after, st.attention_flops_fixed, st.attention_flops_packed);
    std::ostringstream man;
    for (std::size_t b = 0; b < bins.size(); ++b) {
      man << "bin " << b << " fill " << bins[b].fill() << " members";
      for (auto id : bins[b].member_ids) man << " " << id;
      man << " cu_seqlens";
      for (auto c : vlasim::cu_seqlens(bins[b])) man << " " << c;
      man << "\n";
    }
    std::fputs(stats, stdout);
    if (manifest) std::fputs(man.str().c_str(), stdout);
    if (!out_dir.empty()) {
      ::mkdir(out_dir.c_str(), 0755);
      std::ofstream(out_dir + "/stats.json") << stats;
      std::ofstream(out_dir + "/manifest.tsv") << man.str();
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
