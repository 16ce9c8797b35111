// vlasim/util/kv_file.hpp — structured-text configs with a strict schema (reconstructed drop-in
// header for proj/CMakeLists.txt:16 src/util/kv_file.cpp; contract SPEC.md:652-654, 701-702:
// "unknown keys rejected (strict schema) with the offending key named").
//
// Format: one `key = value` per line; `[section]` prefixes the keys that follow ("section.key");
// '#' starts a comment; blank lines ignored.  A duplicate key, a malformed line or (with
// require_known) a key outside the schema → ConfigError naming the file, line and key.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <string_view>
#include <vector>

namespace vlasim {

class KvFile {
 public:
  struct Entry {
    std::string value;
    int line = 0;
  };

  static KvFile parse_file(const std::string& path);
  static KvFile parse_text(std::string_view text, const std::string& name = "<config>");

  // Strict schema: every key must be one of `allowed` (fully qualified "section.key"; an entry
  // "section.prefix.*" admits every key that starts with "section.prefix.").
  void require_known(const std::vector<std::string>& allowed) const;

  bool has(const std::string& key) const { return entries_.count(key) != 0; }
  std::string get(const std::string& key, const std::string& def = "") const;
  std::int64_t get_int(const std::string& key, std::int64_t def) const;
  double get_double(const std::string& key, double def) const;
  const std::map<std::string, Entry>& entries() const { return entries_; }
  const std::string& name() const { return name_; }

 private:
  std::string name_;
  std::map<std::string, Entry> entries_;
};

}  // namespace vlasim
