// kv_file.cpp — strict-schema structured-text configs (include/vlasim/util/kv_file.hpp).
#include "vlasim/util/kv_file.hpp"

#include <cctype>
#include <fstream>
#include <sstream>

#include "vlasim/util/errors.hpp"

namespace vlasim {
namespace {

std::string trim(std::string_view s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string_view::npos) return {};
  const auto e = s.find_last_not_of(" \t\r");
  return std::string(s.substr(b, e - b + 1));
}

bool valid_key(const std::string& k) {
  if (k.empty()) return false;
  for (char c : k)
    if (!(std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.')) return false;
  return true;
}

}  // namespace

KvFile KvFile::parse_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open config file " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return parse_text(ss.str(), path);
}

KvFile KvFile::parse_text(std::string_view text, const std::string& name) {
  KvFile f;
  f.name_ = name;
  std::string section;
  int lineno = 0;
  std::size_t pos = 0;
  while (pos <= text.size()) {
    const std::size_t nl = text.find('\n', pos);
    std::string_view raw = text.substr(pos, nl == std::string_view::npos ? std::string_view::npos : nl - pos);
    pos = nl == std::string_view::npos ? text.size() + 1 : nl + 1;
    ++lineno;
    const auto hash = raw.find('#');
    const std::string line = trim(hash == std::string_view::npos ? raw : raw.substr(0, hash));
    if (line.empty()) continue;
    const std::string where = name + ":" + std::to_string(lineno);
    if (line.front() == '[') {
      if (line.back() != ']') throw ConfigError(where + ": malformed section header '" + line + "'");
      section = trim(std::string_view(line).substr(1, line.size() - 2));
      if (!valid_key(section)) throw ConfigError(where + ": bad section name '" + section + "'");
      continue;
    }
    const auto eq = line.find('=');
    if (eq == std::string::npos) throw ConfigError(where + ": expected `key = value`, got '" + line + "'");
    const std::string key = trim(std::string_view(line).substr(0, eq));
    const std::string value = trim(std::string_view(line).substr(eq + 1));
    if (!valid_key(key)) throw ConfigError(where + ": bad key '" + key + "'");
    const std::string full = section.empty() ? key : section + "." + key;
    if (f.entries_.count(full))
      throw ConfigError(where + ": duplicate key '" + full + "' (first at line " +
                        std::to_string(f.entries_[full].line) + ")");
    f.entries_[full] = Entry{value, lineno};
  }
  return f;
}

void KvFile::require_known(const std::vector<std::string>& allowed) const {
  for (const auto& [key, e] : entries_) {
    bool ok = false;
    for (const auto& a : allowed)  // "prefix.*" admits every key under the prefix
      ok = ok || a == key || (a.size() > 1 && a.back() == '*' && key.rfind(a.substr(0, a.size() - 1), 0) == 0);
    if (!ok) throw ConfigError(name_ + ":" + std::to_string(e.line) + ": unknown key '" + key + "'");
  }
}

std::string KvFile::get(const std::string& key, const std::string& def) const {
  auto it = entries_.find(key);
  return it == entries_.end() ? def : it->second.value;
}

std::int64_t KvFile::get_int(const std::string& key, std::int64_t def) const {
  auto it = entries_.find(key);
  if (it == entries_.end()) return def;
  std::size_t used = 0;
  std::int64_t v = 0;
  try {
    v = std::stoll(it->second.value, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != it->second.value.size())
    throw ConfigError(name_ + ":" + std::to_string(it->second.line) + ": key '" + key + "' needs an integer, got '" +
                      it->second.value + "'");
  return v;
}

double KvFile::get_double(const std::string& key, double def) const {
  auto it = entries_.find(key);
  if (it == entries_.end()) return def;
  std::size_t used = 0;
  double v = 0;
  try {
    v = std::stod(it->second.value, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != it->second.value.size())
    throw ConfigError(name_ + ":" + std::to_string(it->second.line) + ": key '" + key + "' needs a number, got '" +
                      it->second.value + "'");
  return v;
}

}  // namespace vlasim
