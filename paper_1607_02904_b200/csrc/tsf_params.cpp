// Tersoff parameter-file parser (grammar of proj/src/params.cpp:119-192).
#include "tsf_params.hpp"

#include <charconv>
#include <cmath>
#include <fstream>
#include <sstream>

namespace tsf {

namespace {

struct Word {
  std::string text;
  int line;
};

// '#' starts a comment running to the end of the line; blanks are space,
// tab and CR; entries may wrap across lines (params.cpp:21-55).
std::vector<Word> split_words(std::string_view text) {
  std::vector<Word> words;
  int line = 1;
  bool comment = false;
  std::string cur;
  int cur_line = 1;
  auto emit = [&] {
    if (!cur.empty()) words.push_back({std::move(cur), cur_line});
    cur.clear();
  };
  for (char ch : text) {
    if (ch == '\n') {
      emit();
      comment = false;
      ++line;
    } else if (comment) {
    } else if (ch == '#') {
      emit();
      comment = true;
    } else if (ch == ' ' || ch == '\t' || ch == '\r') {
      emit();
    } else {
      if (cur.empty()) cur_line = line;
      cur += ch;
    }
  }
  emit();
  return words;
}

constexpr const char* kNames[14] = {"m", "gamma", "lambda3", "c", "d", "h", "eta",
                                    "beta", "lambda2", "B", "R", "D", "lambda1", "A"};

double to_number(const Word& w, std::string_view src, const char* field) {
  double v = 0;
  const char* b = w.text.data();
  const char* e = b + w.text.size();
  auto res = std::from_chars(b, e, v);
  if (res.ec != std::errc{} || res.ptr != e)
    throw ParseError(std::string(src) + ":" + std::to_string(w.line) +
                     ": expected a number for field '" + field + "', got '" + w.text + "'");
  return v;
}

// Field constraints of params.cpp:74-92.  One extension (LAMMPS-format
// files): a cross row (i, j, k) with j != k may carry
// eta = 0 — LAMMPS SiC-type files write n = beta = 0 there, because the bond
// order b_ij and the pair terms only ever read the (i, j, j) row
// (potential.hpp:204-222); rows (i, j, j) keep the reference's eta > 0.
void check_entry(const Entry& e, const std::string& who, bool cross) {
  const double v[14] = {double(e.m), e.gamma, e.lambda3, e.c, e.d, e.h, e.eta,
                        e.beta, e.lambda2, e.big_b, e.big_r, e.big_d, e.lambda1, e.big_a};
  auto bad = [&](const std::string& why) { throw ParseError("entry " + who + ": " + why); };
  for (int f = 0; f < 14; ++f)
    if (!std::isfinite(v[f])) bad(std::string("field '") + kNames[f] + "' is not finite");
  if (e.m != 1 && e.m != 3) bad("field 'm' must be 1 or 3");
  if (!(e.big_d > 0)) bad("field 'D' must be positive");
  if (!(e.big_r > e.big_d)) bad("field 'R' must exceed D");
  if (cross ? !(e.eta >= 0) : !(e.eta > 0))
    bad(cross ? "field 'eta' must be non-negative" : "field 'eta' must be positive");
  if (e.beta < 0) bad("field 'beta' must be non-negative");
  if (e.d == 0) bad("field 'd' must be nonzero");
  if (e.big_a < 0) bad("field 'A' must be non-negative");
  if (e.big_b < 0) bad("field 'B' must be non-negative");
  if (e.gamma < 0) bad("field 'gamma' must be non-negative");
}

std::string shortest(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, r.ptr);
}

}  // namespace

Params::Params(std::vector<std::string> species, std::vector<Entry> entries)
    : species_(std::move(species)), entries_(std::move(entries)) {
  const std::size_t s = species_.size();
  if (s == 0) throw ParseError("parameter table has no species");
  if (entries_.size() != s * s * s)
    throw ParseError("parameter table needs " + std::to_string(s * s * s) + " entries for " +
                     std::to_string(s) + " species, got " + std::to_string(entries_.size()));
  for (std::size_t i = 0; i < s; ++i)
    for (std::size_t j = 0; j < s; ++j)
      for (std::size_t k = 0; k < s; ++k)
        check_entry(entries_[(i * s + j) * s + k],
                    species_[i] + " " + species_[j] + " " + species_[k], j != k);
  for (const Entry& e : entries_) r_cut_max_ = std::max(r_cut_max_, e.cutoff());
}

int Params::species_id(std::string_view name) const {
  for (std::size_t i = 0; i < species_.size(); ++i)
    if (species_[i] == name) return int(i);
  return -1;
}

std::vector<double> Params::flat_rows() const {
  std::vector<double> rows;
  rows.reserve(entries_.size() * kFieldCount);
  for (const Entry& e : entries_) {
    const double cut = e.cutoff();
    const double r[kFieldCount] = {e.big_a, e.big_b, e.lambda1, e.lambda2, e.lambda3,
                                   e.beta,  e.eta,   e.c,       e.d,       e.h,
                                   e.gamma, double(e.m), e.big_r, e.big_d, cut, cut * cut};
    rows.insert(rows.end(), r, r + kFieldCount);
  }
  return rows;
}

bool Params::ramp_depends_on_ik_only() const {
  const int s = species_count();
  for (int i = 0; i < s; ++i)
    for (int k = 0; k < s; ++k)
      for (int j = 0; j < s; ++j) {
        const Entry& a = entry(i, k, k);
        const Entry& b = entry(i, j, k);
        if (a.big_r != b.big_r || a.big_d != b.big_d) return false;
      }
  return true;
}

std::string Params::serialize() const {
  std::string out =
      "# element1 element2 element3 m gamma lambda3 c d h eta beta lambda2 B R D lambda1 A\n";
  const int s = species_count();
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j)
      for (int k = 0; k < s; ++k) {
        const Entry& e = entry(i, j, k);
        out += species_[i] + " " + species_[j] + " " + species_[k] + " " + std::to_string(e.m);
        for (double v : {e.gamma, e.lambda3, e.c, e.d, e.h, e.eta, e.beta, e.lambda2, e.big_b,
                         e.big_r, e.big_d, e.lambda1, e.big_a})
          out += " " + shortest(v);
        out += "\n";
      }
  return out;
}

Params parse_params(std::string_view text, std::string_view src) {
  const std::vector<Word> w = split_words(text);
  if (w.empty()) throw ParseError(std::string(src) + ": no entries found");
  if (w.size() % 17 != 0)
    throw ParseError(std::string(src) + ":" + std::to_string(w.back().line) +
                     ": truncated entry (each entry needs 3 names and 14 numbers)");
  std::vector<std::string> names;
  auto id_of = [&](const std::string& n) {
    for (std::size_t i = 0; i < names.size(); ++i)
      if (names[i] == n) return int(i);
    names.push_back(n);
    return int(names.size()) - 1;
  };
  struct Pending {
    int t[3];
    Entry e;
    int line;
  };
  std::vector<Pending> pend;
  for (std::size_t b = 0; b < w.size(); b += 17) {
    Pending p;
    p.line = w[b].line;
    for (int q = 0; q < 3; ++q) p.t[q] = id_of(w[b + q].text);
    double v[14];
    for (int f = 0; f < 14; ++f) v[f] = to_number(w[b + 3 + f], src, kNames[f]);
    if (v[0] != std::floor(v[0]))
      throw ParseError(std::string(src) + ":" + std::to_string(w[b + 3].line) +
                       ": field 'm' must be an integer");
    Entry& e = p.e;
    e.m = int(v[0]);
    e.gamma = v[1];
    e.lambda3 = v[2];
    e.c = v[3];
    e.d = v[4];
    e.h = v[5];
    e.eta = v[6];
    e.beta = v[7];
    e.lambda2 = v[8];
    e.big_b = v[9];
    e.big_r = v[10];
    e.big_d = v[11];
    e.lambda1 = v[12];
    e.big_a = v[13];
    pend.push_back(p);
  }
  const int s = int(names.size());
  std::vector<Entry> table(std::size_t(s) * s * s);
  std::vector<char> have(table.size(), 0);
  for (const Pending& p : pend) {
    const std::size_t idx = std::size_t((p.t[0] * s + p.t[1]) * s + p.t[2]);
    if (have[idx])
      throw ParseError(std::string(src) + ":" + std::to_string(p.line) +
                       ": duplicate entry for triplet " + names[p.t[0]] + " " +
                       names[p.t[1]] + " " + names[p.t[2]]);
    have[idx] = 1;
    table[idx] = p.e;
  }
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j)
      for (int k = 0; k < s; ++k)
        if (!have[std::size_t((i * s + j) * s + k)])
          throw ParseError(std::string(src) + ": missing entry for triplet " + names[i] + " " +
                           names[j] + " " + names[k]);
  return Params(std::move(names), std::move(table));
}

Params load_params(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open parameter file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_params(ss.str(), path);
}

Params builtin_silicon() {
  // Si(B), Tersoff PRB 38, 9902 (1988); the values of proj/data/Si.tersoff.
  return parse_params(
      "Si Si Si 3.0 1.0 1.3258 4.8381 2.0417 0.0000 22.956 0.33675 1.3258 95.373 3.0 0.2 "
      "3.2394 3264.7\n",
      "<builtin Si>");
}

}  // namespace tsf
