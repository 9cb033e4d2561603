// Host-side Tersoff parameter table: parsing, validation, flattening.
//
// Same file grammar, species interning and validation as the reference
// (proj/src/params.cpp:119-192 grammar, :74-92 constraints, :94-111 table),
// written fresh.  Errors carry the reference's wording so callers that match
// on messages keep working.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace tsf {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// One ordered (i, j, k) species triplet; members in file column order
// (params.hpp:16-36).  Two-body terms read (i,j,j), three-body terms (i,j,k).
struct Entry {
  int m = 1;
  double gamma = 1, lambda3 = 0, c = 0, d = 1, h = 0, eta = 1, beta = 0, lambda2 = 0,
         big_b = 0, big_r = 0, big_d = 0, lambda1 = 0, big_a = 0;
  double cutoff() const { return big_r + big_d; }
};

// Column order of a flattened row (params.hpp:78-83).
enum Field : int { kA = 0, kB, kLam1, kLam2, kLam3, kBeta, kEta, kC, kD, kH, kGamma, kM,
                   kBigR, kBigD, kCut, kCutSq, kFieldCount };

class Params {
 public:
  Params(std::vector<std::string> species, std::vector<Entry> entries);

  int species_count() const { return int(species_.size()); }
  const std::vector<std::string>& species() const { return species_; }
  int species_id(std::string_view name) const;
  const Entry& entry(int i, int j, int k) const {
    const int s = species_count();
    return entries_[std::size_t((i * s + j) * s + k)];
  }
  double r_cut_max() const { return r_cut_max_; }
  // S^3 x 16 doubles, FlatParams<double> layout.
  std::vector<double> flat_rows() const;
  // True when the cutoff ramp (R, D) of (i, j, k) depends on (i, k) only, so
  // fc(r_ik) can be evaluated once per neighbor instead of once per triplet.
  bool ramp_depends_on_ik_only() const;
  std::string serialize() const;

 private:
  std::vector<std::string> species_;
  std::vector<Entry> entries_;
  double r_cut_max_ = 0;
};

Params parse_params(std::string_view text, std::string_view source_name);
Params load_params(const std::string& path);
Params builtin_silicon();

}  // namespace tsf
