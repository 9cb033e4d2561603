// Metal units (proj/include/tmd/units.hpp:10-13) and element masses
// (proj/src/units.cpp:10-27).
#pragma once

#include <string_view>

namespace tsf {

inline constexpr double kMvv2e = 1.0364269e-4;      // (g/mol)(A/ps)^2 -> eV
inline constexpr double kBoltzmann = 8.617333e-5;   // eV/K

inline double element_mass(std::string_view el, double fallback) {
  struct M {
    const char* name;
    double mass;
  };
  static constexpr M table[] = {{"H", 1.008},     {"He", 4.0026},   {"B", 10.81},
                                {"C", 12.011},    {"N", 14.007},    {"O", 15.999},
                                {"Al", 26.9815},  {"Si", 28.0855},  {"P", 30.9738},
                                {"S", 32.06},     {"Ga", 69.723},   {"Ge", 72.63},
                                {"As", 74.9216},  {"In", 114.818},  {"Sn", 118.71},
                                {"Sb", 121.76}};
  for (const M& m : table)
    if (el == m.name) return m.mass;
  return fallback;
}

}  // namespace tsf
