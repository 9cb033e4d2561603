// Synthetic inputs: diamond lattice, jittered lattice, Maxwell-Boltzmann
// velocities.  Bit-identical to the reference generators so the GPU path and
// the CPU oracle can be driven with the same seeded systems:
//   make_diamond_lattice  proj/src/engine.cpp:28-58
//   init_velocities       proj/src/engine.cpp:64-116 (mt19937_64, Box-Muller
//                         cosine branch, COM removal, exact rescale)
//   perturbed_lattice     proj/src/verify.cpp:83-104
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <string_view>
#include <vector>

#include "tsf_params.hpp"
#include "tsf_units.hpp"

namespace tsf {

namespace {

// Conventional cubic cell of the diamond structure: two interpenetrating FCC
// sublattices, the second shifted by a0/4 along the body diagonal.
constexpr double kDiamondBasis[8][3] = {
    {0.00, 0.00, 0.00}, {0.00, 0.50, 0.50}, {0.50, 0.00, 0.50}, {0.50, 0.50, 0.00},
    {0.25, 0.25, 0.25}, {0.25, 0.75, 0.75}, {0.75, 0.25, 0.75}, {0.75, 0.75, 0.25}};

double wrap_into(double x, double len) {
  x -= len * std::floor(x / len);
  if (x < 0.0) x += len;
  if (x >= len) x -= len;
  return x;
}

}  // namespace

void diamond_lattice(int nx, int ny, int nz, double a0, std::int32_t sid, double* xyz,
                     std::int32_t* species, double* box) {
  if (nx < 1 || ny < 1 || nz < 1) throw ConfigError("lattice cell counts must be positive");
  if (!(a0 > 0.0)) throw ConfigError("lattice constant must be positive");
  if (sid < 0) throw ConfigError("species id must be non-negative");
  box[0] = a0 * nx;
  box[1] = a0 * ny;
  box[2] = a0 * nz;
  std::size_t a = 0;
  for (int cx = 0; cx < nx; ++cx)
    for (int cy = 0; cy < ny; ++cy)
      for (int cz = 0; cz < nz; ++cz)
        for (const auto& b : kDiamondBasis) {
          xyz[3 * a + 0] = a0 * (cx + b[0]);
          xyz[3 * a + 1] = a0 * (cy + b[1]);
          xyz[3 * a + 2] = a0 * (cz + b[2]);
          species[a] = sid;
          ++a;
        }
}

void perturbed_lattice(const Params& p, int cells, double jitter, std::uint64_t seed,
                       double* xyz, std::int32_t* species, double* masses, double* box) {
  const double a0 = 1.697 * p.r_cut_max();
  diamond_lattice(cells, cells, cells, a0, 0, xyz, species, box);
  const int ns = p.species_count();
  for (int s = 0; s < ns; ++s) masses[s] = element_mass(p.species()[std::size_t(s)], 28.0);
  std::mt19937_64 rng(seed);
  auto draw = [&](double lo, double hi) {
    return lo + (hi - lo) * (double(rng() >> 11) * 0x1p-53);
  };
  const std::size_t n = std::size_t(cells) * cells * cells * 8;
  for (std::size_t a = 0; a < n; ++a) {
    species[a] = std::int32_t(a % std::size_t(ns));
    for (int c = 0; c < 3; ++c) xyz[3 * a + c] = wrap_into(xyz[3 * a + c] + draw(-jitter, jitter), box[c]);
  }
}

void maxwell_boltzmann(std::int64_t n, const std::int32_t* species, const double* masses,
                       double temperature, std::uint64_t seed, double* v) {
  if (temperature < 0.0) throw ConfigError("temperature must be non-negative");
  if (n == 0) return;
  if (temperature == 0.0) {
    for (std::int64_t q = 0; q < 3 * n; ++q) v[q] = 0.0;
    return;
  }
  std::mt19937_64 rng(seed);
  auto unit = [&] { return double((rng() >> 11) + 1) * 0x1p-53; };  // (0, 1]
  auto normal = [&] {
    const double u1 = unit();
    const double u2 = unit();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
  };
  for (std::int64_t a = 0; a < n; ++a) {
    const double m = masses[species[a]];
    const double sigma = std::sqrt(kBoltzmann * temperature / (m * kMvv2e));
    const double gx = normal();
    const double gy = normal();
    const double gz = normal();
    v[3 * a + 0] = sigma * gx;
    v[3 * a + 1] = sigma * gy;
    v[3 * a + 2] = sigma * gz;
  }
  double mtot = 0.0, px = 0.0, py = 0.0, pz = 0.0;
  for (std::int64_t a = 0; a < n; ++a) {
    const double m = masses[species[a]];
    mtot += m;
    px = px + v[3 * a + 0] * m;
    py = py + v[3 * a + 1] * m;
    pz = pz + v[3 * a + 2] * m;
  }
  const double inv = 1.0 / mtot;
  const double cx = px * inv, cy = py * inv, cz = pz * inv;
  for (std::int64_t a = 0; a < n; ++a) {
    v[3 * a + 0] = v[3 * a + 0] - cx;
    v[3 * a + 1] = v[3 * a + 1] - cy;
    v[3 * a + 2] = v[3 * a + 2] - cz;
  }
  double ke = 0.0;
  for (std::int64_t a = 0; a < n; ++a) {
    const double vx = v[3 * a], vy = v[3 * a + 1], vz = v[3 * a + 2];
    ke += 0.5 * masses[species[a]] * (vx * vx + vy * vy + vz * vz) * kMvv2e;
  }
  const double t_now = 2.0 * ke / (3.0 * double(n) * kBoltzmann);
  if (t_now > 0.0) {
    const double scale = std::sqrt(temperature / t_now);
    for (std::int64_t q = 0; q < 3 * n; ++q) v[q] = v[q] * scale;
  }
}

}  // namespace tsf
