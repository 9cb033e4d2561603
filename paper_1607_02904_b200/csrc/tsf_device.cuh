// Device-side geometry shared by the neighbor, filter, force and MD kernels.
//
// HBM layout:
//   pos     double4[n]        {x, y, z, species}  — one 32 B sector per gather
//   forces  double[n][3]      AoS, the layout of std::vector<Vec3>
//   lists   int32 ELL, column-major: nbr[s * npad + i], count[i]
//           (consecutive atoms read consecutive words: coalesced)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tsf {

constexpr int kMaxSpecies = 4;          // S^3 <= 64 parameter rows
constexpr int kBlock = 128;             // threads per block, force + list kernels

struct Box {
  double len[3];
  int per[3];
};

// minimum_image_1d(d, L) = d - L * floor(d / L + 0.5) (proj/include/tmd/box.hpp:28-30)
// with the reference's exact rounding sequence: IEEE divide, no contraction.
__device__ __forceinline__ double min_image_exact(double d, double len) {
  const double q = __dadd_rn(__ddiv_rn(d, len), 0.5);
  return __dsub_rn(d, __dmul_rn(len, floor(q)));
}

// Bitwise the same value as min_image_exact.  |d| <= L/4 gives
// floor(d/L + 0.5) == 0 under any rounding, hence d itself, so the divide
// only runs for displacements that cross a periodic face.
__device__ __forceinline__ double min_image(double d, double len) {
  if (fabs(d) <= 0.25 * len) return d;
  return min_image_exact(d, len);
}

// norm_sq (vec3.hpp:25-30), left to right, no FMA.
__device__ __forceinline__ double norm_sq_exact(double x, double y, double z) {
  return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
}

__device__ __forceinline__ void displacement(const double4& a, const double4& b, const Box& box,
                                             double& dx, double& dy, double& dz) {
  dx = __dsub_rn(b.x, a.x);
  dy = __dsub_rn(b.y, a.y);
  dz = __dsub_rn(b.z, a.z);
  if (box.per[0]) dx = min_image(dx, box.len[0]);
  if (box.per[1]) dy = min_image(dy, box.len[1]);
  if (box.per[2]) dz = min_image(dz, box.len[2]);
}

__device__ __forceinline__ int species_of(const double4& p) { return int(p.w); }


}  // namespace tsf
