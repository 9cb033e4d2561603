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

// Device-side bounds checks of a checked build (make EXTRA=-DTSF_BOUNDS_CHECK;
// tools/checked_build.sh): every list entry, slot and gather index the hot
// kernels use is asserted in range, and a violation traps with its location.
// compute-sanitizer is not available on this pool, so this build plus the
// small-case sweep (tools/sanitize_case.py) stands in for memcheck.
#ifdef TSF_BOUNDS_CHECK
#include <cstdio>
#define TSF_DCHECK(cond, what)                                                       \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("tsf bounds check failed: %s (%s:%d)\n", what, __FILE__, __LINE__);     \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define TSF_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

namespace tsf {

constexpr int kMaxSpecies = 4;          // S^3 <= 64 parameter rows
constexpr int kBlock = 128;             // threads per block, force + list kernels

struct Box {
  double len[3];
  int per[3];
  double quarter[3];   // len / 4 (exact), min_image's no-wrap bound (set_geometry)
};

// Reference cell grid (neighbor.cpp:50-77): edge >= cutoff + skin.  Atoms are
// stored sorted by cell id (cz ny + cy) nx + cx, so a cell is a slot range.
struct CellGrid {
  int nc[3];
  double org[3], ext[3];
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
__device__ __forceinline__ double min_image(double d, double len, double quarter) {
  if (fabs(d) <= quarter) return d;
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
  if (box.per[0]) dx = min_image(dx, box.len[0], box.quarter[0]);
  if (box.per[1]) dy = min_image(dy, box.len[1], box.quarter[1]);
  if (box.per[2]) dz = min_image(dz, box.len[2], box.quarter[2]);
}

__device__ __forceinline__ int species_of(const double4& p) { return int(p.w); }

// Neighbor lists: "ELL4" — column-major ELL in blocks of 4 slots, so a thread
// fetches 4 entries of its atom with one 128-bit load (coalesced across the
// consecutive atoms of a warp) and a 4-lane group reads 16 contiguous bytes.
// Capacities are multiples of 4.
__host__ __device__ __forceinline__ std::size_t ell_at(int s, int a, int npad) {
  return (std::size_t(s >> 2) * std::size_t(npad) + std::size_t(a)) * 4 + std::size_t(s & 3);
}

// Float shadow of the positions (slot order, {x, y, z, species}) for cheap
// pre-tests.  A pre-test decides "inside" / "outside" only when the float
// squared distance clears the cutoff by more than its worst-case error
// (`margin`, set from the coordinate magnitude, tsf::prefilter_margin); pairs
// inside the band fall back to the exact FP64 test, so every decision is the
// reference's.
struct BoxF {
  float len[3];
  float half[3];
  int per[3];
  float inv[3];   // 1/len (IEEE, host) on periodic axes, 0 on open ones
};

enum : int { kOut = 0, kIn = 1, kUnsure = 2 };

// Programmatic dependent launch (launch_pdl): griddep_wait() returns once the
// preceding grid in the stream has completed and its writes are visible — a
// no-op for a kernel launched normally — so a kernel that starts with it keeps
// stream semantics; griddep_launch() lets the next launch_pdl kernel be
// scheduled (and sit in its own griddep_wait) while this one drains, which
// hides the launch gap between the force chain's kernels.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;"); }

// atomicMax(p, v) by one lane, skipped when p already holds >= v: the
// tracked maxima only grow between resets (which are stream-ordered before
// the kernel), so a stale read can only cost a redundant atomic — and
// same-address atomics from every warp of a 2M-atom pass serialise in L2.
__device__ __forceinline__ void lane_max(int* p, int v) {
  if (v > __ldcg(p)) atomicMax(p, v);
}

// Largest |coordinate| ever packed into the shadow (float bits, atomicMax);
// the pre-test bands are derived from it in-kernel, so no host round trip.
__device__ __forceinline__ void track_coord_max(int* cmax, const double4& p) {
  const float m = __double2float_ru(fmax(fabs(p.x), fmax(fabs(p.y), fabs(p.z))));
  const unsigned act = __activemask();
  const int v = __reduce_max_sync(act, __float_as_int(m));
  if ((threadIdx.x & 31) == __ffs(act) - 1) lane_max(cmax, v);
}

// The near lists' reference (Ctx::near_list): the positions at the last list
// build (ref) and, per slot, the displacement from there at the last near-list
// refresh (d0; zero after a build).  ref == nullptr: no list of ours to track.
struct DispRef {
  const double4* ref;
  const float4* d0;
};

// |displacement since the near lists' reference|^2 from the displacement d
// since the build: d - d0 (d0 is a float rounding of an exact displacement of
// at most skin/2: its error, < 2^-25 A, lies far inside the lists' margin mu).
__device__ __forceinline__ float near_disp2(const DispRef& r, int s, double dx, double dy,
                                            double dz) {
  const float4 o = r.d0[s];
  dx -= double(o.x);
  dy -= double(o.y);
  dz -= double(o.z);
  return __double2float_ru(norm_sq_exact(dx, dy, dz));
}

// Largest squared displacement of a slot since the near lists' reference
// (float bits rounded up, atomicMax; Ctx::near_list).  A NaN position
// propagates (its bits exceed +inf's), which disables the filter's near-list path.
__device__ __forceinline__ void track_disp(int* dmax, const DispRef& r, int s,
                                           const double4& p, const Box& box) {
  if (!r.ref) return;
  double dx, dy, dz;
  displacement(r.ref[s], p, box, dx, dy, dz);
  const float d2 = near_disp2(r, s, dx, dy, dz);
  const unsigned act = __activemask();
  const int v = __reduce_max_sync(act, __float_as_int(d2));
  if ((threadIdx.x & 31) == __ffs(act) - 1) lane_max(dmax, v);
}

// [lo, hi] around cut^2: outside it the float r^2 decides the cutoff test
// exactly as FP64 would.  Error model: each float coordinate is off by <=
// |x| 2^-24, the float displacement (with a float box wrap) by ed <=
// (3 M + cut) 2^-24, the float r^2 by <= 2 sqrt(3) cut ed + 3 ed^2 + a few
// float roundings of cut^2; doubled for safety.
__device__ __forceinline__ void band_for(double cut, const int* cmax, float& lo, float& hi) {
  const double u = 5.9604644775390625e-08;  // 2^-24
  const double M = double(__int_as_float(*cmax));
  const double ed = (3.0 * M + cut) * u * 1.01;
  const double er2 = 2.0 * (3.4641016151377544 * cut * ed + 3.0 * ed * ed + 8.0 * u * cut * cut);
  lo = __double2float_rd(cut * cut - er2);
  hi = __double2float_ru(cut * cut + er2);
}

// Short-list bound per (species of i, species of k): the largest squared
// cutoff of any parameter row (i, *, k).  Every pair the force kernel can
// accept passes it (the kernel tests the same exact FP64 r^2 against
// cutsq[i][j][k]); the reference's own filter uses r_cut_max for all pairs
// (kernels.hpp:187-188), which list exports reproduce.
struct PairBounds {
  double c2[kMaxSpecies * kMaxSpecies];
  double cut[kMaxSpecies * kMaxSpecies];
  int ns;
};

// Per-thread wrap constants for the float pre-test: 1/L = 0 on open axes.
struct WrapF {
  float inv[3], l[3];
};

__device__ __forceinline__ WrapF wrap_of(const BoxF& box) {
  WrapF w;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    w.inv[ax] = box.inv[ax];   // (host-computed: three IEEE divides per thread were
                               // 5% of the MD filter's instructions)
    w.l[ax] = box.len[ax];
  }
  return w;
}

__device__ __forceinline__ float dist2f(const float4& a, const float4& b, const WrapF& w) {
  float d[3] = {b.x - a.x, b.y - a.y, b.z - a.z};
  // float minimum image d - L rint(d / L) (3 instructions per axis).  It can
  // pick the other image than the exact test only at |d| ~ L/2, where both
  // images have the same length up to rounding — inside the error band, so
  // such a pair takes the exact FP64 test.
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) d[ax] = fmaf(-w.l[ax], rintf(d[ax] * w.inv[ax]), d[ax]);
  return d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
}

__device__ __forceinline__ int prefilter(const float4& a, const float4& b, const WrapF& w,
                                         float lo, float hi) {
  const float r2 = dist2f(a, b, w);
  return r2 < lo ? kIn : (r2 > hi ? kOut : kUnsure);
}

__device__ __forceinline__ int prefilter(const float4& a, const float4& b, const BoxF& box,
                                         float lo, float hi) {
  return prefilter(a, b, wrap_of(box), lo, hi);
}


}  // namespace tsf
