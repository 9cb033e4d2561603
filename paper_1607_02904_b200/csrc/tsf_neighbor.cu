// GPU cell-list neighbor build with a cell-sorted atom layout, the paper's
// cutoff filter (short list) and the rebuild trigger.
//
// Output contract (bit-exact with the reference):
//   build_neighbor_list  proj/src/neighbor.cpp:37-132  — full, symmetric list of
//     every b != a with |min_image(x_b - x_a)|^2 <= (rc + skin)^2, decided with
//     the reference's FP64 rounding sequence (no contraction).  The cell grid
//     is the reference's (same edge, same binning arithmetic, same
//     deduplicated 27-stencil), so even ulp-level binning decisions at cell
//     faces select the same candidate set.  Exported segments are mapped back
//     to user indices and sorted ascending (neighbor.cpp:114).
//   filter_all_segments  proj/src/neighbor.cpp:143-180 — skin entries with
//     r^2 <= r_cut_max^2, order kept; verbatim copy when the filter is off.
//     (Exports; the force path keeps r^2 <= max_j cutsq[i][j][k] per species
//     pair, which drops only pairs whose every term is an exact zero.)
//   needs_rebuild        proj/src/neighbor.cpp:134-141 — any |dx|^2 > (skin/2)^2.
//
// Layout and kernels:
//   * every build re-sorts the atoms by (cell, user index) with a radix sort:
//     a cell's atoms are a contiguous slot range, and threads of a warp
//     (neighbouring atoms) gather the same cache lines;
//   * candidates are tested on a float shadow of the positions (16 B gathers
//     instead of 32 B) with a rigorous error band; only pairs inside the band
//     take the exact FP64 test (tsf_device.cuh), so decisions stay bit-exact;
//   * lists are ELL, column-major (nbr[s * npad + a]) + count[a], in slots.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>

#include "tsf_context.hpp"

namespace tsf {

namespace {

__device__ __forceinline__ int clamp_cell(double p, double org, double ext, int n) {
  // int(floor(((p - o) / e) * n)) clamped to [0, n-1]  (neighbor.cpp:19-28)
  const double f = __dmul_rn(__ddiv_rn(__dsub_rn(p, org), ext), double(n));
  int c = int(floor(f));
  return c < 0 ? 0 : (c > n - 1 ? n - 1 : c);
}

// atomicMax from one lane per converged subset, only when it can raise the
// value: one address takes every warp's update (64k per 2M-atom launch), and
// same-address atomics serialise in L2 — once the maximum is reached a plain
// cached read filters almost all of them out.
__device__ __forceinline__ void warp_atomic_max(int* p, int v) {
  const unsigned act = __activemask();
  const int m = __reduce_max_sync(act, v);
  if ((threadIdx.x & 31) == __ffs(act) - 1 && m > __ldcg(p)) atomicMax(p, m);
}

// Cell id per atom, written at its USER index: a stable radix sort of the
// cell ids alone (20-odd bits: 3 passes instead of 7 over a 52-bit
// (cell, user) key) then yields (cell, user) order; counts per cell; largest
// occupancy.
// With an interior split (n_int >= 0, the decomposition's overlap mode) the
// key is class-major: user atoms below n_int (interior owned) sort first, so
// their slots are [0, n_int); the "cell" index is then class * ncells + cell,
// keeping every (class, cell) run contiguous for the skin build.
// Non-centre ghosts (user index >= n_ctr, decompositions) form the last class,
// so every centre holds a slot below n_ctr and the force launches stop there.
__global__ void k_cell_key(const double4* __restrict__ pos, const int* __restrict__ perm, int n,
                           CellGrid g, int n_int, int n_ctr, unsigned* __restrict__ keys,
                           int* __restrict__ vals, int* __restrict__ count,
                           int* __restrict__ max_occ) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double4 p = pos[s];
  const int cx = clamp_cell(p.x, g.org[0], g.ext[0], g.nc[0]);
  const int cy = clamp_cell(p.y, g.org[1], g.ext[1], g.nc[1]);
  const int cz = clamp_cell(p.z, g.org[2], g.ext[2], g.nc[2]);
  const unsigned user = unsigned(perm ? perm[s] : s);
  const int ncells = g.nc[0] * g.nc[1] * g.nc[2];
  int cls = n_int >= 0 && int(user) >= n_int ? 1 : 0;
  if (n_ctr >= 0 && int(user) >= n_ctr) cls = n_int >= 0 ? 2 : 1;
  const int c = (cz * g.nc[1] + cy) * g.nc[0] + cx + cls * ncells;
  keys[user] = unsigned(c);
  vals[user] = int(user);
  warp_atomic_max(max_occ, atomicAdd(count + c, 1) + 1);
}

// Apply the new order: slot t takes user atom users[t], found at its old slot
// inv[user] (sorted: inv describes the current slots) or at slot user.
__global__ void k_reorder(const unsigned* __restrict__ keys, const int* __restrict__ users, int n,
                          int sorted, const double4* __restrict__ pos_in,
                          const double* __restrict__ vel_in, double4* __restrict__ pos_out,
                          double* __restrict__ vel_out, int* __restrict__ perm,
                          int* __restrict__ inv, int* __restrict__ cell_of) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int user = users[t];
  const int s = sorted ? inv[user] : user;   // read, then rewritten, by this thread only
  pos_out[t] = pos_in[s];
  vel_out[3 * t] = vel_in[3 * s];
  vel_out[3 * t + 1] = vel_in[3 * s + 1];
  vel_out[3 * t + 2] = vel_in[3 * s + 2];
  perm[t] = user;
  inv[user] = t;
  cell_of[t] = int(keys[t]);
}

// Unique wrapped neighbor coordinates along one axis (the per-axis factor of
// the deduplicated 27-stencil, neighbor.cpp:84-103).
__device__ __forceinline__ int axis_stencil(int c, int n, int per, int out[3]) {
  int m = 0;
  for (int d = -1; d <= 1; ++d) {
    int w = c + d;
    if (per) w = (w + n) % n;
    if (w < 0 || w >= n) continue;
    bool dup = false;
    for (int q = 0; q < m; ++q) dup |= out[q] == w;
    if (!dup) out[m++] = w;
  }
  return m;
}

// The exact FP64 decision for a pair inside the float band (rare; out of
// line — __noinline__ — it measured 27% slower: the call ABI costs more than
// the code size saves).
__device__ __forceinline__ bool exact_within(const double4* __restrict__ pos, int a, int b,
                                          const Box& box, double c2) {
  double dx, dy, dz;
  displacement(pos[a], pos[b], box, dx, dy, dz);
  return norm_sq_exact(dx, dy, dz) <= c2;
}

struct ListArgs {
  const double4* pos;
  const float4* posf;
  const int* cmax;
  int n, npad;
  Box box;
  BoxF boxf;
  CellGrid g;
  const int* cell_of;
  const int* start;
  int ncls;          // slot classes (1, or 2 with an interior split)
};

// near-list outputs of a build (Ctx::near_list); nbr[0] == nullptr: none
struct NearOut {
  int* nbr[2];
  int* cnt[2];
  int* hist;         // [6]: atoms with > 4 / 8 / 12 entries in list 0, then list 1
  double cut[2];     // r_cut_max + h_q
  double h[2];
};

// Near-list entries carry a "sure" bit: the pair lay within the smallest
// filter bound of any species pair minus h_q at the build, so while the list
// is valid (2 |d|max < h_q) it is inside every bound — kept without a gather.
constexpr unsigned kSure = 0x80000000u;

// near-list inputs of the filter (Ctx::near_list); nbr[0] == nullptr: none
struct NearIn {
  const int* nbr[2];
  const int* cnt[2];
  const int* dmax;   // squared displacement max since the near lists' reference (float bits)
  float t[2];
  int pre[2];
  const int* skip;   // speculative MD step: return at once when *skip != 0
  // refresh (full-range force-path filters only; refresh = 0 elsewhere): with
  // both lists stale the filter reads the skin list and rewrites both near
  // lists (the lists above, written) and the reference displacements
  int refresh;
  double cut[2];       // near_cut[q]
  double sure_cut[2];  // smallest pair bound - h_q
  const double4* ref;  // build positions
  float4* d0;          // per slot: displacement since the build at the refresh
  int* refreshed;      // flags[kFlagNearRefresh]
};

// Skin list, one thread per slot: candidates are the stencil cells' slot
// ranges (contiguous in the cell-sorted layout), tested on the float shadow
// with the exact FP64 fallback inside the error band.  Slots are sorted by
// (class, cell, user index) and a cell index is lexicographic in (z, y, x),
// so walking the classes, then each axis's stencil coordinates in ascending
// order, visits the candidates in ascending slot order: entries are written
// straight to the ELL list as they pass — no per-thread buffer, no sort (the
// earlier form kept a local-memory buffer and insertion-sorted it: 0.88 ms at
// 2M atoms).  The near lists take the same pass, on the same float r^2.
// axis_stencil's coordinates, ascending, in registers: returns the count;
// unused trailing entries hold INT_MAX.
__device__ __forceinline__ int axis_stencil_sorted(int c, int n, int per, int v[3]) {
  int v0 = c - 1, v2 = c + 1;
  bool k0, k2;
  if (per) {
    v0 = v0 < 0 ? v0 + n : v0;
    v2 = v2 >= n ? v2 - n : v2;
    k0 = v0 != c;
    k2 = v2 != c && v2 != v0;
  } else {
    k0 = v0 >= 0;
    k2 = v2 < n;
  }
  int x0 = k0 ? v0 : 0x7fffffff, x1 = c, x2 = k2 ? v2 : 0x7fffffff;
  int t;
  if (x0 > x1) { t = x0; x0 = x1; x1 = t; }
  if (x1 > x2) { t = x1; x1 = x2; x2 = t; }
  if (x0 > x1) { t = x0; x0 = x1; x1 = t; }
  v[0] = x0;
  v[1] = x1;
  v[2] = x2;
  return 1 + int(k0) + int(k2);
}

__global__ void __launch_bounds__(kBlock) k_skin_list(ListArgs a, double bc, double bc2, int cap,
                                                      int* __restrict__ nbr,
                                                      int* __restrict__ cnt,
                                                      int* __restrict__ max_count,
                                                      NearOut near, PairBounds sure) {
  const int at = blockIdx.x * blockDim.x + threadIdx.x;
  if (at >= a.n) return;
  float lo, hi;
  band_for(bc, a.cmax, lo, hi);
  // near lists (Ctx::near_list): every entry not provably beyond near_cut[q]
  // — a float r^2 above the band's upper edge means the exact FP64 r^2 is
  // beyond near_cut[q]^2 too; sure: the float r^2 below the band's lower
  // edge around (bound - h_q)^2
  const bool nl = near.nbr[0] != nullptr;
  float hi0 = 0, hi1 = 0, slo0 = 0, slo1 = 0;
  if (nl) {
    float t;
    band_for(near.cut[0], a.cmax, t, hi0);
    band_for(near.cut[1], a.cmax, t, hi1);
    band_for(fmax(sure.cut[0] - near.h[0], 0.0), a.cmax, slo0, t);
    band_for(fmax(sure.cut[0] - near.h[1], 0.0), a.cmax, slo1, t);
  }
  const CellGrid& g = a.g;
  const float4 pfa = a.posf[at];
  const WrapF wrap = wrap_of(a.boxf);
  const int ncells = g.nc[0] * g.nc[1] * g.nc[2];
  const int home = a.cell_of[at] % ncells;   // class-major index when split
  const int cx = home % g.nc[0], cy = (home / g.nc[0]) % g.nc[1];
  const int cz = home / (g.nc[0] * g.nc[1]);
  int sx[3], sy[3], sz[3];
  const int mx = axis_stencil_sorted(cx, g.nc[0], a.box.per[0], sx);
  const int my = axis_stencil_sorted(cy, g.nc[1], a.box.per[1], sy);
  const int mz = axis_stencil_sorted(cz, g.nc[2], a.box.per[2], sz);
  int m = 0, w0 = 0, w1 = 0;
  // (selects, not indexing, keep the stencil coordinates in registers)
  auto pick = [](const int* v, int i) { return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]); };
  for (int cls = 0; cls < a.ncls; ++cls)
    for (int iz = 0; iz < mz; ++iz)
      for (int iy = 0; iy < my; ++iy) {
        const int row = (pick(sz, iz) * g.nc[1] + pick(sy, iy)) * g.nc[0] + cls * ncells;
        for (int ix = 0; ix < mx; ++ix) {
          const int c = row + pick(sx, ix);
          TSF_DCHECK(c >= 0 && c < ncells * a.ncls, "k_skin_list stencil cell");
          const int b1 = a.start[c + 1];
          TSF_DCHECK(a.start[c] >= 0 && b1 <= a.n && a.start[c] <= b1, "k_skin_list cell range");
          for (int b = a.start[c]; b < b1; ++b) {
            if (b == at) continue;
            const float r2 = dist2f(pfa, a.posf[b], wrap);
            bool in = r2 < lo;
            if (!in && !(r2 > hi)) in = exact_within(a.pos, at, b, a.box, bc2);
            if (!in) continue;
            if (m < cap) {
              nbr[ell_at(m, at, a.npad)] = b;
              if (nl) {
                if (!(r2 > hi0))
                  near.nbr[0][ell_at(w0++, at, a.npad)] = int(unsigned(b) | (r2 < slo0 ? kSure : 0u));
                if (!(r2 > hi1))
                  near.nbr[1][ell_at(w1++, at, a.npad)] = int(unsigned(b) | (r2 < slo1 ? kSure : 0u));
              }
            }
            ++m;
          }
        }
      }
  warp_atomic_max(max_count, m);
  if (m > cap) return;  // host grows the capacity and rebuilds
  cnt[at] = m;
  if (nl) {
    near.cnt[0][at] = w0;
    near.cnt[1][at] = w1;
    const unsigned act = __activemask();
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int c = __popc(__ballot_sync(act, (q < 3 ? w0 : w1) > 4 * (q % 3 + 1)));
      if ((threadIdx.x & 31) == __ffs(act) - 1 && c) atomicAdd(near.hist + q, c);
    }
  }
}

// Short list, one thread per slot: skin entries that pass their pair's bound,
// in segment order.  The first 16 entries' ELL4 blocks are all requested
// before any is tested, so a thread keeps 64 B of list in flight (one block
// at a time measured latency-bound: 14.7 cycles/issue, 18% of HBM; a quad of
// lanes per slot was slower still, profiles/r01/ncu).  Float pre-test, exact
// FP64 inside the band; a verbatim copy when the filter is off.
#ifndef TSF_FILTER_MINB
#define TSF_FILTER_MINB 8
#endif

// Pre-test bands per species pair (shared memory); with one species the
// single band lives in registers (MULTI = false).
struct FilterBands {
  const float* lo;
  const float* hi;
  const double* c2;
  int ns;
  float lo0, hi0;
  double c20;
  WrapF wrap;
  int* err;   // flags[0] of a force-path filter (NaN distances), else nullptr
};


// Float pre-test of the 4 entries of ELL4 block e, branch-free so the four
// shadow gathers issue together: `in` / `unsure` bits for the first `valid`
// entries (the rest gather the atom's own shadow and are masked off); prs
// holds the species-pair index of each entry (MULTI), 4 bits each.
template <bool MULTI>
__device__ __forceinline__ void test_block(const ListArgs& a, const FilterBands& fb, int at,
                                           const float4& pfa, int si, int4& e, int valid,
                                           int& in, int& unsure, int& prs) {
  // sure entries (near lists, kSure) are kept without a gather; the bit is
  // stripped here so the entries written out are plain slots
  const int sure = int((unsigned(e.x) >> 31) | ((unsigned(e.y) >> 30) & 2u) |
                       ((unsigned(e.z) >> 29) & 4u) | ((unsigned(e.w) >> 28) & 8u));
  e.x &= 0x7fffffff;
  e.y &= 0x7fffffff;
  e.z &= 0x7fffffff;
  e.w &= 0x7fffffff;
  TSF_DCHECK(valid <= 0 || (e.x >= 0 && e.x < a.n && e.x != at), "k_filter entry 0");
  TSF_DCHECK(valid <= 1 || (e.y >= 0 && e.y < a.n && e.y != at), "k_filter entry 1");
  TSF_DCHECK(valid <= 2 || (e.z >= 0 && e.z < a.n && e.z != at), "k_filter entry 2");
  TSF_DCHECK(valid <= 3 || (e.w >= 0 && e.w < a.n && e.w != at), "k_filter entry 3");
  const int bb[4] = {valid > 0 && !(sure & 1) ? e.x : at, valid > 1 && !(sure & 2) ? e.y : at,
                     valid > 2 && !(sure & 4) ? e.z : at, valid > 3 && !(sure & 8) ? e.w : at};
  float4 pf[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) pf[u] = a.posf[bb[u]];
  in = 0;
  unsure = 0;
  prs = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int v;
    if (MULTI) {
      const int pr = si * fb.ns + min(max(int(pf[u].w), 0), fb.ns - 1);
      v = prefilter(pfa, pf[u], fb.wrap, fb.lo[pr], fb.hi[pr]);
      prs |= pr << (4 * u);
    } else {
      v = prefilter(pfa, pf[u], fb.wrap, fb.lo0, fb.hi0);
    }
    in |= (v == kIn) << u;
    unsure |= (v == kUnsure) << u;
  }
  const int vm = (1 << max(0, min(valid, 4))) - 1;
  in = (in | sure) & vm;
  unsure &= vm & ~sure;
}

// Rare: entries inside the float error band take the exact FP64 test (the
// entry is re-read from the list so no register array is indexed at run time).
template <bool MULTI>
__device__ __forceinline__ unsigned resolve_unsure(const ListArgs& a, const FilterBands& fb,
                                                   const int* skin, int at, int s_base,
                                                   unsigned unsure, unsigned long long prs) {
  unsigned in = 0;
  while (unsure) {
    const int q = __ffs(unsure) - 1;
    unsure &= unsure - 1;
    const int b = skin[ell_at(s_base + q, at, a.npad)] & 0x7fffffff;
    const double c2 = MULTI ? fb.c2[(prs >> (4 * q)) & 15] : fb.c20;
    double dx, dy, dz;
    displacement(a.pos[at], a.pos[b], a.box, dx, dy, dz);
    const double r2 = norm_sq_exact(dx, dy, dz);
    if (r2 <= c2) {
      in |= 1u << q;
    } else if (fb.err && r2 != r2) {
      // a NaN coordinate: the float pre-test sends it here (neither in nor
      // out); the reference's cutoff tests let the NaN into zeta and throw
      // NumericError (potential_ref.cpp:109-112) — flag it the same way
      atomicOr(fb.err + kFlagFilterNaN, 1);
    }
  }
  return in;
}

// Append the kept entries of ELL4 block e (bits 0..3) to the short list.
__device__ __forceinline__ void keep_block(int* out, int at, int npad, int4 e, int bits, int& w) {
  if (bits & 1) out[ell_at(w++, at, npad)] = e.x;
  if (bits & 2) out[ell_at(w++, at, npad)] = e.y;
  if (bits & 4) out[ell_at(w++, at, npad)] = e.z;
  if (bits & 8) out[ell_at(w++, at, npad)] = e.w;
}

// Filter the first m entries of list L for slot `at` into `out`; the first
// `pre` ELL4 blocks (4 pre entries, pre <= 4, grid-uniform) are requested up
// front.
template <bool MULTI>
__device__ __forceinline__ int filter_list(const ListArgs& a, const FilterBands& fb, int at,
                                           const int* __restrict__ L, int m, int pre,
                                           int* __restrict__ out) {
  int4 e[4];
  // streamed once per step: evict-first keeps the gathered shadow in L2.
  // Loaded without waiting for the count (every list has >= 16 allocated
  // entries; those past the count are masked off in test_block), so count
  // and list cost one DRAM round trip, not two.
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (b < pre) e[b] = __ldcs(reinterpret_cast<const int4*>(L + ell_at(4 * b, at, a.npad)));
  if (m <= 4 * pre) {
    // every entry "sure" (a near list's usual case in a crystal): nothing to
    // test, no shadow gather — the blocks go out with the bits stripped
    bool all = true;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int v = m - 4 * b;
      all = all && (b >= pre || ((v <= 0 || e[b].x < 0) && (v <= 1 || e[b].y < 0) &&
                                 (v <= 2 || e[b].z < 0) && (v <= 3 || e[b].w < 0)));
    }
    if (all) {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (b < pre && 4 * b < m) {
          const int4 q = make_int4(e[b].x & 0x7fffffff, e[b].y & 0x7fffffff, e[b].z & 0x7fffffff,
                                   e[b].w & 0x7fffffff);
          *reinterpret_cast<int4*>(out + ell_at(4 * b, at, a.npad)) = q;
        }
      return m;
    }
  }
  const float4 pfa = a.posf[at];   // (after the all-sure copy, which needs none)
  const int si = MULTI ? min(max(int(pfa.w), 0), fb.ns - 1) : 0;
  // test all of them before any store or exact fallback: nothing between the
  // gathers keeps the compiler from issuing them back to back
  unsigned keep = 0, uns = 0;
  unsigned long long prs = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (b < pre) {
      int in, un, pr;
      test_block<MULTI>(a, fb, at, pfa, si, e[b], m - 4 * b, in, un, pr);
      keep |= unsigned(in) << (4 * b);
      uns |= unsigned(un) << (4 * b);
      if (MULTI) prs |= static_cast<unsigned long long>(unsigned(pr) & 0xffffu) << (16 * b);
    }
  }
  if (uns) keep |= resolve_unsure<MULTI>(a, fb, L, at, 0, uns, prs);
  int w = 0;
  const int nv = min(m, 4 * pre);
  if (keep == (1u << nv) - 1u) {
    // every entry kept (a crystal's near list: all sure): the blocks go out
    // as loaded, one 16-byte store each (entries past the count are never read)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (b < pre && 4 * b < nv) *reinterpret_cast<int4*>(out + ell_at(4 * b, at, a.npad)) = e[b];
    w = nv;
  } else {
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (b < pre) keep_block(out, at, a.npad, e[b], int(keep >> (4 * b)) & 15, w);
  }
  for (int s0 = 4 * pre; s0 < m; s0 += 4) {
    int4 q = __ldcs(reinterpret_cast<const int4*>(L + ell_at(s0, at, a.npad)));
    int in, un, pr;
    test_block<MULTI>(a, fb, at, pfa, si, q, m - s0, in, un, pr);
    unsigned k = unsigned(in);
    if (un) k |= resolve_unsure<MULTI>(a, fb, L, at, s0, unsigned(un), unsigned(pr));
    keep_block(out, at, a.npad, q, int(k), w);
  }
  return w;
}

// Near-list refresh (Ctx::near_d0): the short list from the skin list as
// filter_list does, and both near lists rewritten on the same float r^2 — the
// entries within near_cut[q] of the CURRENT positions, sure bits against
// sure_cut[q] (k_skin_list's rules) — plus this slot's displacement since the
// build, the new reference of the displacement maximum.  Valid by the build's
// argument: any pair within a cutoff before the next rebuild is in the skin
// list, and lies within r_cut_max + 2 |d|max of its distance now.
template <bool MULTI>
__device__ __forceinline__ int filter_refresh(const ListArgs& a, const FilterBands& fb,
                                           const NearIn& near, int at,
                                           const int* __restrict__ L, int m,
                                           int* __restrict__ out) {
  const float4 pfa = a.posf[at];
  const int si = MULTI ? min(max(int(pfa.w), 0), fb.ns - 1) : 0;
  float hi0, hi1, slo0, slo1, t;
  band_for(near.cut[0], a.cmax, t, hi0);
  band_for(near.cut[1], a.cmax, t, hi1);
  band_for(fmax(near.sure_cut[0], 0.0), a.cmax, slo0, t);
  band_for(fmax(near.sure_cut[1], 0.0), a.cmax, slo1, t);
  int* n0 = const_cast<int*>(near.nbr[0]);
  int* n1 = const_cast<int*>(near.nbr[1]);
  int w = 0, w0 = 0, w1 = 0;
  for (int s0 = 0; s0 < m; s0 += 4) {
    const int4 q = __ldcs(reinterpret_cast<const int4*>(L + ell_at(s0, at, a.npad)));
    const int e[4] = {q.x, q.y, q.z, q.w};
    float4 pf[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) pf[u] = a.posf[s0 + u < m ? e[u] : at];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (s0 + u >= m) continue;
      const float r2 = dist2f(pfa, pf[u], fb.wrap);
      const int pr = MULTI ? si * fb.ns + min(max(int(pf[u].w), 0), fb.ns - 1) : 0;
      const float lo = MULTI ? fb.lo[pr] : fb.lo0, hi = MULTI ? fb.hi[pr] : fb.hi0;
      bool in = r2 < lo;
      if (!in && !(r2 > hi)) {
        double dx, dy, dz;
        displacement(a.pos[at], a.pos[e[u]], a.box, dx, dy, dz);
        const double d2 = norm_sq_exact(dx, dy, dz);
        in = d2 <= (MULTI ? fb.c2[pr] : fb.c20);
        if (!in && fb.err && d2 != d2) atomicOr(fb.err + kFlagFilterNaN, 1);
      }
      if (in) out[ell_at(w++, at, a.npad)] = e[u];
      if (!(r2 > hi0)) n0[ell_at(w0++, at, a.npad)] = int(unsigned(e[u]) | (r2 < slo0 ? kSure : 0u));
      if (!(r2 > hi1)) n1[ell_at(w1++, at, a.npad)] = int(unsigned(e[u]) | (r2 < slo1 ? kSure : 0u));
    }
  }
  const_cast<int*>(near.cnt[0])[at] = w0;
  const_cast<int*>(near.cnt[1])[at] = w1;
  double dx, dy, dz;
  displacement(near.ref[at], a.pos[at], a.box, dx, dy, dz);
  near.d0[at] = make_float4(float(dx), float(dy), float(dz), 0.0f);
  return w;
}

template <bool MULTI>
__global__ void __launch_bounds__(kBlock, TSF_FILTER_MINB) k_filter(
    ListArgs a, PairBounds pb, int apply, const int* __restrict__ skin,
    const int* __restrict__ skin_cnt, int* __restrict__ out, int* __restrict__ out_cnt,
    int* __restrict__ max_count, int* __restrict__ hist, void* __restrict__ zero_f,
    int zero_bytes, int slot_lo, int slot_hi, NearIn near, int* __restrict__ zero_flags,
    int* __restrict__ over4) {
  __shared__ float slo[kMaxSpecies * kMaxSpecies], shi[kMaxSpecies * kMaxSpecies];
  __shared__ double sc2[kMaxSpecies * kMaxSpecies];
  // a speculative step whose list went stale (this step's kick, or an
  // earlier step of a multi-step segment)
  if (near.skip && (near.skip[0] | near.skip[kFlagMovedAny - kFlagMoved])) return;
  // error bits and tier queue counts of the force launches that follow
  if (zero_flags && blockIdx.x == 0 && threadIdx.x < 4) zero_flags[threadIdx.x] = 0;
  const int ns = pb.ns;
  if (apply && int(threadIdx.x) < ns * ns) {
    float lo, hi;
    band_for(pb.cut[threadIdx.x], a.cmax, lo, hi);
    slo[threadIdx.x] = lo;
    shi[threadIdx.x] = hi;
    sc2[threadIdx.x] = pb.c2[threadIdx.x];
  }
  __syncthreads();
  const int at = slot_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (at >= slot_hi) return;
  // the force accumulator of the atomic-mode kernel that follows, zeroed here
  // (this thread is waiting on its list anyway) instead of by a memset: the
  // launch's 3 (hi - lo) words, thread g taking words g, g + m, g + 2m —
  // three fully coalesced stores (a stride-3 triple per thread left each
  // store instruction a third of its sectors)
  if (zero_bytes) {
    const std::size_t m = std::size_t(slot_hi - slot_lo);
    const std::size_t w = 3 * std::size_t(slot_lo) + std::size_t(at - slot_lo);
    if (zero_bytes == 8) {
      double* z = static_cast<double*>(zero_f) + w;
      z[0] = 0.0;
      z[m] = 0.0;
      z[2 * m] = 0.0;
    } else {
      float* z = static_cast<float*>(zero_f) + w;
      z[0] = 0.0f;
      z[m] = 0.0f;
      z[2 * m] = 0.0f;
    }
  }
  // grid-uniform: the smallest near list no atom has moved far enough since
  // the build to invalidate (Ctx::near_list), else the skin list
  const int* L = skin;
  const int* Lc = skin_cnt;
  int pre = 4;
  bool refresh = false;
  if (near.nbr[0]) {
    const float d2 = __int_as_float(*near.dmax);
    const int q = d2 < near.t[0] ? 0 : d2 < near.t[1] ? 1 : 2;
    if (q < 2) {
      // selects, not an index: a run-time index into the parameter struct
      // copies it to local memory in every thread
      L = q == 0 ? near.nbr[0] : near.nbr[1];
      Lc = q == 0 ? near.cnt[0] : near.cnt[1];
      pre = q == 0 ? near.pre[0] : near.pre[1];
    } else {
      refresh = near.refresh != 0 && !(d2 != d2);   // grid-uniform
    }
  }
  const int m = Lc[at];
  int w = 0;
  if (apply) {
    const FilterBands fb{slo, shi, sc2, ns, slo[0], shi[0], sc2[0], wrap_of(a.boxf), zero_flags};
    if (refresh) {
      if (at == slot_lo) *near.refreshed = 1;
      w = filter_refresh<MULTI>(a, fb, near, at, L, m, out);
    } else {
      w = filter_list<MULTI>(a, fb, at, L, m, pre, out);
    }
  } else {
    for (int s = 0; s < m; ++s) out[ell_at(s, at, a.npad)] = skin[ell_at(s, at, a.npad)];
    w = m;
  }
  out_cnt[at] = w;
  if (over4) {   // force path: does the packed tier behind G = 4 have work?
    const unsigned act = __activemask();
    if (__any_sync(act, w > 4) && (threadIdx.x & 31) == __ffs(act) - 1 && __ldcg(over4) == 0)
      *over4 = 1;
  }
  // largest count and occupancy histogram for the force kernel's group width,
  // after rebuilds only (same-address atomics from every warp are not free):
  // hist[0] = atoms with more than 4 short neighbours, hist[1] = more than 8
  if (max_count) {
    warp_atomic_max(max_count, w);
    const unsigned act = __activemask();
    const int c4 = __popc(__ballot_sync(act, w > 4)), c8 = __popc(__ballot_sync(act, w > 8));
    if ((threadIdx.x & 31) == __ffs(act) - 1) {
      if (c4) atomicAdd(hist, c4);
      if (c8) atomicAdd(hist + 1, c8);
    }
  }
}

__global__ void k_needs_rebuild(const double4* __restrict__ pos,
                                const double4* __restrict__ ref, int n, Box box,
                                double limit_sq, int* __restrict__ flag) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  bool moved = false;
  if (a < n) {
    double dx, dy, dz;
    displacement(ref[a], pos[a], box, dx, dy, dz);
    moved = norm_sq_exact(dx, dy, dz) > limit_sq;
  }
  if (__any_sync(0xffffffffu, moved) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Occupied extent of open axes (neighbor.cpp:50-77); order-preserving integer
// keys let atomicMin/Max reduce doubles exactly.
__device__ __forceinline__ unsigned long long ordered_key(double v) {
  const unsigned long long b = __double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_extent(const double4* __restrict__ pos, int n,
                         unsigned long long* __restrict__ mnmx) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double4 p = pos[a];
  const double v[3] = {p.x, p.y, p.z};
  // warp-reduced, then one lane per warp and only when it moves a bound (six
  // same-address atomics per atom serialised in L2)
  const unsigned act = __activemask();
  const bool first = (threadIdx.x & 31) == __ffs(act) - 1;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    unsigned long long lo = ordered_key(v[ax]), hi = lo;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long l2 = __shfl_xor_sync(act, lo, o), h2 = __shfl_xor_sync(act, hi, o);
      const bool ok = (act >> ((threadIdx.x & 31) ^ o)) & 1u;   // partner active
      if (ok) {
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
      }
    }
    if (first) {
      if (lo < __ldcg(mnmx + ax)) atomicMin(mnmx + ax, lo);
      if (hi > __ldcg(mnmx + 3 + ax)) atomicMax(mnmx + 3 + ax, hi);
    }
  }
}

double from_key(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & ~0x8000000000000000ull) : ~k;
  double v;
  std::memcpy(&v, &b, sizeof v);
  return v;
}

int blocks_for(std::int64_t n) { return int((n + kBlock - 1) / kBlock); }

template <typename T>
void swap_buf(DevBuf<T>& a, DevBuf<T>& b) {
  std::swap(a.ptr, b.ptr);
  std::swap(a.cap, b.cap);
}

// Slot classes of a list build: [interior owned] [other centres] [non-centre
// ghosts] — the first only with an interior split, the last only when the
// context has ghosts (tsf_set_owned / tsf_set_centers below n).
int ghost_class_limit(const Ctx& c) {
  const std::int64_t lim = c.n_owned >= 0 ? std::min<std::int64_t>(c.n_owned, c.n) : c.n;
  return lim < c.n ? int(lim) : -1;
}

int slot_classes(const Ctx& c) {
  return (c.n_interior >= 0 ? 2 : 1) + (ghost_class_limit(c) >= 0 ? 1 : 0);
}

ListArgs list_args(Ctx& c) {
  ListArgs a;
  a.pos = c.pos.get();
  a.posf = c.posf.get();
  a.cmax = c.flags.get() + 5;
  a.n = int(c.n);
  a.npad = c.npad;
  a.box = c.box;
  a.boxf = c.boxf;
  a.g = c.grid;
  a.cell_of = c.cell_of.get();
  a.start = c.cell_start.get();
  a.ncls = slot_classes(c);
  return a;
}

// The filter's bound per (species of i, species of k) for a mode: the
// reference's r_cut_max (exports), or the largest cutsq of any row (i, *, k)
// (the force path, PairBounds).
PairBounds pair_bounds(const Ctx& c, FilterMode mode) {
  PairBounds pb{};
  if (mode != FilterMode::Copy) {
    const int ns = c.params.species_count();
    pb.ns = ns;
    const double rc = c.params.r_cut_max();
    for (int i = 0; i < ns; ++i)
      for (int k = 0; k < ns; ++k) {
        double c2 = rc * rc, cut = rc;   // the reference's test (neighbor.cpp:146)
        if (mode == FilterMode::Pair) {
          c2 = 0;
          for (int j = 0; j < ns; ++j) {
            const double cc = c.params.entry(i, j, k).cutoff();
            c2 = std::max(c2, cc * cc);   // the force kernel's cutsq values
          }
          cut = std::sqrt(c2);
        }
        pb.c2[i * ns + k] = c2;
        pb.cut[i * ns + k] = cut;
      }
    // Symmetric bounds: the deterministic scatter has atom a collect the
    // force slots of the centres in its OWN short list (k_gather), so k must
    // list i whenever i lists k.  A LAMMPS-format table may give (i,*,k) and
    // (k,*,i) different R/D; the larger bound only adds entries whose terms
    // are exact zeros (outside every cutoff of their rows).
    if (mode == FilterMode::Pair)
      for (int i = 0; i < ns; ++i)
        for (int k = i + 1; k < ns; ++k) {
          const double c2 = std::max(pb.c2[i * ns + k], pb.c2[k * ns + i]);
          const double cut = std::max(pb.cut[i * ns + k], pb.cut[k * ns + i]);
          pb.c2[i * ns + k] = pb.c2[k * ns + i] = c2;
          pb.cut[i * ns + k] = pb.cut[k * ns + i] = cut;
        }
  } else {
    pb.ns = 1;
  }
  return pb;
}

// The bound sure bits are tested against: the smallest pair bound of the
// table (one "species pair"), so that a species change between list builds —
// set_system keeps the list — cannot make a sure entry wrong.
PairBounds sure_bound(const Ctx& c, bool near) {
  PairBounds sb{{}, {}, 1};
  if (near) {
    const PairBounds pb = pair_bounds(c, FilterMode::Pair);
    double m = pb.cut[0];
    for (int q = 1; q < pb.ns * pb.ns; ++q) m = std::min(m, pb.cut[q]);
    sb.cut[0] = m;
    sb.c2[0] = m * m;
  }
  return sb;
}

void launch_skin(Ctx& c, double bc2, int cap) {
  const bool near = c.near_cut[0] > 0.0;
  const double rf = near ? c.params.r_cut_max() : 0.0;
  k_skin_list<<<blocks_for(c.n), kBlock, 0, c.stream>>>(
      list_args(c), std::sqrt(bc2), bc2, cap, c.skin_list.nbr.get(), c.skin_list.cnt.get(),
      c.flags.get() + 3,
      NearOut{{near ? c.near_list[0].nbr.get() : nullptr, c.near_list[1].nbr.get()},
              {c.near_list[0].cnt.get(), c.near_list[1].cnt.get()},
              c.flags.get() + 11,
              {c.near_cut[0], c.near_cut[1]},
              {c.near_cut[0] - rf, c.near_cut[1] - rf}},
      sure_bound(c, near));
  ++c.launches;
}

// TSF_NEAR_REFRESH=0: stale near lists fall back to the skin list (A/B; read
// per eager filter launch, so tests can switch it)
bool near_refresh_enabled() {
  const char* e = std::getenv("TSF_NEAR_REFRESH");
  return !(e && e[0] == '0');
}

int bits_for(std::int64_t v) {
  int b = 1;
  while ((std::int64_t(1) << b) <= v) ++b;
  return b;
}

}  // namespace

void list_build(Ctx& c, double cutoff, double skin) {
  if (!(cutoff > 0.0)) throw ConfigError("neighbor cutoff must be positive");
  if (skin < 0.0) throw ConfigError("neighbor skin must be non-negative");
  for (int ax = 0; ax < 3; ++ax)
    if (!(c.box.len[ax] > 0.0)) throw ConfigError("simulation box edges must be positive");
  const double bc = cutoff + skin;
  const double bc2 = bc * bc;
  for (int ax = 0; ax < 3; ++ax)
    if (c.box.per[ax] && c.box.len[ax] < 2.0 * bc)
      throw ConfigError("periodic box edge " + std::to_string(c.box.len[ax]) +
                        " A is below 2*(cutoff+skin) = " + std::to_string(2.0 * bc) +
                        " A; minimum image would be ambiguous");
  c.cutoff = cutoff;
  c.skin = skin;
  const int n = int(c.n);
  // near list (Ctx::near_list): entries within r_cut_max + h, h = s/2, s the
  // list's reach past every cutoff; usable while 2 |d|max + mu < h, mu
  // absorbing the FP64 rounding of the displacements that test relies on
  c.near_ok = false;
  c.near_cut[0] = c.near_cut[1] = 0.0;
  const char* near_env = std::getenv("TSF_NEAR");   // TSF_NEAR=0: off (A/B runs)
  if (c.has_potential && !(near_env && near_env[0] == '0')) {
    const double rf = c.params.r_cut_max();
    const double mu = 1e-6 * std::max(1.0, rf);
    if (bc - rf > 16.0 * mu) {
      for (int q = 0; q < 2; ++q) {
        const double h = 0.25 * (q + 1) * (bc - rf);
        const double t = 0.5 * (h - mu);
        c.near_cut[q] = rf + h;
        c.near_t[q] = std::nextafter(float(t * t), 0.0f);
      }
    }
  }

  // grid (neighbor.cpp:50-77)
  double lo[3] = {0, 0, 0}, hi[3] = {c.box.len[0], c.box.len[1], c.box.len[2]};
  if (!c.box.per[0] || !c.box.per[1] || !c.box.per[2]) {
    DevBuf<unsigned long long> mm;
    mm.reserve(6);
    unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    TSF_CUDA(cudaMemcpyAsync(mm.get(), init, sizeof init, cudaMemcpyHostToDevice, c.stream));
    if (n > 0) {
      k_extent<<<blocks_for(n), kBlock, 0, c.stream>>>(c.pos.get(), n, mm.get());
      ++c.launches;
    }
    unsigned long long got[6];
    TSF_CUDA(cudaMemcpyAsync(got, mm.get(), sizeof got, cudaMemcpyDeviceToHost, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    for (int ax = 0; ax < 3; ++ax) {
      if (c.box.per[ax]) continue;
      double mn = 0.0, mx = c.box.len[ax];
      if (n > 0) {
        mn = from_key(got[ax]);
        mx = from_key(got[3 + ax]);
      }
      lo[ax] = mn;
      hi[ax] = std::max(mx, mn + bc);
    }
  }
  CellGrid& g = c.grid;
  for (int ax = 0; ax < 3; ++ax) {
    g.org[ax] = lo[ax];
    g.ext[ax] = hi[ax] - lo[ax];
    g.nc[ax] = std::max(1, int(std::floor(g.ext[ax] / bc)));
  }
  const std::int64_t ncells = std::int64_t(g.nc[0]) * g.nc[1] * g.nc[2] * slot_classes(c);
  if (ncells > (1ll << 30)) throw ConfigError("cell grid too large");

  // ---- re-sort the atoms by (cell, user index) ----
  const std::size_t nn = std::size_t(std::max(n, 1));
  c.cell_of.reserve(nn);
  c.cell_count.reserve(std::size_t(ncells) + 1);
  c.cell_start.reserve(std::size_t(ncells) + 1);
  c.sort_keys.reserve(nn);
  c.sort_keys_out.reserve(nn);
  c.sort_vals.reserve(nn);
  c.sort_vals_out.reserve(nn);
  c.perm.reserve(nn);
  c.inv.reserve(nn);
  c.tmp4.reserve(nn);
  c.tmp3.reserve(3 * nn);
  const int end_bit = bits_for(ncells);
  std::size_t t_sort = 0, t_scan = 0;
  TSF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_sort, c.sort_keys.get(),
                                           c.sort_keys_out.get(), c.sort_vals.get(),
                                           c.sort_vals_out.get(), std::max(n, 1), 0, end_bit,
                                           c.stream));
  TSF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, c.cell_count.get(), c.cell_start.get(),
                                         int(ncells + 1), c.stream));
  c.scan_tmp.reserve(std::max(t_sort, t_scan));
  TSF_CUDA(cudaMemsetAsync(c.cell_count.get(), 0, sizeof(int) * (ncells + 1), c.stream));
  TSF_CUDA(cudaMemsetAsync(c.flags.get() + 6, 0, sizeof(int), c.stream));
  if (n > 0) {
    k_cell_key<<<blocks_for(n), kBlock, 0, c.stream>>>(
        c.pos.get(), c.sorted ? c.perm.get() : nullptr, n, g,
        c.n_interior >= 0 ? int(std::min<std::int64_t>(c.n_interior, n)) : -1,
        ghost_class_limit(c), c.sort_keys.get(),
        c.sort_vals.get(), c.cell_count.get(), c.flags.get() + 6);
    ++c.launches;
    TSF_CUDA(cub::DeviceRadixSort::SortPairs(c.scan_tmp.get(), t_sort, c.sort_keys.get(),
                                             c.sort_keys_out.get(), c.sort_vals.get(),
                                             c.sort_vals_out.get(), n, 0, end_bit, c.stream));
    ++c.launches;
    k_reorder<<<blocks_for(n), kBlock, 0, c.stream>>>(
        c.sort_keys_out.get(), c.sort_vals_out.get(), n, c.sorted ? 1 : 0, c.pos.get(), c.vel.get(),
        c.tmp4.get(),
        c.tmp3.get(), c.perm.get(), c.inv.get(), c.cell_of.get());
    ++c.launches;
    swap_buf(c.pos, c.tmp4);
    swap_buf(c.vel, c.tmp3);
    refresh_shadow(c);
    c.sorted = true;
    c.forces_current = false;
  }
  TSF_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.get(), t_scan, c.cell_count.get(),
                                         c.cell_start.get(), int(ncells + 1), c.stream));
  ++c.launches;

  c.tiled = true;

  // ---- skin list in slot indices ----
  int cap = c.skin_list.cap > 0 ? c.skin_list.cap : 32;
  for (int attempt = 0; attempt < 3; ++attempt) {
    c.skin_list.nbr.reserve(std::size_t(cap) * c.npad + 1);
    c.skin_list.cnt.reserve(std::size_t(c.npad) + 1);
    if (c.near_cut[0] > 0.0) {
      for (ListState& l : c.near_list) {
        l.nbr.reserve(std::size_t(cap) * c.npad + 1);
        l.cnt.reserve(std::size_t(c.npad) + 1);
      }
      TSF_CUDA(cudaMemsetAsync(c.flags.get() + 11, 0, 6 * sizeof(int), c.stream));
    }
    TSF_CUDA(cudaMemsetAsync(c.skin_list.cnt.get(), 0, sizeof(int) * c.npad, c.stream));
    TSF_CUDA(cudaMemsetAsync(c.flags.get() + 3, 0, sizeof(int), c.stream));
    if (n > 0) launch_skin(c, bc2, cap);
    int f[17] = {0};
    TSF_CUDA(cudaMemcpyAsync(f, c.flags.get(), sizeof f, cudaMemcpyDeviceToHost, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    const int mx = f[3];
    c.skin_list.max_count = mx;
    if (mx <= cap) {
      c.skin_list.cap = cap;
      c.skin_list.valid = true;
      c.adopted_valid = false;
      // the filter requests 4 near_pre entries of a near list up front: the
      // fewest blocks that leave at most 1/256 of the atoms to the serial tail
      const int tail = n / 256;
      for (int q = 0; q < 2; ++q) {
        c.near_list[q].cap = cap;
        const int* o = f + 11 + 3 * q;
        c.near_pre[q] = o[0] <= tail ? 1 : o[1] <= tail ? 2 : o[2] <= tail ? 3 : 4;
      }
      if (std::getenv("TSF_VERBOSE"))
        std::fprintf(stderr,
                     "tsf: list build n=%d skin max %d; near lists: over 4/8/12 %d %d %d, "
                     "%d %d %d -> pre %d %d\n",
                     n, mx, f[11], f[12], f[13], f[14], f[15], f[16], c.near_pre[0],
                     c.near_pre[1]);
      break;
    }
    if (mx > 512)
      throw ConfigError("more than 512 neighbors within cutoff+skin of one atom (" +
                        std::to_string(mx) + ")");
    cap = mx <= 32 ? 32 : mx <= 64 ? 64 : mx <= 128 ? 128 : 512;
  }
  snapshot_reference_positions(c);
  c.near_ok = c.near_cut[0] > 0.0;
  c.short_max_stale = true;
  c.short_list.valid = false;
  ++c.list_version;
  // interior atoms hold slots [0, n_interior) after a split build
  c.split_slots = c.n_interior >= 0 ? std::min<std::int64_t>(c.n_interior, n) : -1;
  c.center_slots = ghost_class_limit(c);
}

void snapshot_reference_positions(Ctx& c) {
  const std::size_t nn = std::size_t(std::max<std::int64_t>(c.n, 1));
  c.pos_ref.reserve(nn);
  c.near_d0.reserve(nn);
  TSF_CUDA(cudaMemcpyAsync(c.pos_ref.get(), c.pos.get(), sizeof(double4) * c.n,
                           cudaMemcpyDeviceToDevice, c.stream));
  TSF_CUDA(cudaMemsetAsync(c.near_d0.get(), 0, sizeof(float4) * nn, c.stream));
  TSF_CUDA(cudaMemsetAsync(c.flags.get() + 10, 0, sizeof(int), c.stream));
  TSF_CUDA(cudaMemsetAsync(c.flags.get() + kFlagNearRefresh, 0, sizeof(int), c.stream));
}

void list_filter(Ctx& c, FilterMode mode, void* zero_forces, int zero_bytes, int lo, int hi,
                 bool zero_flags) {
  if (hi < 0) hi = int(c.n);
  ListState& s = c.short_list;
  s.cap = c.skin_list.cap;
  s.nbr.reserve(std::size_t(s.cap) * c.npad + 1);
  s.cnt.reserve(std::size_t(c.npad) + 1);
  const bool reread = c.short_max_stale || c.short_apply != int(mode);
  if (reread) {
    TSF_CUDA(cudaMemsetAsync(c.flags.get() + 4, 0, sizeof(int), c.stream));
    TSF_CUDA(cudaMemsetAsync(c.flags.get() + 8, 0, 2 * sizeof(int), c.stream));
  }
  const PairBounds pb = pair_bounds(c, mode);
  if (c.n > 0) {
    // (a TMA-staged, persistent variant measured slower: 0.138 vs 0.114 ms at
    // 2M atoms — its staging buffers take the L1 the position gathers hit,
    // 58% -> 9% hit rate)
    NearIn near{};
    if (c.near_ok && mode != FilterMode::Copy) {
      near.nbr[0] = c.near_list[0].nbr.get();
      near.nbr[1] = c.near_list[1].nbr.get();
      near.cnt[0] = c.near_list[0].cnt.get();
      near.cnt[1] = c.near_list[1].cnt.get();
      near.dmax = c.flags.get() + 10;
      near.t[0] = c.near_t[0];
      near.t[1] = c.near_t[1];
      near.pre[0] = c.near_pre[0];
      near.pre[1] = c.near_pre[1];
      // refresh only where a force launch (its k_reduce restarts the
      // maximum) follows a filter over every slot: two-phase evaluations
      // decide per phase and keep the stale-list fallback
      near.refresh = mode == FilterMode::Pair && lo == 0 && hi == int(c.n) && zero_flags &&
                     near_refresh_enabled();
      const double rf = c.params.r_cut_max();
      const PairBounds sb = sure_bound(c, true);
      for (int q = 0; q < 2; ++q) {
        near.cut[q] = c.near_cut[q];
        near.sure_cut[q] = sb.cut[0] - (c.near_cut[q] - rf);
      }
      near.ref = c.pos_ref.get();
      near.d0 = c.near_d0.get();
      near.refreshed = c.flags.get() + kFlagNearRefresh;
    }
    near.skip = c.speculative ? c.flags.get() + kFlagMoved : nullptr;
    (pb.ns > 1 ? k_filter<true> : k_filter<false>)<<<blocks_for(std::max(hi - lo, 1)), kBlock, 0,
                                                       c.stream>>>(
        list_args(c), pb, mode != FilterMode::Copy ? 1 : 0, c.skin_list.nbr.get(),
        c.skin_list.cnt.get(), s.nbr.get(), s.cnt.get(), reread ? c.flags.get() + 4 : nullptr,
        c.flags.get() + 8, zero_forces, zero_forces ? zero_bytes : 0, lo, hi, near,
        zero_flags ? c.flags.get() : nullptr,
        zero_flags && !c.main_packed ? c.flags.get() + kFlagOver4 : nullptr);
    // (a packed main launch has no tier to gate: irregular systems skip the mark)
    c.filter_marks_over4 = zero_flags && !c.main_packed;
    ++c.launches;
  }
  s.valid = true;
  if (reread) {
    // The short-count distribution sizes the force kernel's lane group; read
    // it back only after a rebuild — between rebuilds outgrown atoms take the
    // overflow path, so the steady state never synchronizes here.
    int f[10] = {0};
    TSF_CUDA(cudaMemcpyAsync(f, c.flags.get(), sizeof f, cudaMemcpyDeviceToHost, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    s.max_count = f[4];
    s.over4 = f[8];
    s.over8 = f[9];
    c.short_max_stale = false;
    c.short_apply = int(mode);
  }
}

bool list_needs_rebuild(Ctx& c) {
  if (!c.skin_list.valid) return true;
  TSF_CUDA(cudaMemsetAsync(c.flags.get() + kFlagMoved, 0, sizeof(int), c.stream));
  if (c.n > 0) {
    k_needs_rebuild<<<blocks_for(c.n), kBlock, 0, c.stream>>>(
        c.pos.get(), c.pos_ref.get(), int(c.n), c.box, 0.25 * c.skin * c.skin,
        c.flags.get() + kFlagMoved);
    ++c.launches;
  }
  int f = 0;
  TSF_CUDA(cudaMemcpyAsync(&f, c.flags.get() + kFlagMoved, sizeof(int), cudaMemcpyDeviceToHost,
                           c.stream));
  TSF_CUDA(cudaStreamSynchronize(c.stream));
  return f != 0;
}

}  // namespace tsf
