// Tersoff energy / forces / virial on the short list — the hot path.
//
// Replaces evaluate_forces' kernels (proj/include/tmd/kernels.hpp:175-494,
// proj/src/potential_ref.cpp:75-134; paper Alg. 2/3 and Fig. 3).
//
// Mapping ("lane group per atom", the GPU form of the paper's scheme (a)):
//   * a group of G lanes (G = 4, 8, 16 or 32; G >= the atom's short count)
//     owns central atom i; lane l holds short neighbour j_l, its FP64
//     displacement (the reference's exact rounding, so the cutoff decisions are
//     the reference's), r, 1/r, unit vector and f_C(r), f_C'(r), staged in
//     shared memory as 128-bit vectors;
//   * zeta pass: at rotation t lane l pairs with k = slot (l + t) mod n_i
//     (t = 1..n_i-1 visits every k != j once); the triplet's d zeta/d x_j is
//     accumulated in registers and d zeta/d x_k cached in registers (Alg. 3's
//     derivative cache with k_max = G - 1; recomputed for G > 8);
//   * pair block: V, dV/dr, dV/dzeta with the log-space bond order;
//   * scatter pass: at rotation t lane l hands its cached d zeta/d x_k times
//     dV/dzeta_j to lane (l + t) mod n_i with one shuffle — the transposed
//     reduction — so every lane ends with P_l, the total force atom i's terms
//     put on neighbour j_l, and F_i = -sum_l P_l (translation invariance);
//   * atomic mode: one atomicAdd per neighbour slot and component, one for i;
//     deterministic mode: P_l goes to a slot buffer and k_gather sums every
//     atom's incoming slots in list order — bitwise reproducible;
//   * energy and virial (W_ab = sum_l d_a P_b) are reduced per block into a
//     partials array and summed in fixed order; atoms taken by the tier
//     launches (queued in atomic order) keep theirs per atom in deterministic
//     mode, summed in atom order by k_queued_ev — bitwise reproducible.
// The grid is persistent (occupancy x 148 blocks striding over atom tiles)
// and software-pipelined: while tile k computes, the positions of tile k+1
// and the list entries of tile k+2 are already in flight (the dependent
// count -> index -> position loads were 35% of the stall samples, ncu).
// Atoms whose short count exceeds G are queued and processed by the same code
// in tier launches — G = 16 (two atoms per warp), then G = 32 for what is
// left — that exit at once when their queue is empty.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "tsf_context.hpp"

namespace tsf {

namespace {

template <typename R>
struct ForceArgs {
  Row<R> row0;         // single-species row: read straight from the constant bank
  double cut0;
  const double4* pos;
  int n_owned;         // end of the slot range to cover (all local atoms: n)
  int slot_base;       // start of the slot range (two-phase evaluation: 0 or n_interior)
  int n_all;           // local atoms (neighbour indices lie in [0, n_all))
  const int* perm;     // slot -> user index (nullptr: identity)
  int center_limit;    // only user atoms below this act as centers (ghosts above)
  int energy_limit;    // only centers below this count energy and virial (owned atoms;
                       // the ghost centers between them give the owned atoms' forces)
  int npad;
  Box box;
  const int* nbr;      // short list, ELL column-major
  const int* cnt;
  const void* rows;
  const double* cutsq;
  int ns;
  void* forces;        // atomic mode: Acc[n][3]
  void* slot_x;        // deterministic mode: Acc[cap * npad] per component
  void* slot_y;
  void* slot_z;
  void* fself;         // deterministic mode: Acc[n][3]
  double* partials;    // [blocks][kRedWidth]
  int partial_base;
  // Atoms with more short entries than the group width are queued for a
  // wider tier launch (main G=4/8 -> G=16 -> G=32); the last tier flags them.
  const int* ovf_in;        // tier launches: queued slots and their count
  const int* ovf_in_count;
  int* ovf_out;             // nullptr: more than G entries is an error (unless ovf_scan)
  int* ovf_out_count;
  // ovf_scan: the main launch leaves atoms over its width to a packed tier
  // launch that finds them itself (short count > scan_g) — no queue
  int ovf_scan;
  int scan_g;
  const int* over4;         // scanning tier: flags[kFlagOver4] (nullptr: always scan)
  double* atom_ev;          // deterministic tiers: per-atom energy + virial [n][8]
  int* flags;               // [0] error bits
  const int* skip;          // speculative MD step: return at once when *skip != 0
};

constexpr unsigned kFull = 0xffffffffu;

// non-blocking L2 prefetch (no register is written)
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Which exponentials use the branch-free constant-bank exp (tsf_math.cuh
// exp_cb, Estrin) instead of libdevice's: 0 none, 1 the triplet's, 2 also the
// pair terms'.  Measured (tools/ab.py, si2m f64 kernel): 0 0.320 ms, 1 0.344,
// 2 0.345 — libdevice's exp (one integer scale, a rarely taken range branch)
// beats the branch-free two-factor form despite the ILP the latter allows.
#ifndef TSF_EXP_FIN
#define TSF_EXP_FIN 0
#endif

// Parameter-table specialisations.
enum Spec : int {
  kSingle = 0,   // one species, m = 3: the row comes from the constant bank
  kHoist = 1,    // several species, ramp (R, D) depends on (i, k) only
  kGeneric = 2,  // anything else: ramp and cutoff test per triplet
};

template <typename R>
struct Nbr {
  R ux, uy, uz, r, ir;
};

// One triplet's zeta term and its gradients as scalar coefficients on the two
// unit vectors: d z/d x_j = u_k A + u_j B, d z/d x_k = u_j C + u_k D.  The
// 3-vectors are never formed per triplet: the j-gradient sums become
// sum(u_k A) and sum(B), and the scatter pass sends (C, D) times dV/dzeta —
// two scalars instead of three components — to the lane that owns k, which
// holds u_k itself and reads u_j from the staging (11 fewer FP64 operations
// per triplet than the vector form, a third fewer values in the k-cache).
template <typename R>
struct Grad {
  R z, A, B, C, D;
};

// Per-lane neighbour record in shared memory, 128-bit vectors.
template <typename R> struct Stage;
template <> struct Stage<double> {
  double2 a[kBlock];   // ux, uy
  double2 b[kBlock];   // uz, r
  double2 c[kBlock];   // 1/r, fc
  double2 d[kBlock];   // fc', meta (species, -1 when not a usable k; int bits)
  __device__ void put(int t, const Nbr<double>& n, double fc, double dfc, int meta) {
    a[t] = make_double2(n.ux, n.uy);
    b[t] = make_double2(n.uz, n.r);
    c[t] = make_double2(n.ir, fc);
    d[t] = make_double2(dfc, __hiloint2double(0, meta));
  }
  __device__ void get(int t, Nbr<double>& n, double& fc, double& dfc, int& meta) const {
    const double2 va = a[t], vb = b[t], vc = c[t], vd = d[t];
    n.ux = va.x; n.uy = va.y; n.uz = vb.x; n.r = vb.y; n.ir = vc.x;
    fc = vc.y; dfc = vd.x; meta = __double2loint(vd.y);
  }
  __device__ void unit(int t, double& ux, double& uy, double& uz) const {
    const double2 va = a[t];
    ux = va.x; uy = va.y; uz = b[t].x;
  }
};
template <> struct Stage<float> {
  float4 a[kBlock];    // ux, uy, uz, r
  float4 b[kBlock];    // 1/r, fc, fc', meta (int bits)
  __device__ void put(int t, const Nbr<float>& n, float fc, float dfc, int meta) {
    a[t] = make_float4(n.ux, n.uy, n.uz, n.r);
    b[t] = make_float4(n.ir, fc, dfc, __int_as_float(meta));
  }
  __device__ void get(int t, Nbr<float>& n, float& fc, float& dfc, int& meta) const {
    const float4 va = a[t], vb = b[t];
    n.ux = va.x; n.uy = va.y; n.uz = va.z; n.r = va.w; n.ir = vb.x;
    fc = vb.y; dfc = vb.z; meta = __float_as_int(vb.w);
  }
  __device__ void unit(int t, float& ux, float& uy, float& uz) const {
    const float4 va = a[t];
    ux = va.x; uy = va.y; uz = va.z;
  }
};

// One (i, j, k) triplet: zeta term and its j and k gradients
// (potential.hpp:132-198; the i gradient is never formed: F_i = -sum P).
// A triplet that does not count enters with fck = dfck = 0 and ok = false:
// every output is then exactly zero (the exponent argument is zeroed too, so
// no inf can meet the zero), which replaces seven selects per triplet.
// CUB: 1 the exponent is cubic (m = 3), 0 linear, -1 read from the row.
template <typename R, int CUB = -1, bool EXPNB = false>
__device__ __forceinline__ Grad<R> triplet(const Nbr<R>& j, const Nbr<R>& k, R fck, R dfck,
                                           bool ok, const Row<R>& p) {
  Grad<R> o;
  R cs = j.ux * k.ux + j.uy * k.uy + j.uz * k.uz;
  // clamp to [-1, 1] (potential.hpp:155).  FP64: one compare — fmin/fmax on
  // doubles cost ~12 instructions here (1-3% of the kernel, tools/ab.py);
  // identical for every finite cs.  Float: two FMNMX are cheaper.
  if constexpr (std::is_same<R, double>::value) {
    if (fabs(cs) > R(1)) cs = copysign(R(1), cs);
  } else {
    cs = fminf(1.0f, fmaxf(-1.0f, cs));
  }
  const R t = p.h - cs;
  const R den = p.d2 + t * t;
  const R iden = Fn<R>::rcp(den);
  const R g = p.gamma + p.gcd2 * (t * t) * iden;
  const R dg = R(-2) * p.gc2 * t * iden * iden;
  // e^{(lam3 q)^m} = exp_row(tc q^m), d/dq = td q^(m-1) e^{...} (make_row)
  const R q = ok ? j.r - k.r : R(0);
  const bool cubic = CUB > 0 || (CUB < 0 && p.m3 != R(0));
  const R q2 = q * q;
  const R x = cubic ? p.tc * (q2 * q) : p.tc * q;
  R ex;
  if constexpr (!std::is_same<R, double>::value) {
    ex = Fn<R>::exp_row(x);   // base 2
  } else if constexpr (EXPNB) {
    ex = Fn<R>::exp_nb(x);
  } else if constexpr (CUB < 0) {
    // multi-species tables: Tersoff's 1989 SiC / SiGe rows carry lambda3 = 0,
    // where the factor is exactly e^0 = 1 (uniform branch; 11% of the SiC
    // kernel's instructions were that exp)
    if (p.tc != R(0)) ex = TSF_EXP_FIN >= 1 ? Fn<R>::exp_fin(x) : Fn<R>::exp_(x);
    else ex = R(1);
  } else {
    ex = TSF_EXP_FIN >= 1 ? Fn<R>::exp_fin(x) : Fn<R>::exp_(x);
  }
  const R gx = g * ex;
  o.z = fck * gx;
  const R fge = o.z * (cubic ? p.td * q2 : p.td);                      // dz/dr_ij via exp
  const R fgd = fck * dg * ex;                                          // dz/dcos
  const R cge = dfck * gx;                                              // dz/dr_ik via f_C
  // dcos/dx_j = (u_k - u_j cos)/r_ij, dcos/dx_k = (u_j - u_k cos)/r_ik, folded:
  //   dz/dx_j = u_k A + u_j (fge - cos A),             A = fgd / r_ij
  //   dz/dx_k = u_j C + u_k (cge - fge - cos C),       C = fgd / r_ik
  o.A = fgd * j.ir;
  o.B = fge - cs * o.A;
  o.C = fgd * k.ir;
  o.D = (cge - fge) - cs * o.C;
  return o;
}

// Loads one tile needs before it can compute: count + list entry (stage A),
// then the two positions (stage B, dependent on stage A).
struct TileIdx {
  int i, n, j;
  bool ghost;     // a decomposition ghost: receives forces, is not a centre
};

// Resident blocks per SM the register allocation must allow (B200, si2m /
// liquid512k sweeps): FP64 4 (128 registers; unbounded it takes 168 and
// runs 12% slower, 5+ blocks spill), float 6 (80 registers, +5%).
#ifndef TSF_FORCE_MINB_F64
#define TSF_FORCE_MINB_F64 4
#endif
#ifndef TSF_FORCE_MINB_F32
#define TSF_FORCE_MINB_F32 6
#endif
#ifndef TSF_FORCE_MINB_F64_G8
#define TSF_FORCE_MINB_F64_G8 TSF_FORCE_MINB_F64
#endif
#ifndef TSF_FORCE_MINB_F32_G8
#define TSF_FORCE_MINB_F32_G8 5   // unrolled G = 8 cache: 96 registers, no spills
#endif
template <typename R, int G>
constexpr int kForceMinBlocks = G == 8 ? TSF_FORCE_MINB_F64_G8 : TSF_FORCE_MINB_F64;
template <int G>
constexpr int kForceMinBlocks<float, G> = G == 8 ? TSF_FORCE_MINB_F32_G8 : TSF_FORCE_MINB_F32;

}  // namespace
}  // namespace tsf
#include "tsf_force_packed.cuh"
namespace tsf {
namespace {

#ifndef TSF_MERGE_TIER
#define TSF_MERGE_TIER 1
#endif
// MERGE: the FP64 single-species G = 4 main launch runs the packed tier
// itself (packed_work, OVF) after its tiles — the atoms over 4 found by the
// same count scan — so the separate tier launch leaves the chain (both use
// 128 registers; the float main kernel's 80 would not survive the merge).
// Small systems only (kMergeMaxAtoms): at 32k atoms the evaluation is a chain
// of latency-bound launches (-11% per evaluation, -7% per MD step), while at
// 2M the merged code's spills in the main loop cost more than the launch.
constexpr std::int64_t kMergeMaxAtoms = 1 << 20;
template <typename R, int G, int SPEC, bool OVF>
constexpr bool kMergeTier =
    TSF_MERGE_TIER && G == 4 && SPEC == kSingle && !OVF && std::is_same<R, double>::value;

template <typename R, typename Acc, int G, int SPEC, bool DET, bool OVF, bool FOREIGN = false,
          bool VIR = true, bool EXPNB = false, bool MERGE = false>
__global__ void __launch_bounds__(kBlock, (kForceMinBlocks<R, G>))
    k_force(const __grid_constant__ ForceArgs<R> a) {
#ifndef TSF_CACHE_G16
#define TSF_CACHE_G16 1
#endif
  // cache of d zeta / d x_k for the scatter pass (else recomputed there)
  constexpr bool kCache = G <= 8 || (G == 16 && TSF_CACHE_G16);
  constexpr int kUnroll = kCache && G <= 8 ? G - 1 : 2;   // full unroll keeps it in registers
  // FP64 G = 8 and G = 16: early exit at the warp's largest count keeps the
  // loop rolled and the cache in (L1-backed) local memory — for FP64 G = 8
  // 2-6% faster than the unrolled, register-capped form; float G = 8 unrolls
  // (liquid512k / sic256k sweeps, tools/ab.py)
  constexpr bool kRolled = (G == 8 && std::is_same<R, double>::value) || G == 16;
  constexpr int kRows = kMaxSpecies * kMaxSpecies * kMaxSpecies;
  __shared__ Row<R> srow[SPEC == kSingle ? 1 : kRows];
  __shared__ double scut[SPEC == kSingle ? 1 : kRows];
  __shared__ Stage<R> st;
  __shared__ double s_r2[SPEC == kGeneric ? kBlock : 1];
  __shared__ double s_red[kBlock / 32][kRedWidth];
  constexpr bool kMerge = MERGE && kMergeTier<R, G, SPEC, OVF>;
  __shared__ std::conditional_t<kMerge, PackedShared<R, Acc, SPEC, DET, true>, char> s_tier;

  griddep_wait();     // launch_pdl: the previous launch has completed
  griddep_launch();
  if (a.skip && (a.skip[0] | a.skip[kFlagMovedAny - kFlagMoved])) return;   // stale list
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  Acc e_acc = 0;
  Acc w_acc[6] = {0, 0, 0, 0, 0, 0};

  const int n_ovf = OVF ? *a.ovf_in_count : 0;
  if (OVF && n_ovf == 0) {              // nothing queued: leave a zero partial
    if (tid < kRedWidth)
      a.partials[std::size_t(a.partial_base + blockIdx.x) * kRedWidth + tid] = 0.0;
    return;
  }

  const int ns = a.ns;
  const Row<R>* rows = static_cast<const Row<R>*>(a.rows);
  const Row<R>& row0 = a.row0;
  const double cut0 = a.cut0;
  if (SPEC != kSingle) {
    for (int q = tid; q < ns * ns * ns; q += blockDim.x) {
      srow[q] = rows[q];
      scut[q] = a.cutsq[q];
    }
    __syncthreads();
  }

  const int gl = tid & (G - 1);
  const int gbase = tid - gl;          // block-local thread id of slot 0
  const int wbase = lane - gl;         // warp lane of slot 0
  constexpr int kAtomsPerBlock = kBlock / G;
  const int ntiles = (a.n_owned - a.slot_base + kAtomsPerBlock - 1) / kAtomsPerBlock;
  const int nwarps_total = gridDim.x * (kBlock / 32);
  const int last = a.n_all - 1;
  const bool has_ghosts = a.center_limit < a.n_owned;
  // ghost centres (tsf_set_centers) exist only in FOREIGN instantiations: a
  // runtime test in the common kernel cost 1-2% (tools/ab.py)
  const bool has_foreign = FOREIGN && a.energy_limit < a.center_limit;

  // stage A loads: count and this lane's list entry (clamped into range; the
  // entry past the count is unused, it only keeps the dependent load legal)
  auto load_idx = [&](int tile) {
    TileIdx t;
    t.i = a.slot_base + tile * kAtomsPerBlock + tid / G;
    const bool in = tile < ntiles && t.i < a.n_owned;
    if (!in) t.i = 0;
    TSF_DCHECK(!in || (t.i >= 0 && t.i < a.n_all), "k_force centre slot");
    t.n = in ? a.cnt[t.i] : 0;
    const int v = in ? a.nbr[ell_at(gl, t.i, a.npad)] : 0;
    TSF_DCHECK(!in || gl >= t.n || (v >= 0 && v <= last && v != t.i), "k_force list entry");
    t.j = unsigned(v) <= unsigned(last) ? v : 0;
    // ghost tests two tiles ahead (the perm[] load at the tile start was 24%
    // of the stall samples, ncu); skipped when the context has no ghosts
    t.ghost = has_ghosts && in && (a.perm ? a.perm[t.i] : t.i) >= a.center_limit;
    return t;
  };

  constexpr int kPerWarp = 32 / G;     // tier launches: queued atoms per warp
  int work = OVF ? blockIdx.x * (kBlock / 32) + tid / 32 : blockIdx.x;
  TileIdx nxt{0, 0, 0, false}, nxt2{0, 0, 0, false};
  double4 pi_n = make_double4(0, 0, 0, 0), pj_n = pi_n;
  if (!OVF) {
    nxt = load_idx(work);
    pi_n = a.pos[nxt.i];
    pj_n = a.pos[nxt.j];
    nxt2 = load_idx(work + gridDim.x);
  }

  while (true) {
    int i, n_i, j;
    double4 pi, pj;
    bool active, foreign;
    if (OVF) {
      if (work * kPerWarp >= n_ovf) break;   // warp-uniform
      const int q = work * kPerWarp + lane / G;
      active = q < n_ovf;
      i = a.ovf_in[active ? q : work * kPerWarp];
      foreign = has_foreign && (a.perm ? a.perm[i] : i) >= a.energy_limit;
      n_i = active ? a.cnt[i] : 0;
      j = gl < n_i ? a.nbr[ell_at(gl, i, a.npad)] : i;
      pi = a.pos[i];
      pj = a.pos[j];
    } else {
      if (work >= ntiles) break;       // block-uniform
      i = nxt.i;
      n_i = nxt.n;
      j = nxt.j;
      const bool ghost = nxt.ghost;
      // a ghost centre (ghost-centre decompositions only: no load otherwise)
      foreign = has_foreign && (a.perm ? a.perm[i] : i) >= a.energy_limit;
      pi = pi_n;
      pj = pj_n;
      // keep the pipeline full: positions of the next tile, list of the one after
      nxt = nxt2;
      pi_n = a.pos[nxt.i];
      pj_n = a.pos[nxt.j];
      nxt2 = load_idx(work + 2 * gridDim.x);
      active = a.slot_base + work * kAtomsPerBlock + tid / G < a.n_owned;
      // ghost copies (decomposition) receive forces but are not centers
      if (active && ghost) {
        if (DET) {
          // a ghost contributes nothing here (its owner evaluates it): zero
          // its self term and the slots k_gather reads for its neighbours
          if (gl == 0) {
            Acc* f = static_cast<Acc*>(a.fself) + 3 * std::size_t(i);
            f[0] = f[1] = f[2] = Acc(0);
          }
          for (int sl = gl; sl < n_i; sl += G) {
            const std::size_t q = std::size_t(sl) * a.npad + i;
            static_cast<Acc*>(a.slot_x)[q] = Acc(0);
            static_cast<Acc*>(a.slot_y)[q] = Acc(0);
            static_cast<Acc*>(a.slot_z)[q] = Acc(0);
          }
        }
        active = false;
      }
      if (!active) n_i = 0;
    }
    // atoms over the width go to the next tier's queue.  The FP64 G = 4 main
    // launch (3C-SiC in f64 queues 45% of its atoms) and the tier launches
    // take one atomic per warp, and a warp's atoms land side by side in slot
    // order, so the next launch reads neighbouring slots — SiC f64 step -8%
    // against an atomic per atom (arrival order, every queued atom serialised
    // on one address).  The other main launches queue few atoms and keep the
    // per-atom form (tools/ab.py: the vote cost the float G = 4 kernel 1%).
    if constexpr ((G == 4 && std::is_same<R, double>::value) || OVF) {
      const bool over = n_i > G;
      const unsigned lead = a.ovf_scan ? 0u : __ballot_sync(kFull, over && gl == 0);
      if (lead) {                      // warp-uniform
        if (a.ovf_out) {
          const int first = __ffs(lead) - 1;
          int base = 0;
          if (lane == first) base = atomicAdd(a.ovf_out_count, __popc(lead));
          base = __shfl_sync(kFull, base, first);
          if (over && gl == 0) a.ovf_out[base + __popc(lead & ((1u << lane) - 1u))] = i;
        } else if (over && gl == 0) {
          atomicOr(a.flags, kErrShortOverflow);
        }
      }
      if (over) {
        n_i = 0;
        active = false;
      }
    } else {
      if (n_i > G) {
        if (gl == 0 && !a.ovf_scan) {
          if (a.ovf_out) a.ovf_out[atomicAdd(a.ovf_out_count, 1)] = i;
          else atomicOr(a.flags, kErrShortOverflow);
        }
        n_i = 0;
        active = false;
      }
    }
    const bool slot = gl < n_i;
    double dx = 0, dy = 0, dz = 0, r2 = 1.0;
    if (slot) {
      displacement(pi, pj, a.box, dx, dy, dz);
      r2 = norm_sq_exact(dx, dy, dz);
    }
    const int si = SPEC == kSingle ? 0 : species_of(pi);
    const int sj = SPEC == kSingle ? 0 : species_of(pj);
    const int row_jj = (si * ns + sj) * ns + sj;
    const bool pair_ok = slot && r2 <= (SPEC == kSingle ? cut0 : scut[row_jj]);
    const Row<R>& pjj = SPEC == kSingle ? row0 : srow[row_jj];

    Nbr<R> me;
    me.ir = Fn<R>::rsqrt_(R(r2));      // one rsqrt gives 1/r and r
    me.r = R(r2) * me.ir;
    me.ux = R(dx) * me.ir;
    me.uy = R(dy) * me.ir;
    me.uz = R(dz) * me.ir;
    R fc, dfc;
    cutoff_ramp(me.r, pjj, fc, dfc);
    // the radial pair terms depend on r only: issued before the zeta pass so
    // their two exp chains overlap it instead of lengthening the pair block
    // (r <= 1 on empty slots, the pair cutoff otherwise: EXPNB's bound holds)
    const R fr = pjj.a * (EXPNB ? Fn<R>::exp_nb(pjj.e1 * me.r) : Fn<R>::exp_row(pjj.e1 * me.r));
    const R fa = -(pjj.b * (EXPNB ? Fn<R>::exp_nb(pjj.e2 * me.r) : Fn<R>::exp_row(pjj.e2 * me.r)));
    // meta: species of this slot as a k, or -1 when it can never be one.
    // With the ramp (and so the cutoff) fixed by (i, k), "usable as k" is
    // exactly "pair (i, k) inside its own cutoff".
    const int meta = SPEC == kGeneric ? (slot ? sj : -1) : (pair_ok ? sj : -1);
    // single species at G = 4 (kNoMask): a slot that is no usable k stages
    // f_C = f_C' = 0, so its triplets are exact zeros without a mask — and
    // a lane whose own pair is out has dV/dzeta = 0, which zeroes everything
    // its triplets send (every exponential argument is bounded: dispatch
    // requires Row::exp_ok for kSingle)
    constexpr bool kNoMask = SPEC == kSingle && G == 4;
    if (kNoMask) st.put(tid, me, pair_ok ? fc : R(0), pair_ok ? dfc : R(0), meta);
    else st.put(tid, me, fc, dfc, meta);
    if (SPEC == kGeneric) s_r2[tid] = r2;
    __syncwarp();

    const int rowbase = (si * ns + sj) * ns;
    // Wider groups serve irregular systems (liquid, SiC): stop the rotations
    // at the warp's largest count instead of G - 1.  (G = 4 keeps the
    // straight-line loop: crystals fill every lane and it schedules better.)
    const int tmax = G > 4 ? __reduce_max_sync(kFull, n_i) : G;

    // ---- zeta pass: partner k = slot (l + t) mod n_i ----
    // zeta, the j-gradient as u_j sum(B) + sum(u_k A), the k-coefficients (C, D)
    R zeta = 0, sb = 0, gjx = 0, gjy = 0, gjz = 0;
    R ckc[kCache ? G : 1], ckd[kCache ? G : 1];
#pragma unroll kUnroll
    for (int t = 1; t < G; ++t) {
      if (G > 4 && t >= tmax) {           // warp-uniform
        if (kRolled) break;
        continue;
      }
      int m = gl + t;   // G = 4: (l + t) mod 4 whatever n_i <= 4 (empty slots: meta masks them)
      if (G == 4) m &= 3;
      else if (m >= n_i) m -= n_i;
      const int src = gbase + (m & (G - 1));
      Nbr<R> k;
      R fck, dfck;
      int kmeta;
      st.get(src, k, fck, dfck, kmeta);
      bool ok = pair_ok && (G == 4 || t < n_i) && kmeta >= 0;
      const Row<R>* prow = &pjj;
      if (SPEC != kSingle) {
        const int sk = max(kmeta, 0);
        prow = &srow[rowbase + sk];
        if (SPEC == kGeneric) {
          ok = ok && s_r2[src] <= scut[rowbase + sk];
          cutoff_ramp(k.r, *prow, fck, dfck);
        }
      }
      if (!kNoMask) {
        fck = ok ? fck : R(0);
        dfck = ok ? dfck : R(0);
      }
      const Grad<R> tr =
          triplet<R, (SPEC == kSingle ? 1 : -1), EXPNB>(me, k, fck, dfck, kNoMask || ok, *prow);
      zeta += tr.z;
      sb += tr.B;
      gjx += k.ux * tr.A;
      gjy += k.uy * tr.A;
      gjz += k.uz * tr.A;
      if constexpr (kCache) {
        ckc[t] = tr.C;
        ckd[t] = tr.D;
      }
    }

    // ---- pair block (potential.hpp:204-222) ----
    R dvdr = 0, dvdz = 0, v = 0;
    if (pair_ok) {
      const R dfr = -pjj.lam1 * fr;
      const R dfa = -pjj.lam2 * fa;
      R b, db;
      bond_order(zeta, pjj, b, db);
      const R rep = fr + b * fa;
      v = R(0.5) * fc * rep;
      dvdr = R(0.5) * (dfc * rep + fc * (dfr + b * dfa));
      dvdz = R(0.5) * fc * fa * db;
      // one test: a non-finite term makes the sum non-finite (the terms are
      // far below the range where finite ones could overflow it)
      if (!isfinite(v + dvdr + dvdz)) atomicOr(a.flags, kErrNonFinite);
    }
    // P_l = -(u_l (dV/dr + dV/dzeta sum B + sum_s D_s) + dV/dzeta sum(u_k A)
    //        + sum_s u_s C_s), s over the lanes whose k is l
    R alpha = dvdr + dvdz * sb;
    R px = -(gjx * dvdz);
    R py = -(gjy * dvdz);
    R pz = -(gjz * dvdz);

    // ---- scatter pass: lane (l + t) mod n receives lane l's (C, D) dV/dzeta ----
    // Every lane of a group shares n_i, and a sender's coefficients for
    // rotation t are zero unless t < n_i and its triplet counts, so receivers
    // need no mask (an empty slot's staged unit vector is 0).
#pragma unroll kUnroll
    for (int t = 1; t < G; ++t) {
      if (G > 4 && t >= tmax) {           // warp-uniform
        if (kRolled) break;
        continue;
      }
      R sc, sd;
      if constexpr (kCache) {
        sc = ckc[t] * dvdz;
        sd = ckd[t] * dvdz;
      } else {
        int m = gl + t;   // G = 4: (l + t) mod 4 whatever n_i <= 4 (empty slots: meta masks them)
        if (G == 4) m &= 3;
        else if (m >= n_i) m -= n_i;
        const int src = gbase + (m & (G - 1));
        Nbr<R> k;
        R fck, dfck;
        int kmeta;
        st.get(src, k, fck, dfck, kmeta);
        bool ok = pair_ok && (G == 4 || t < n_i) && kmeta >= 0;
        const Row<R>* prow = &pjj;
        if (SPEC != kSingle) {
          const int sk = max(kmeta, 0);
          prow = &srow[rowbase + sk];
          if (SPEC == kGeneric) {
            ok = ok && s_r2[src] <= scut[rowbase + sk];
            cutoff_ramp(k.r, *prow, fck, dfck);
          }
        }
        fck = ok ? fck : R(0);
        dfck = ok ? dfck : R(0);
        const Grad<R> tr = triplet<R, (SPEC == kSingle ? 1 : -1), EXPNB>(me, k, fck, dfck, ok, *prow);
        sc = tr.C * dvdz;
        sd = tr.D * dvdz;
      }
      int s = gl - t;
      if (G == 4) s &= 3;
      else if (s < 0) s += n_i;
      const int from = s & (G - 1);
      const R rc = __shfl_sync(kFull, sc, wbase + from);
      alpha += __shfl_sync(kFull, sd, wbase + from);
      R sux, suy, suz;
      st.unit(gbase + from, sux, suy, suz);
      px -= sux * rc;
      py -= suy * rc;
      pz -= suz * rc;
    }
    px -= me.ux * alpha;
    py -= me.uy * alpha;
    pz -= me.uz * alpha;
    // (kNoMask: an empty slot's P is already +-0 — dV/dzeta = 0 and every
    // sender's coefficients for it carry its staged f_C = 0)
    if (!kNoMask && !slot) px = py = pz = 0;

    // F_i = -sum over the group's slots
    R fx = px, fy = py, fz = pz;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      fx += __shfl_xor_sync(kFull, fx, o);
      fy += __shfl_xor_sync(kFull, fy, o);
      fz += __shfl_xor_sync(kFull, fz, o);
    }

    if constexpr (OVF && DET) {
      // queue order (and so the block) varies run to run: keep this atom's
      // energy and virial per atom; k_queued_ev sums them in atom order
      const R rx = R(dx), ry = R(dy), rz = R(dz);
      Acc ev[7] = {Acc(v), Acc(rx * px), Acc(ry * py), Acc(rz * pz),
                   Acc(rx * py), Acc(rx * pz), Acc(ry * pz)};
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        if (!slot || (FOREIGN && foreign) || (!VIR && q > 0)) ev[q] = Acc(0);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) ev[q] += __shfl_xor_sync(kFull, ev[q], o);
      }
      if (active && gl == 0)
#pragma unroll
        for (int q = 0; q < 7; ++q) a.atom_ev[8 * std::size_t(i) + q] = double(ev[q]);
    }
    if (slot) {
      if constexpr (!(OVF && DET)) if (!FOREIGN || !foreign) {   // ghost centres: forces only
        e_acc += Acc(v);
        if constexpr (VIR) {   // (no caller asked for the virial: not formed)
          const R rx = R(dx), ry = R(dy), rz = R(dz);
          w_acc[0] += Acc(rx * px);
          w_acc[1] += Acc(ry * py);
          w_acc[2] += Acc(rz * pz);
          w_acc[3] += Acc(rx * py);
          w_acc[4] += Acc(rx * pz);
          w_acc[5] += Acc(ry * pz);
        }
      }
      TSF_DCHECK(j >= 0 && j <= last && i >= 0 && i <= last, "k_force scatter target");
      if (DET) {
        const std::size_t q = std::size_t(gl) * a.npad + i;
        static_cast<Acc*>(a.slot_x)[q] = Acc(px);
        static_cast<Acc*>(a.slot_y)[q] = Acc(py);
        static_cast<Acc*>(a.slot_z)[q] = Acc(pz);
      } else {
        Acc* f = static_cast<Acc*>(a.forces) + 3 * std::size_t(j);
        atomicAdd(f + 0, Acc(px));
        atomicAdd(f + 1, Acc(py));
        atomicAdd(f + 2, Acc(pz));
      }
    }
    if (active && gl == 0) {
      if (DET) {
        Acc* f = static_cast<Acc*>(a.fself) + 3 * std::size_t(i);
        f[0] = Acc(-fx);
        f[1] = Acc(-fy);
        f[2] = Acc(-fz);
      } else {
        Acc* f = static_cast<Acc*>(a.forces) + 3 * std::size_t(i);
        atomicAdd(f + 0, Acc(-fx));
        atomicAdd(f + 1, Acc(-fy));
        atomicAdd(f + 2, Acc(-fz));
      }
    }
    work += OVF ? nwarps_total : gridDim.x;
    __syncwarp();                      // staging is rewritten by the next tile
  }

  if constexpr (kMerge) {
    // the atoms over 4 (left above), by the packed tier's own scan
    if (a.ovf_scan) packed_work<R, Acc, SPEC, DET, true, FOREIGN, VIR>(a, s_tier, e_acc, w_acc);
  }

  // ---- block reduction of energy + virial, fixed order ----
  double red[7] = {double(e_acc), double(w_acc[0]), double(w_acc[1]), double(w_acc[2]),
                   double(w_acc[3]), double(w_acc[4]), double(w_acc[5])};
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) red[q] += __shfl_down_sync(kFull, red[q], o);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 7; ++q) s_red[tid / 32][q] = red[q];
  __syncthreads();
  if (tid < kRedWidth) {
    double s = 0;
    if (tid < 7)
      for (int w = 0; w < kBlock / 32; ++w) s += s_red[w][tid];
    a.partials[std::size_t(a.partial_base + blockIdx.x) * kRedWidth + tid] = s;
  }
}

// Sum of the block partials in a fixed order.  The partials are read as one
// flat array: thread t always holds quantity q = t % 8 (1024 % kRedWidth == 0),
// so every warp load is 256 contiguous bytes; lanes of equal q meet in two
// shuffles, the 32 warps' sums in shared memory — the reduction sits on every
// step's critical path, and at 32k atoms it was a quarter of the step.
static_assert(kRedWidth == 8, "k_reduce maps one quantity per thread mod 8");
__global__ void __launch_bounds__(1024) k_reduce(const double* __restrict__ partials, int nblocks,
                                                double* __restrict__ out, int* __restrict__ fold,
                                                int* __restrict__ near_flags,
                                                int* __restrict__ over4) {
  __shared__ double s[32][kRedWidth];
  griddep_wait();
  const int t = threadIdx.x;
  // speculative MD: this step's "moved" flag joins the segment's (one block,
  // after every launch that reads both)
  if (fold && t == 0 && fold[kFlagMoved]) fold[kFlagMovedAny] = 1;
  // this evaluation's filter refreshed the near lists: the displacement
  // maximum restarts from their new reference (every reader has run)
  if (over4 && t == 0) *over4 = 0;   // the tier has read it
  if (near_flags && t == 0 && near_flags[kFlagNearRefresh]) {
    near_flags[kFlagNearRefresh] = 0;
    near_flags[10] = 0;
    ++near_flags[kFlagNearRefreshCount];
  }
  const int total = nblocks * kRedWidth;
  double acc = 0;
  for (int e = t; e < total; e += 1024) acc += partials[e];
  acc += __shfl_xor_sync(kFull, acc, 8);
  acc += __shfl_xor_sync(kFull, acc, 16);
  if ((t & 31) < kRedWidth) s[t >> 5][t & 31] = acc;
  __syncthreads();
  if (t < 7) {
    double v = 0;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) v += s[w][t];
    out[t] = v;
  }
}

// Deterministic mode: energy + virial of the atoms the tier launches took,
// summed in atom order (block b owns a fixed contiguous chunk) into the
// block partials.  "Queued" repeats the main kernel's rule: an owned,
// non-ghost slot with more short entries than the main width.
__global__ void __launch_bounds__(kBlock) k_queued_ev(const double* __restrict__ atom_ev,
                                                      const int* __restrict__ cnt,
                                                      const int* __restrict__ perm, int n_owned,
                                                      int center_limit, int g,
                                                      const int* __restrict__ queued,
                                                      double* __restrict__ partials) {
  __shared__ double s[kBlock][7];
  const int t = threadIdx.x;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  if (!queued || *queued > 0) {   // (no count: a scanning tier took them)
    const int chunk = (n_owned + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * chunk, hi = min(n_owned, lo + chunk);
    for (int i = lo + t; i < hi; i += kBlock)
      if (cnt[i] > g && (perm ? perm[i] : i) < center_limit)
        for (int q = 0; q < 7; ++q) acc[q] += atom_ev[8 * std::size_t(i) + q];
  }
  for (int q = 0; q < 7; ++q) s[t][q] = acc[q];
  __syncthreads();
  for (int w = kBlock / 2; w > 0; w >>= 1) {
    if (t < w)
      for (int q = 0; q < 7; ++q) s[t][q] += s[t + w][q];
    __syncthreads();
  }
  if (t < kRedWidth) partials[std::size_t(blockIdx.x) * kRedWidth + t] = t < 7 ? s[0][t] : 0.0;
}

// Deterministic scatter: F_a = F_self(a) + sum over a's short neighbours b of
// the slot b wrote for a (lists are symmetric).
template <typename Acc>
__global__ void __launch_bounds__(kBlock) k_gather(int n, int npad, const int* __restrict__ nbr,
                                                   const int* __restrict__ cnt,
                                                   const Acc* __restrict__ sx,
                                                   const Acc* __restrict__ sy,
                                                   const Acc* __restrict__ sz,
                                                   const Acc* __restrict__ fself,
                                                   double* __restrict__ out) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  Acc fx = fself[3 * std::size_t(a)], fy = fself[3 * std::size_t(a) + 1],
      fz = fself[3 * std::size_t(a) + 2];
  const int m = cnt[a];
  for (int s = 0; s < m; ++s) {
    const int b = nbr[ell_at(s, a, npad)];
    TSF_DCHECK(b >= 0 && b < n && b != a, "k_gather list entry");
    const int mb = cnt[b];
    // a's position in b's list, four entries per 128-bit load (one ELL4
    // block; the scalar search took ~2.5 dependent loads per neighbour)
    int t = -1;
    for (int t0 = 0; t0 < mb && t < 0; t0 += 4) {
      const int4 e = *reinterpret_cast<const int4*>(nbr + ell_at(t0, b, npad));
      const int k = e.x == a ? 0 : e.y == a ? 1 : e.z == a ? 2 : e.w == a ? 3 : 4;
      if (k < 4 && t0 + k < mb) t = t0 + k;
    }
    if (t >= 0) {
      const std::size_t q = std::size_t(t) * npad + b;
      fx += sx[q];
      fy += sy[q];
      fz += sz[q];
    }
  }
  out[3 * std::size_t(a)] = double(fx);
  out[3 * std::size_t(a) + 1] = double(fy);
  out[3 * std::size_t(a) + 2] = double(fz);
}

__global__ void k_to_double(const float* __restrict__ in, double* __restrict__ out,
                            std::size_t m) {
  const std::size_t q = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < m) out[q] = double(in[q]);
}

template <typename R>
Row<R> make_row(const Entry& e) {
  Row<R> r{};
  const double pi = 3.14159265358979323846;
  r.a = R(e.big_a);
  r.b = R(e.big_b);
  r.lam1 = R(e.lambda1);
  r.lam2 = R(e.lambda2);
  r.lam3 = R(e.lambda3);
  r.m3 = R(e.m == 3 ? 1 : 0);
  r.beta = R(e.beta);
  r.eta = R(e.eta);
  r.nhie = R(e.eta > 0 ? -0.5 / e.eta : 0.0);   // eta = 0 only on unused cross rows
  r.big_r = R(e.big_r);
  r.inv2d = R(0.5 / e.big_d);
  r.rmd = R(e.big_r - e.big_d);
  r.rpd = R(e.big_r + e.big_d);
  r.nqd = R(-pi / 4 / e.big_d);
  const double c2 = e.c * e.c, d2 = e.d * e.d;
  // bond-order series path (tsf_math.cuh): u < 2^-12 and |u / (2 eta)| < 2^-8
  r.lnu_fast = R(e.eta > 0 ? std::min(std::log(0x1p-12), std::log(0x1p-8 * 2.0 * e.eta))
                           : -1e300);
  {
    // every exp argument of a counted pair / triplet is bounded by the cutoff
    // (r, r_ij, r_ik <= R + D): EXPNB's branch-free exp needs |x| < 708
    const double cut = e.big_r + e.big_d;
    const double tri = e.m == 3 ? std::pow(std::fabs(e.lambda3) * cut, 3.0)
                                : std::fabs(e.lambda3) * cut;
    r.exp_ok = R(tri < 700.0 && std::fabs(e.lambda1) * cut < 700.0 &&
                         std::fabs(e.lambda2) * cut < 700.0 ? 1 : 0);
  }
  {
    const double l2e = std::is_same<R, double>::value ? 1.0 : 1.4426950408889634;   // float: base 2
    const double l3 = e.lambda3;
    r.e1 = R(-e.lambda1 * l2e);
    r.e2 = R(-e.lambda2 * l2e);
    r.tc = R((e.m == 3 ? l3 * l3 * l3 : l3) * l2e);
    r.td = R(e.m == 3 ? 3.0 * l3 * l3 * l3 : l3);
    if (!std::is_same<R, double>::value) r.lnu_fast = R(double(r.lnu_fast) * l2e);   // log2 u
  }
  r.gamma = R(e.gamma);
  r.gcd2 = R(e.gamma * c2 / d2);
  r.gc2 = R(e.gamma * c2);
  r.d2 = R(d2);
  r.h = R(e.h);
  return r;
}

int ceil_div(std::int64_t a, int b) { return int((a + b - 1) / b); }

// Persistent grid: resident blocks per SM x SM count, capped by the tile count.
template <typename K>
int persistent_blocks(K kernel, int tiles) {
  static std::map<const void*, int> cache;   // contexts may live on several threads
  static std::mutex mu;
  const void* key = reinterpret_cast<const void*>(kernel);
  int per_sm;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it == cache.end()) {
      TSF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, 0));
      per_sm = std::max(1, per_sm);
      cache[key] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  int dev = 0, sms = 148;
  TSF_CUDA(cudaGetDevice(&dev));
  TSF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return std::max(1, std::min(tiles, per_sm * sms));
}

constexpr int kOverflowBlocks = 4 * 148;   // per tier launch; idle tiers exit at once

template <typename R, typename Acc, int G, int SPEC, bool DET, bool FOREIGN, bool VIR = true>
int launch_main(Ctx& c, ForceArgs<R> a, bool merge = false) {
  const int tiles = std::max(1, ceil_div(a.n_owned - a.slot_base, kBlock / G));
  auto kern = k_force<R, Acc, G, SPEC, DET, false, FOREIGN, VIR>;
  if constexpr (kMergeTier<R, G, SPEC, false>)
    if (merge) kern = k_force<R, Acc, G, SPEC, DET, false, FOREIGN, VIR, false, true>;
  // one species, FP64, G = 4: the branch-free exp when the row bounds every
  // argument (Si: (lambda3 R)^3 = 76) — TSF_EXPNB=1 turns it on
  if constexpr (SPEC == kSingle && G == 4 && std::is_same<R, double>::value) {
    // measured slower (+6% on si2m: the interleaved chains spill): A/B only
    const char* e = std::getenv("TSF_EXPNB");
    if (a.row0.exp_ok != R(0) && e && e[0] == '1')
      kern = merge ? k_force<R, Acc, G, SPEC, DET, false, FOREIGN, VIR, true, true>
                   : k_force<R, Acc, G, SPEC, DET, false, FOREIGN, VIR, true>;
  }
  const int blocks = persistent_blocks(kern, tiles);
  c.mark(2);
  launch_pdl(kern, blocks, kBlock, c.stream, a);
  c.mark(3);
  ++c.launches;
  return blocks;
}

// read per eager evaluation (graph replays do not come here), so tests can switch them
int packed_mode() {
  const char* e = std::getenv("TSF_PACKED");
  return e ? std::atoi(e) : 1;
}

int packed_over4_pct() {
  const char* e = std::getenv("TSF_PACKED_OVER4");
  return e ? std::atoi(e) : 10;
}

template <typename R, typename Acc, int SPEC, bool DET, bool FOREIGN, bool VIR>
int launch_main_packed(Ctx& c, ForceArgs<R> a) {
  const int chunks = std::max(1, ceil_div(a.n_owned - a.slot_base, 32));
  auto kern = k_force_packed<R, Acc, SPEC, DET, false, FOREIGN, VIR>;
  const int blocks = persistent_blocks(kern, ceil_div(chunks, kBlock / 32));
  c.mark(2);
  launch_pdl(kern, blocks, kBlock, c.stream, a);
  c.mark(3);
  ++c.launches;
  return blocks;
}

// VIR = false: no caller reads the virial (the MD loop, evaluate_forces
// without one, TSF_NO_VIRIAL) — the G = 4 and packed launches then never form
// it (6 FP64 products per slot, 12 accumulator registers); the other widths,
// rare, form it anyway.
template <typename R, typename Acc, int SPEC, bool DET, bool FOREIGN, bool VIR>
void run_force_t(Ctx& c, ForceArgs<R> a) {
  // Group width from the short-count distribution of the last list build
  // (atoms over 4 / over 8); atoms over the width — or that outgrow it
  // between rebuilds — take the G=16 / G=32 tier launches.  Measured per-atom
  // costs (B200, f64; profiles/r01): main G=4 0.26 ns, G=8 0.69 ns, G=16
  // 1.7 ns (no register cache of d zeta/d x_k above 8), a queued atom
  // 2.3-2.6 ns when first measured (about 1 ns with today's tier launches),
  // so G=4 wins below ~15% over-4 atoms (float; ~50% in f64) and G=8 below
  // ~35% over-8 (3C-SiC 256k: 45% / 8% -> G=8 float, G=4 f64; liquid Si
  // 512k -> G=8, 2.0x over G=16).
  const ListState& s = c.short_list;
  const int mx = std::max(1, s.max_count);
  const std::int64_t n = std::max<std::int64_t>(c.n, 1);
  // FP64's G = 8 (rolled, cache in local memory) costs more next to its G = 4
  // than float's unrolled G = 8 does: 3C-SiC 256k (45% over 4) runs 3% faster
  // at G = 4 + tier launches in f64 and 25% slower in float (tools/ab.py)
  const int over4_pct = std::is_same<R, double>::value ? 50 : 15;
  int g = (mx <= 4 || s.over4 * 100 <= over4_pct * n) ? 4
          : (mx <= 8 || s.over8 * 100 <= 35 * n) ? 8
          : 16;
  // TSF_GROUP_WIDTH=4|8|16|32 pins the width (tuning and the tier tests)
  const char* pin = std::getenv("TSF_GROUP_WIDTH");
  const int pinned = pin ? std::atoi(pin) : 0;
  if (pinned == 4 || pinned == 8 || pinned == 16 || pinned == 32) g = pinned;
  // Packed lane groups (tsf_force_packed.cuh): the tier chain becomes ONE
  // packed launch over the queue, and an irregular system (over the
  // TSF_PACKED_OVER4 percent of atoms over 4) runs packed from the start.
  // TSF_PACKED=0 restores the G-tier chain, 2 forces the packed main launch.
  const int pmode = packed_mode();
  const bool packed_main =
      !(pinned == 4 || pinned == 8 || pinned == 16 || pinned == 32) && pmode >= 1 &&
      (pmode == 2 || (mx > 4 && s.over4 * 100 > packed_over4_pct() * n));
  if (packed_main) g = 32;
  c.main_packed = packed_main;
  // Tier chain: atoms over the main width are queued for G = 8 (when the
  // last rebuild saw counts over 4), then G = 16 (counts over 8), then
  // G = 32, which takes whatever is left — including atoms that outgrew the
  // width since the rebuild (an idle tier launch still costs ~3 us).  At
  // 1600 K a few % of Si atoms gain a 5th neighbour: the G = 8 tier takes
  // them at 4 atoms per warp instead of G = 16's 2.  Queue q holds
  // [q n, (q + 1) n) of c.overflow; its count is flags[1 + q] (zeroed with
  // the error bits per evaluation).
  int* qbuf = c.overflow.get();
  int cur = 0;                              // queue the main launch fills
  a.ovf_out = g < 32 ? qbuf : nullptr;
  a.ovf_out_count = a.flags + 1;
  // packed tier (default): the main launch queues nothing, the tier scans
  a.ovf_scan = pmode >= 1 && g < 32 ? 1 : 0;
  const char* merge_env = std::getenv("TSF_MERGE_TIER");   // =0: separate tier launch (A/B)
  const bool merge_tier = kMergeTier<R, 4, SPEC, false> && g == 4 && a.ovf_scan &&
                          c.n <= kMergeMaxAtoms && !(merge_env && merge_env[0] == '0');
  a.scan_g = g;
  a.over4 = c.filter_marks_over4 && c.phase_first ? a.flags + kFlagOver4 : nullptr;
  // two-phase evaluation: the partials of the first phase's main launch
  // precede this one's; tiers and the reduction run with the last phase
  a.partial_base = c.phase_blocks;
  int nb = c.phase_blocks;
  if (packed_main) {
    a.ovf_out = nullptr;
    nb += launch_main_packed<R, Acc, SPEC, DET, FOREIGN, VIR>(c, a);
  } else {
    switch (g) {
      case 4: nb += launch_main<R, Acc, 4, SPEC, DET, FOREIGN, VIR>(c, a, merge_tier); break;
      case 8: nb += launch_main<R, Acc, 8, SPEC, DET, FOREIGN>(c, a); break;
      case 16: nb += launch_main<R, Acc, 16, SPEC, DET, FOREIGN>(c, a); break;
      default: nb += launch_main<R, Acc, 32, SPEC, DET, FOREIGN>(c, a); break;
    }
  }
  c.phase_blocks = nb;
  if (!c.phase_last) return;
  c.phase_blocks = 0;
  auto tier = [&](auto kernel, int blocks, bool last) {
    a.partial_base = nb;
    a.ovf_in = qbuf + std::size_t(cur) * c.n;
    a.ovf_in_count = a.flags + 1 + cur;
    a.ovf_out = last ? nullptr : qbuf + std::size_t(cur + 1) * c.n;
    a.ovf_out_count = a.flags + 2 + cur;
    launch_pdl(kernel, blocks, kBlock, c.stream, a);
    nb += blocks;
    ++c.launches;
    if (!last) ++cur;
  };
  if (pmode >= 1) {
    // one packed launch takes every queued atom, whatever its count.  Full
    // occupancy whatever the last rebuild saw: the queue grows between
    // rebuilds (Si at 1600 K: 0 -> 180k atoms with a 5th neighbour within 60
    // fs of a rebuild), and a quarter grid left 4 warps per SM to serialise
    // it (0.2 ms); an empty queue exits at once either way
    // (merged into the FP64 G = 4 main launches: each phase's main launch
    // takes the atoms over 4 of its own slot range)
    const bool merged = merge_tier;
    if (g < 32 && !merged) {
      a.slot_base = 0;                      // every phase's slots
      tier(k_force_packed<R, Acc, SPEC, DET, true, FOREIGN, VIR>, kOverflowBlocks, true);
    }
  } else {
    if (g < 8 && mx > 4) tier(k_force<R, Acc, 8, SPEC, DET, true, FOREIGN>, kOverflowBlocks, false);
    if (g < 16 && mx > 8) tier(k_force<R, Acc, 16, SPEC, DET, true, FOREIGN>, kOverflowBlocks, false);
    if (g < 32)
      tier(k_force<R, Acc, 32, SPEC, DET, true, FOREIGN>,
           mx > 16 ? kOverflowBlocks : kOverflowBlocks / 4, true);
  }
  if (g < 32) {
    if (DET) {
      k_queued_ev<<<kOverflowBlocks, kBlock, 0, c.stream>>>(
          a.atom_ev, a.cnt, a.perm, a.n_owned, a.energy_limit, g,
          a.ovf_scan ? static_cast<const int*>(nullptr) : a.flags + 1,
          a.partials + std::size_t(nb) * kRedWidth);
      nb += kOverflowBlocks;
      ++c.launches;
    }
  }
  launch_pdl(k_reduce, 1, 1024, c.stream, static_cast<const double*>(c.partials.get()), nb,
             c.result.get(), c.speculative ? c.flags.get() : static_cast<int*>(nullptr),
             c.near_ok ? c.flags.get() : static_cast<int*>(nullptr), c.flags.get() + kFlagOver4);
  ++c.launches;
}

template <typename R, typename Acc, int SPEC, bool DET>
void run_force(Ctx& c, const ForceArgs<R>& a, bool vir) {
  if (a.energy_limit < a.center_limit) run_force_t<R, Acc, SPEC, DET, true, true>(c, a);
  else if (vir) run_force_t<R, Acc, SPEC, DET, false, true>(c, a);
  else run_force_t<R, Acc, SPEC, DET, false, false>(c, a);
}

template <typename R, typename Acc, bool DET>
void dispatch_spec(Ctx& c, const ForceArgs<R>& a, bool vir) {
  // kSingle compiles the cubic triplet exponent in (every single-species
  // table in use has m = 3) and drops the triplet masks at G = 4, which needs
  // every exponential argument within a cutoff bounded (Row::exp_ok); other
  // single-species tables take kHoist
  if (c.params.species_count() == 1 && c.params.entry(0, 0, 0).m == 3 && a.row0.exp_ok != R(0))
    run_force<R, Acc, kSingle, DET>(c, a, vir);
  else if (c.hoist_ramp) run_force<R, Acc, kHoist, DET>(c, a, vir);
  else run_force<R, Acc, kGeneric, DET>(c, a, vir);
}

template <typename R, typename Acc>
void compute_t(Ctx& c, std::uint32_t flags) {
  const bool det = (flags & 0x1u) != 0;
  const bool vir = !(flags & kFlagNoVirial);
  const std::size_t n = std::size_t(c.n);
  const int npad = c.npad;
  const int cap = c.short_list.cap;

  ForceArgs<R> a{};
  a.row0 = make_row<R>(c.params.entry(0, 0, 0));
  a.cut0 = c.params.entry(0, 0, 0).cutoff() * c.params.entry(0, 0, 0).cutoff();
  a.pos = c.pos.get();
  a.slot_base = c.phase_lo;
  a.n_owned = c.phase_hi;
  a.n_all = int(c.n);
  a.perm = c.sorted ? c.perm.get() : nullptr;
  a.center_limit = int(c.n_owned >= 0 ? std::min<std::int64_t>(c.n_owned, c.n) : c.n);
  a.energy_limit = c.n_energy >= 0 ? int(std::min<std::int64_t>(c.n_energy, a.center_limit))
                                   : a.center_limit;
  // the list build put every centre below center_slots (non-centre ghosts
  // behind them): atomic mode stops the launches there.  Deterministic mode
  // keeps the ghost slots — the force launch zeroes their self terms there.
  if (!det && c.center_slots >= 0 && c.center_slots == a.center_limit)
    a.n_owned = std::min(a.n_owned, int(c.center_slots));
  a.npad = npad;
  a.box = c.box;
  a.nbr = c.short_list.nbr.get();
  a.cnt = c.short_list.cnt.get();
  a.rows = std::is_same<R, double>::value ? static_cast<const void*>(c.rows_f64.get())
                                          : static_cast<const void*>(c.rows_f32.get());
  a.cutsq = c.cutsq.get();
  a.ns = c.params.species_count();
  a.flags = c.flags.get();
  a.skip = c.speculative ? c.flags.get() + kFlagMoved : nullptr;
  c.overflow.reserve(std::max<std::size_t>(3 * n, 1));
  {
    // one partial row per block: two phases' main launches (each at most
    // resident-blocks-per-SM x SMs, persistent_blocks), up to three tier
    // launches plus k_queued_ev of kOverflowBlocks each
    int dev = 0, sms = 148;
    TSF_CUDA(cudaGetDevice(&dev));
    TSF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const std::size_t max_main = std::size_t(sms) * (2048 / kBlock);
    c.partials.reserve((2 * max_main + 4 * kOverflowBlocks + 8) * kRedWidth);
  }
  a.partials = c.partials.get();
  if (c.phase_first && !(flags & kFlagFlagsZeroed))
    TSF_CUDA(cudaMemsetAsync(c.flags.get(), 0, 4 * sizeof(int), c.stream));

  constexpr bool kF32 = std::is_same<Acc, float>::value;
  if (det) {
    const std::size_t words = std::size_t(cap) * npad * sizeof(Acc) / sizeof(double) + 1;
    c.px.reserve(words);
    c.py.reserve(words);
    c.pz.reserve(words);
    c.fself.reserve(3 * n * sizeof(Acc) / sizeof(double) + 1);
    a.slot_x = c.px.get();
    a.slot_y = c.py.get();
    a.slot_z = c.pz.get();
    a.fself = c.fself.get();
    c.atom_ev.reserve(8 * n + 1);
    a.atom_ev = c.atom_ev.get();
    dispatch_spec<R, Acc, true>(c, a, vir);
    if (n > 0 && c.phase_last) {
      k_gather<Acc><<<ceil_div(n, kBlock), kBlock, 0, c.stream>>>(
          int(n), npad, a.nbr, a.cnt, static_cast<const Acc*>(a.slot_x),
          static_cast<const Acc*>(a.slot_y), static_cast<const Acc*>(a.slot_z),
          static_cast<const Acc*>(a.fself), c.forces.get());
      ++c.launches;
    }
  } else {
    Acc* target;
    if (kF32) {
      c.fself.reserve(3 * n * sizeof(float) / sizeof(double) + 1);
      target = reinterpret_cast<Acc*>(c.fself.get());
    } else {
      target = reinterpret_cast<Acc*>(c.forces.get());
    }
    if (!(flags & kFlagForcesZeroed) && c.phase_first)
      TSF_CUDA(cudaMemsetAsync(target, 0, 3 * n * sizeof(Acc), c.stream));
    a.forces = target;
    dispatch_spec<R, Acc, false>(c, a, vir);
    if (kF32 && n > 0 && c.phase_last) {
      k_to_double<<<ceil_div(3 * n, 256), 256, 0, c.stream>>>(
          reinterpret_cast<const float*>(target), c.forces.get(), 3 * n);
      ++c.launches;
    }
  }
}

}  // namespace

}  // namespace tsf
