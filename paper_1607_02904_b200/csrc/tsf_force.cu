// Tersoff energy / forces / virial on the short list — the hot path.
//
// Replaces evaluate_forces' kernels (proj/include/tmd/kernels.hpp:175-494,
// proj/src/potential_ref.cpp:75-134; paper Alg. 2/3 and Fig. 3).
//
// Mapping ("lane group per atom", the GPU form of the paper's scheme (a)):
//   * a group of G lanes (G = 4, 8, 16 or 32; G >= the atom's short count)
//     owns central atom i; lane l holds short neighbour j_l, its FP64
//     displacement, r, 1/r, unit vector and — when the ramp depends on (i,k)
//     only — f_C(r) and f_C'(r), staged in shared memory;
//   * zeta pass: at rotation t lane l pairs with k = slot (l + t) mod n_i
//     (t = 1..n_i-1 visits every k != j once, no lane idles on k == j); the
//     triplet's d zeta/d x_j is accumulated in registers and d zeta/d x_k is
//     cached in registers (Alg. 3's derivative cache, k_max = G - 1);
//   * pair block: V, dV/dr, dV/dzeta with the log-space bond order;
//   * scatter pass: at rotation t lane l hands its cached d zeta/d x_k times
//     dV/dzeta_j to lane (l + t) mod n_i with one shuffle — the transposed
//     reduction — so every lane ends with P_l, the total force atom i's terms
//     put on neighbour j_l, and F_i = -sum_l P_l (translation invariance);
//   * atomic mode: one atomicAdd per neighbour slot and component, one for i;
//     deterministic mode: P_l goes to a slot buffer and tsf_gather sums every
//     atom's incoming slots in list order — bitwise reproducible;
//   * energy and virial (W_ab = sum_l d_a P_b) are reduced per block into a
//     partials array and summed in fixed order: deterministic in both modes.
// Atoms whose short count exceeds G are queued and processed by the same code
// with G = 32 (one warp per atom) in a second, tiny launch.
#include <algorithm>
#include <cmath>
#include <vector>

#include "tsf_context.hpp"

namespace tsf {

namespace {

struct ForceArgs {
  const double4* pos;
  int n_owned;
  int npad;
  Box box;
  const int* nbr;
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
  int* overflow;       // queued atom ids
  int* flags;          // [0] error, [1] overflow count
};

constexpr unsigned kFull = 0xffffffffu;

template <typename R>
struct Nbr {
  R ux, uy, uz, r, ir;
};

template <typename R>
struct Grad {
  R z, jx, jy, jz, kx, ky, kz;
};

// One (i, j, k) triplet: zeta term and its j and k gradients
// (potential.hpp:132-198; the i gradient is never formed: F_i = -sum P).
template <typename R, bool HOIST>
__device__ __forceinline__ Grad<R> triplet(const Nbr<R>& j, const Nbr<R>& k, R fck, R dfck,
                                           const Row<R>& p) {
  Grad<R> o;
  R cs = j.ux * k.ux + j.uy * k.uy + j.uz * k.uz;
  cs = fmin(R(1), fmax(R(-1), cs));
  if (!HOIST) cutoff_ramp(k.r, p, fck, dfck);
  const R t = p.h - cs;
  const R den = p.d2 + t * t;
  const R iden = R(1) / den;
  const R g = p.gamma + p.gcd2 * (t * t) * iden;
  const R dg = R(-2) * p.gc2 * t * iden * iden;
  const R arg = p.lam3 * (j.r - k.r);
  const bool cubic = p.m3 != R(0);
  const R ex = Fn<R>::exp_(cubic ? arg * arg * arg : arg);
  const R dex = ex * p.lam3 * (cubic ? R(3) * arg * arg : R(1));
  const R fg = fck * g;
  o.z = fg * ex;
  const R fgd = fck * dg * ex;
  const R fge = fg * dex;
  const R cge = dfck * g * ex;
  // d cos / d x_j and d cos / d x_k
  const R gjx = (k.ux - j.ux * cs) * j.ir, gjy = (k.uy - j.uy * cs) * j.ir,
          gjz = (k.uz - j.uz * cs) * j.ir;
  const R gkx = (j.ux - k.ux * cs) * k.ir, gky = (j.uy - k.uy * cs) * k.ir,
          gkz = (j.uz - k.uz * cs) * k.ir;
  o.jx = gjx * fgd + j.ux * fge;
  o.jy = gjy * fgd + j.uy * fge;
  o.jz = gjz * fgd + j.uz * fge;
  const R ck = cge - fge;
  o.kx = k.ux * ck + gkx * fgd;
  o.ky = k.uy * ck + gky * fgd;
  o.kz = k.uz * ck + gkz * fgd;
  return o;
}

template <typename T>
__device__ __forceinline__ void atomic_add(T* p, T v) {
  atomicAdd(p, v);
}

template <typename R, typename Acc, int G, bool HOIST, bool DET, bool OVF>
__global__ void __launch_bounds__(kBlock) k_force(ForceArgs a) {
  constexpr bool kCache = G <= 8;     // register cache of d zeta / d x_k
  __shared__ Row<R> srow[kMaxSpecies * kMaxSpecies * kMaxSpecies];
  __shared__ double scut[kMaxSpecies * kMaxSpecies * kMaxSpecies];
  __shared__ R s_ux[kBlock], s_uy[kBlock], s_uz[kBlock], s_r[kBlock], s_ir[kBlock];
  __shared__ R s_fc[kBlock], s_dfc[kBlock];
  __shared__ double s_r2[kBlock];
  __shared__ int s_sp[kBlock];
  __shared__ double s_red[kBlock / 32][kRedWidth];

  const int ns = a.ns;
  const int nrows = ns * ns * ns;
  const Row<R>* rows = static_cast<const Row<R>*>(a.rows);
  for (int q = threadIdx.x; q < nrows; q += blockDim.x) {
    srow[q] = rows[q];
    scut[q] = a.cutsq[q];
  }
  __syncthreads();

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int gl = tid & (G - 1);
  const int gbase = tid - gl;          // block-local thread id of slot 0
  const int wbase = lane - gl;         // warp lane of slot 0

  Acc e_acc = 0;
  Acc w_acc[6] = {0, 0, 0, 0, 0, 0};

  const int nwarps_total = gridDim.x * (kBlock / 32);
  const int warp_global = blockIdx.x * (kBlock / 32) + tid / 32;
  int work = OVF ? warp_global : 0;
  const int n_ovf = OVF ? a.flags[1] : 0;

  while (true) {
    int i;
    bool active;
    if (OVF) {
      if (work >= n_ovf) break;        // warp-uniform
      i = a.overflow[work];
      active = true;
    } else {
      i = blockIdx.x * (kBlock / G) + tid / G;
      active = i < a.n_owned;
    }

    int n_i = active ? a.cnt[i] : 0;
    if (!OVF && n_i > G) {
      if (gl == 0) a.overflow[atomicAdd(a.flags + 1, 1)] = i;
      n_i = 0;
      active = false;
    }
    if (OVF && n_i > G) {
      if (gl == 0) atomicOr(a.flags, kErrShortOverflow);
      n_i = 0;
      active = false;
    }
    const bool slot = gl < n_i;
    const double4 pi = a.pos[active ? i : 0];
    const int si = species_of(pi);
    const int j = slot ? a.nbr[std::size_t(gl) * a.npad + i] : (active ? i : 0);
    const double4 pj = a.pos[j];
    const int sj = species_of(pj);
    double dx = 0, dy = 0, dz = 0;
    if (slot) displacement(pi, pj, a.box, dx, dy, dz);
    const double r2 = slot ? norm_sq_exact(dx, dy, dz) : 1.0;
    const int row_jj = (si * ns + sj) * ns + sj;
    const bool pair_ok = slot && r2 <= scut[row_jj];
    const Row<R>& pjj = srow[row_jj];

    Nbr<R> me;
    me.r = Fn<R>::sqrt_(R(r2));
    me.ir = R(1) / me.r;
    me.ux = R(dx) * me.ir;
    me.uy = R(dy) * me.ir;
    me.uz = R(dz) * me.ir;
    R fc, dfc;
    cutoff_ramp(me.r, pjj, fc, dfc);

    s_ux[tid] = me.ux;
    s_uy[tid] = me.uy;
    s_uz[tid] = me.uz;
    s_r[tid] = me.r;
    s_ir[tid] = me.ir;
    s_fc[tid] = fc;
    s_dfc[tid] = dfc;
    s_r2[tid] = r2;
    s_sp[tid] = slot ? sj : -1;
    __syncwarp();

    const int tmax = __reduce_max_sync(kFull, n_i);
    const int rowbase = (si * ns + sj) * ns;

    // ---- zeta pass ----
    R zeta = 0, gjx = 0, gjy = 0, gjz = 0;
    R ckx[kCache ? G : 1], cky[kCache ? G : 1], ckz[kCache ? G : 1];
#pragma unroll
    for (int t = 1; t < G; ++t) {
      if (t < tmax) {
        int m = gl + t;
        if (m >= n_i) m -= n_i;
        const int src = gbase + (t < n_i ? m : gl);
        const int sk = s_sp[src];
        bool ok = pair_ok && t < n_i && sk >= 0;
        const int row = rowbase + (sk >= 0 ? sk : 0);
        ok = ok && s_r2[src] <= scut[row];
        Nbr<R> k{s_ux[src], s_uy[src], s_uz[src], s_r[src], s_ir[src]};
        const Grad<R> tr = triplet<R, HOIST>(me, k, s_fc[src], s_dfc[src], srow[row]);
        if (ok) {
          zeta += tr.z;
          gjx += tr.jx;
          gjy += tr.jy;
          gjz += tr.jz;
        }
        if constexpr (kCache) {
          ckx[t] = ok ? tr.kx : R(0);
          cky[t] = ok ? tr.ky : R(0);
          ckz[t] = ok ? tr.kz : R(0);
        }
      }
    }

    // ---- pair block (potential.hpp:204-222) ----
    R dvdr = 0, dvdz = 0, v = 0;
    if (pair_ok) {
      const R fr = pjj.a * Fn<R>::exp_(-pjj.lam1 * me.r);
      const R dfr = -pjj.lam1 * fr;
      const R fa = -(pjj.b * Fn<R>::exp_(-pjj.lam2 * me.r));
      const R dfa = -pjj.lam2 * fa;
      R b, db;
      bond_order(zeta, pjj, b, db);
      const R rep = fr + b * fa;
      v = R(0.5) * fc * rep;
      dvdr = R(0.5) * (dfc * rep + fc * (dfr + b * dfa));
      dvdz = R(0.5) * fc * fa * db;
      if (!isfinite(v) || !isfinite(dvdr) || !isfinite(dvdz)) atomicOr(a.flags, kErrNonFinite);
    }
    R px = -(me.ux * dvdr) - gjx * dvdz;
    R py = -(me.uy * dvdr) - gjy * dvdz;
    R pz = -(me.uz * dvdr) - gjz * dvdz;

    // ---- scatter pass: lane (l + t) mod n receives lane l's k-gradient ----
#pragma unroll
    for (int t = 1; t < G; ++t) {
      if (t < tmax) {
        R sx, sy, sz;
        if constexpr (kCache) {
          sx = ckx[t] * dvdz;
          sy = cky[t] * dvdz;
          sz = ckz[t] * dvdz;
        } else {
          int m = gl + t;
          if (m >= n_i) m -= n_i;
          const int src = gbase + (t < n_i ? m : gl);
          const int sk = s_sp[src];
          bool ok = pair_ok && t < n_i && sk >= 0;
          const int row = rowbase + (sk >= 0 ? sk : 0);
          ok = ok && s_r2[src] <= scut[row];
          Nbr<R> k{s_ux[src], s_uy[src], s_uz[src], s_r[src], s_ir[src]};
          const Grad<R> tr = triplet<R, HOIST>(me, k, s_fc[src], s_dfc[src], srow[row]);
          sx = ok ? tr.kx * dvdz : R(0);
          sy = ok ? tr.ky * dvdz : R(0);
          sz = ok ? tr.kz * dvdz : R(0);
        }
        int s = gl - t;
        if (s < 0) s += n_i;
        const int from = wbase + ((t < n_i && s >= 0) ? s : gl);
        const R rx = __shfl_sync(kFull, sx, from);
        const R ry = __shfl_sync(kFull, sy, from);
        const R rz = __shfl_sync(kFull, sz, from);
        if (slot && t < n_i) {
          px -= rx;
          py -= ry;
          pz -= rz;
        }
      }
    }
    if (!slot) px = py = pz = 0;

    // F_i = -sum over the group's slots
    R fx = px, fy = py, fz = pz;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      fx += __shfl_xor_sync(kFull, fx, o);
      fy += __shfl_xor_sync(kFull, fy, o);
      fz += __shfl_xor_sync(kFull, fz, o);
    }

    if (slot) {
      e_acc += Acc(v);
      const R rx = R(dx), ry = R(dy), rz = R(dz);
      w_acc[0] += Acc(rx * px);
      w_acc[1] += Acc(ry * py);
      w_acc[2] += Acc(rz * pz);
      w_acc[3] += Acc(rx * py);
      w_acc[4] += Acc(rx * pz);
      w_acc[5] += Acc(ry * pz);
      if (DET) {
        const std::size_t q = std::size_t(gl) * a.npad + i;
        static_cast<Acc*>(a.slot_x)[q] = Acc(px);
        static_cast<Acc*>(a.slot_y)[q] = Acc(py);
        static_cast<Acc*>(a.slot_z)[q] = Acc(pz);
      } else {
        Acc* f = static_cast<Acc*>(a.forces) + 3 * std::size_t(j);
        atomic_add(f + 0, Acc(px));
        atomic_add(f + 1, Acc(py));
        atomic_add(f + 2, Acc(pz));
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
        atomic_add(f + 0, Acc(-fx));
        atomic_add(f + 1, Acc(-fy));
        atomic_add(f + 2, Acc(-fz));
      }
    }
    if (!OVF) break;
    work += nwarps_total;
    __syncwarp();
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

// Sum of the block partials in a fixed order: pairwise over a strided split.
__global__ void __launch_bounds__(256) k_reduce(const double* __restrict__ partials, int nblocks,
                                               double* __restrict__ out) {
  __shared__ double s[256][7];
  const int t = threadIdx.x;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int b = t; b < nblocks; b += 256)
    for (int q = 0; q < 7; ++q) acc[q] += partials[std::size_t(b) * kRedWidth + q];
  for (int q = 0; q < 7; ++q) s[t][q] = acc[q];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w)
      for (int q = 0; q < 7; ++q) s[t][q] += s[t + w][q];
    __syncthreads();
  }
  if (t < 7) out[t] = s[0][t];
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
    const int b = nbr[std::size_t(s) * npad + a];
    const int mb = cnt[b];
    for (int t = 0; t < mb; ++t) {
      if (nbr[std::size_t(t) * npad + b] == a) {
        const std::size_t q = std::size_t(t) * npad + b;
        fx += sx[q];
        fy += sy[q];
        fz += sz[q];
        break;
      }
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
  r.nhie = R(-0.5 / e.eta);
  r.big_r = R(e.big_r);
  r.inv2d = R(0.5 / e.big_d);
  r.rmd = R(e.big_r - e.big_d);
  r.rpd = R(e.big_r + e.big_d);
  r.nqd = R(-pi / 4 / e.big_d);
  const double c2 = e.c * e.c, d2 = e.d * e.d;
  r.gamma = R(e.gamma);
  r.gcd2 = R(e.gamma * c2 / d2);
  r.gc2 = R(e.gamma * c2);
  r.d2 = R(d2);
  r.h = R(e.h);
  return r;
}

int ceil_div(std::int64_t a, int b) { return int((a + b - 1) / b); }

template <typename R, typename Acc, int G, bool HOIST, bool DET>
void launch_group(Ctx& c, ForceArgs a, int& nblocks_main) {
  const int atoms_per_block = kBlock / G;
  nblocks_main = std::max(1, ceil_div(a.n_owned, atoms_per_block));
  a.partial_base = 0;
  c.mark(2);
  k_force<R, Acc, G, HOIST, DET, false><<<nblocks_main, kBlock, 0, c.stream>>>(a);
  c.mark(3);
  ++c.launches;
}

template <typename R, typename Acc, bool HOIST, bool DET>
void launch_overflow(Ctx& c, ForceArgs a, int base, int nblocks) {
  a.partial_base = base;
  k_force<R, Acc, 32, HOIST, DET, true><<<nblocks, kBlock, 0, c.stream>>>(a);
  ++c.launches;
}

template <typename R, typename Acc, bool HOIST, bool DET>
void run_force(Ctx& c, ForceArgs a) {
  // Group width from the largest short count seen at the last list build
  // (atoms that outgrow it between rebuilds take the overflow launch).
  const int mx = std::max(1, c.short_list.max_count);
  const int g = mx <= 4 ? 4 : mx <= 8 ? 8 : mx <= 16 ? 16 : 32;
  int nb = 0;
  switch (g) {
    case 4: launch_group<R, Acc, 4, HOIST, DET>(c, a, nb); break;
    case 8: launch_group<R, Acc, 8, HOIST, DET>(c, a, nb); break;
    case 16: launch_group<R, Acc, 16, HOIST, DET>(c, a, nb); break;
    default: launch_group<R, Acc, 32, HOIST, DET>(c, a, nb); break;
  }
  const int ovf_blocks = 2 * 148;
  launch_overflow<R, Acc, HOIST, DET>(c, a, nb, ovf_blocks);
  k_reduce<<<1, 256, 0, c.stream>>>(c.partials.get(), nb + ovf_blocks, c.result.get());
  ++c.launches;
}

template <typename R, typename Acc>
void compute_t(Ctx& c, std::uint32_t flags) {
  const bool det = (flags & 0x1u) != 0;
  const std::size_t n = std::size_t(c.n);
  const int npad = c.npad;
  const int cap = c.short_list.cap;

  ForceArgs a{};
  a.pos = c.pos.get();
  a.n_owned = int(c.n);
  a.npad = npad;
  a.box = c.box;
  a.nbr = c.short_list.nbr.get();
  a.cnt = c.short_list.cnt.get();
  a.rows = std::is_same<R, double>::value ? static_cast<const void*>(c.rows_f64.get())
                                          : static_cast<const void*>(c.rows_f32.get());
  a.cutsq = c.cutsq.get();
  a.ns = c.params.species_count();
  a.flags = c.flags.get();
  c.overflow.reserve(std::max<std::size_t>(n, 1));
  a.overflow = c.overflow.get();
  // partial slots: main grid (<= n/4 + 1 blocks) + overflow grid
  c.partials.reserve((n / 4 + 2 + 2 * 148) * kRedWidth);
  a.partials = c.partials.get();
  TSF_CUDA(cudaMemsetAsync(c.flags.get(), 0, 2 * sizeof(int), c.stream));

  const bool hoist = c.hoist_ramp;
  constexpr bool kF32 = std::is_same<Acc, float>::value;
  if (det) {
    c.px.reserve(std::size_t(cap) * npad * sizeof(Acc) / sizeof(double) + 1);
    c.py.reserve(std::size_t(cap) * npad * sizeof(Acc) / sizeof(double) + 1);
    c.pz.reserve(std::size_t(cap) * npad * sizeof(Acc) / sizeof(double) + 1);
    c.fself.reserve(3 * n * sizeof(Acc) / sizeof(double) + 1);
    a.slot_x = c.px.get();
    a.slot_y = c.py.get();
    a.slot_z = c.pz.get();
    a.fself = c.fself.get();
    if (hoist) run_force<R, Acc, true, true>(c, a);
    else run_force<R, Acc, false, true>(c, a);
    if (n > 0) {
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
    TSF_CUDA(cudaMemsetAsync(target, 0, 3 * n * sizeof(Acc), c.stream));
    a.forces = target;
    if (hoist) run_force<R, Acc, true, false>(c, a);
    else run_force<R, Acc, false, false>(c, a);
    if (kF32 && n > 0) {
      k_to_double<<<ceil_div(3 * n, 256), 256, 0, c.stream>>>(
          reinterpret_cast<const float*>(target), c.forces.get(), 3 * n);
      ++c.launches;
    }
  }
}

}  // namespace

void upload_params(Ctx& c) {
  const int s = c.params.species_count();
  if (s > kMaxSpecies)
    throw ConfigError("at most " + std::to_string(kMaxSpecies) + " species are supported");
  std::vector<Row<double>> r64;
  std::vector<Row<float>> r32;
  std::vector<double> cut;
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j)
      for (int k = 0; k < s; ++k) {
        const Entry& e = c.params.entry(i, j, k);
        r64.push_back(make_row<double>(e));
        r32.push_back(make_row<float>(e));
        const double cc = e.cutoff();
        cut.push_back(cc * cc);
      }
  c.rows_f64.reserve(r64.size());
  c.rows_f32.reserve(r32.size());
  c.cutsq.reserve(cut.size());
  TSF_CUDA(cudaMemcpyAsync(c.rows_f64.get(), r64.data(), sizeof(Row<double>) * r64.size(),
                           cudaMemcpyHostToDevice, c.stream));
  TSF_CUDA(cudaMemcpyAsync(c.rows_f32.get(), r32.data(), sizeof(Row<float>) * r32.size(),
                           cudaMemcpyHostToDevice, c.stream));
  TSF_CUDA(cudaMemcpyAsync(c.cutsq.get(), cut.data(), sizeof(double) * cut.size(),
                           cudaMemcpyHostToDevice, c.stream));
  TSF_CUDA(cudaStreamSynchronize(c.stream));
  c.hoist_ramp = c.params.ramp_depends_on_ik_only();
}

void compute(Ctx& c, Precision prec, std::uint32_t flags) {
  switch (prec) {
    case Precision::F64: compute_t<double, double>(c, flags); break;
    case Precision::Mixed: compute_t<float, double>(c, flags); break;
    case Precision::F32: compute_t<float, float>(c, flags); break;
  }
}

}  // namespace tsf
