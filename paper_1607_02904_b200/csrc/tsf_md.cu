// Slot <-> user-order movement at the I/O boundary and the GPU-resident
// velocity-Verlet pieces (proj/src/engine.cpp:142-166: half-kick, drift + wrap,
// ..., half-kick).
#include "tsf_context.hpp"
#include "tsf_units.hpp"

namespace tsf {

namespace {

int blocks_for(std::int64_t n, int b = kBlock) { return int((n + b - 1) / b); }

// the reference position writers track displacements against
// (Ctx::near_list), ref = nullptr when no list of ours describes the slots
DispRef disp_ref(const Ctx& c) {
  return DispRef{c.near_ok ? c.pos_ref.get() : nullptr, c.near_d0.get()};
}

// slot s holds user atom perm[s] (perm == nullptr: identity)
__device__ __forceinline__ int user_of(const int* __restrict__ perm, int s) {
  return perm ? perm[s] : s;
}

__device__ __forceinline__ float4 shadow(const double4& p) {
  return make_float4(float(p.x), float(p.y), float(p.z), float(p.w));
}

__global__ void k_pack(const double* __restrict__ xyz, const int* __restrict__ species,
                       const int* __restrict__ perm, int n, double4* __restrict__ pos,
                       float4* __restrict__ posf, int* __restrict__ cmax,
                       DispRef dref, Box box) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int u = user_of(perm, s);
  const double4 p = make_double4(xyz[3 * u], xyz[3 * u + 1], xyz[3 * u + 2], double(species[u]));
  pos[s] = p;
  posf[s] = shadow(p);
  track_coord_max(cmax, p);
  track_disp(cmax + 5, dref, s, p, box);
}

__global__ void k_refresh_shadow(const double4* __restrict__ pos, int n,
                                 float4* __restrict__ posf, int* __restrict__ cmax,
                                 DispRef dref, Box box) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double4 p = pos[s];
  posf[s] = shadow(p);
  track_coord_max(cmax, p);
  track_disp(cmax + 5, dref, s, p, box);
}

__global__ void k_unpack(const double4* __restrict__ pos, const int* __restrict__ perm, int n,
                         double* __restrict__ xyz) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int u = user_of(perm, s);
  const double4 p = pos[s];
  xyz[3 * u] = p.x;
  xyz[3 * u + 1] = p.y;
  xyz[3 * u + 2] = p.z;
}

// out[perm[s]] = in[s] for 3-vectors (to user order), or out[s] = in[perm[s]]
template <bool kToUser>
__global__ void k_permute3(const double* __restrict__ in, const int* __restrict__ perm, int n,
                           double* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int u = user_of(perm, s);
  const int src = kToUser ? s : u, dst = kToUser ? u : s;
  out[3 * dst] = in[3 * src];
  out[3 * dst + 1] = in[3 * src + 1];
  out[3 * dst + 2] = in[3 * src + 2];
}

__global__ void k_unsort_pos(const double4* __restrict__ in, const int* __restrict__ perm, int n,
                             double4* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  out[perm[s]] = in[s];
}

__device__ __forceinline__ int slot_of(const int* __restrict__ inv, int u) {
  return inv ? inv[u] : u;
}

__global__ void k_gather_pos(const double4* __restrict__ pos, const int* __restrict__ inv,
                             const int* __restrict__ idx, int m, double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const double4 p = pos[slot_of(inv, idx[q])];
  out[3 * q] = p.x;
  out[3 * q + 1] = p.y;
  out[3 * q + 2] = p.z;
}

__global__ void k_scatter_pos(double4* __restrict__ pos, float4* __restrict__ posf,
                              int* __restrict__ cmax, const int* __restrict__ inv,
                              const int* __restrict__ species, int lo, int m,
                              const double* __restrict__ in, DispRef dref, Box box) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const int s = slot_of(inv, lo + q);
  const double4 p = make_double4(in[3 * q], in[3 * q + 1], in[3 * q + 2], double(species[lo + q]));
  pos[s] = p;
  posf[s] = shadow(p);
  track_coord_max(cmax, p);
  track_disp(cmax + 5, dref, s, p, box);
}

__global__ void k_gather_f(const double* __restrict__ f, const int* __restrict__ inv, int lo,
                           int m, double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const int s = slot_of(inv, lo + q);
  out[3 * q] = f[3 * s];
  out[3 * q + 1] = f[3 * s + 1];
  out[3 * q + 2] = f[3 * s + 2];
}

// indices are unique per call (one owner copy per ghost), so no atomics
__global__ void k_add_f(double* __restrict__ f, const int* __restrict__ inv,
                        const int* __restrict__ idx, int m, const double* __restrict__ in) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const int s = slot_of(inv, idx[q]);
  f[3 * s] += in[3 * q];
  f[3 * s + 1] += in[3 * q + 1];
  f[3 * s + 2] += in[3 * q + 2];
}

// wrap_1d (box.hpp:41-46)
__device__ __forceinline__ double wrap(double x, double len) {
  x = __dsub_rn(x, __dmul_rn(len, floor(__ddiv_rn(x, len))));
  if (x < 0.0) x = __dadd_rn(x, len);
  if (x >= len) x = __dsub_rn(x, len);
  return x;
}

struct Masses {
  double m[kMaxSpecies];
};

// (__grid_constant__: the species-indexed mass is read from the parameter
// bank; a plain by-value struct indexed at run time is copied to local memory)
__global__ void k_kick(double4* __restrict__ pos, float4* __restrict__ posf,
                       int* __restrict__ cmax, double* __restrict__ vel, const double* __restrict__ f, int n,
                       const __grid_constant__ Masses ms,
                       double dt, int drift, int kicks, Box box,
                       const double4* __restrict__ ref, double limit_sq,
                       int* __restrict__ moved_flag, const int* __restrict__ perm,
                       int center_limit, DispRef dref,
                       int* __restrict__ seg_flags, int seg_step) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  // a multi-step segment stops at the first step whose kick moved an atom
  // past skin/2: later kicks leave the state as it was (the host rebuilds and
  // resumes from that step)
  if (seg_flags && seg_flags[kFlagMovedAny]) return;
  if (a >= n) return;
  // a decomposition's ghost copies are integrated by their owners and
  // refreshed by the forward exchange (center_limit < n only then)
  if (center_limit < n && (perm ? perm[a] : a) >= center_limit) return;
  double4 p = pos[a];
  const double k = __ddiv_rn(__dmul_rn(0.5, dt), __dmul_rn(ms.m[species_of(p)], kMvv2e));
  // kicks = 2: the closing half-kick of step s and the opening one of s+1
  // (same forces, no sample between them) in one pass — the same two
  // roundings as two launches, so the trajectory is bitwise unchanged
  const double fx = f[3 * a], fy = f[3 * a + 1], fz = f[3 * a + 2];
  double vx = __dadd_rn(vel[3 * a], __dmul_rn(fx, k));
  double vy = __dadd_rn(vel[3 * a + 1], __dmul_rn(fy, k));
  double vz = __dadd_rn(vel[3 * a + 2], __dmul_rn(fz, k));
  if (kicks == 2) {
    vx = __dadd_rn(vx, __dmul_rn(fx, k));
    vy = __dadd_rn(vy, __dmul_rn(fy, k));
    vz = __dadd_rn(vz, __dmul_rn(fz, k));
  }
  vel[3 * a] = vx;
  vel[3 * a + 1] = vy;
  vel[3 * a + 2] = vz;
  if (drift) {
    p.x = __dadd_rn(p.x, __dmul_rn(vx, dt));
    p.y = __dadd_rn(p.y, __dmul_rn(vy, dt));
    p.z = __dadd_rn(p.z, __dmul_rn(vz, dt));
    if (box.per[0]) p.x = wrap(p.x, box.len[0]);
    if (box.per[1]) p.y = wrap(p.y, box.len[1]);
    if (box.per[2]) p.z = wrap(p.z, box.len[2]);
    pos[a] = p;
    posf[a] = shadow(p);
    track_coord_max(cmax, p);
    if (moved_flag || dref.ref) {   // needs_rebuild (neighbor.cpp:134-141) on the new position
      double dx, dy, dz;
      displacement(ref[a], p, box, dx, dy, dz);
      const double d2 = norm_sq_exact(dx, dy, dz);
      const unsigned act = __activemask();
      if (moved_flag && __any_sync(act, d2 > limit_sq) && (threadIdx.x & 31) == __ffs(act) - 1 &&
          __ldcg(moved_flag) == 0) {   // (thousands of warps at a rebuild step: one address)
        atomicOr(moved_flag, 1);
        if (seg_flags) seg_flags[kFlagMovedStep] = seg_step;   // same value from every writer
      }
      if (dref.ref) {   // track_disp on the displacement just computed
        const int v = __reduce_max_sync(act, __float_as_int(near_disp2(dref, a, dx, dy, dz)));
        if ((threadIdx.x & 31) == __ffs(act) - 1) lane_max(cmax + 5, v);
      }
    }
  }
}

// Kinetic energy sum(0.5 m v^2 mvv2e) (system.cpp:16-21), block partials in a
// fixed order then one block finishing the sum: deterministic.
__global__ void __launch_bounds__(256) k_ke_partial(const double4* __restrict__ pos,
                                                    const double* __restrict__ vel, int n,
                                                    const __grid_constant__ Masses ms,
                                                    double* __restrict__ part,
                                                    const int* __restrict__ perm,
                                                    int center_limit) {
  __shared__ double s[256];
  double acc = 0;
  for (int a = blockIdx.x * 256 + threadIdx.x; a < n; a += gridDim.x * 256) {
    if (center_limit < n && (perm ? perm[a] : a) >= center_limit) continue;   // ghosts
    const double m = ms.m[species_of(pos[a])];
    const double vx = vel[3 * a], vy = vel[3 * a + 1], vz = vel[3 * a + 2];
    acc += 0.5 * m * (vx * vx + vy * vy + vz * vz) * kMvv2e;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void k_ke_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double s[256];
  double acc = 0;
  for (int b = threadIdx.x; b < nb; b += 256) acc += part[b];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

Masses masses_of(const Ctx& c) {
  Masses m{};
  for (std::size_t s = 0; s < c.masses.size() && s < std::size_t(kMaxSpecies); ++s)
    m.m[s] = c.masses[s];
  return m;
}

const int* perm_of(const Ctx& c) { return c.sorted ? c.perm.get() : nullptr; }
const int* inv_of(const Ctx& c) { return c.sorted ? c.inv.get() : nullptr; }

}  // namespace

namespace {
__global__ void k_check_species(const int* __restrict__ species, int n, int ns,
                                int* __restrict__ flags) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  const bool bad = a < n && (species[a] < 0 || species[a] >= ns);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, kErrBadSpecies);
}
}  // namespace

namespace {
__global__ void k_scale(double* __restrict__ v, std::size_t m, double f) {
  const std::size_t q = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < m) v[q] *= f;
}
}  // namespace

void md_scale_velocities(Ctx& c, double factor) {
  if (c.n == 0) return;
  k_scale<<<blocks_for(3 * c.n), kBlock, 0, c.stream>>>(c.vel.get(), 3 * std::size_t(c.n),
                                                        factor);
  ++c.launches;
}

void validate_species(Ctx& c, int nspecies) {
  if (c.n == 0) return;
  // flags[7]: survives the per-evaluation reset of flags[0..1]
  k_check_species<<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.species.get(), int(c.n), nspecies,
                                                            c.flags.get() + 7);
  ++c.launches;
}

void gather_positions(Ctx& c, const int* d_idx, std::int64_t m, double* d_xyz) {
  if (m <= 0) return;
  k_gather_pos<<<blocks_for(m), kBlock, 0, c.stream>>>(c.pos.get(), inv_of(c), d_idx, int(m),
                                                       d_xyz);
  ++c.launches;
}

void scatter_positions(Ctx& c, std::int64_t lo, std::int64_t m, const double* d_xyz) {
  if (m <= 0) return;
  k_scatter_pos<<<blocks_for(m), kBlock, 0, c.stream>>>(c.pos.get(), c.posf.get(),
                                                        c.flags.get() + 5, inv_of(c),
                                                        c.species.get(), int(lo), int(m), d_xyz,
                                                        disp_ref(c), c.box);
  ++c.launches;
  c.forces_current = false;
}

void gather_forces(Ctx& c, std::int64_t lo, std::int64_t m, double* d_f) {
  if (m <= 0) return;
  k_gather_f<<<blocks_for(m), kBlock, 0, c.stream>>>(c.forces.get(), inv_of(c), int(lo), int(m),
                                                     d_f);
  ++c.launches;
}

void add_forces(Ctx& c, const int* d_idx, std::int64_t m, const double* d_f) {
  if (m <= 0) return;
  k_add_f<<<blocks_for(m), kBlock, 0, c.stream>>>(c.forces.get(), inv_of(c), d_idx, int(m), d_f);
  ++c.launches;
}

void pack_positions(Ctx& c) {
  if (c.n == 0) return;
  k_pack<<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.xyz_stage.get(), c.species.get(),
                                                   perm_of(c), int(c.n), c.pos.get(),
                                                   c.posf.get(), c.flags.get() + 5, disp_ref(c),
                                                   c.box);
  ++c.launches;
}

void refresh_shadow(Ctx& c) {
  if (c.n == 0) return;
  k_refresh_shadow<<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.pos.get(), int(c.n),
                                                             c.posf.get(), c.flags.get() + 5,
                                                             disp_ref(c), c.box);
  ++c.launches;
}

void unpack_positions(Ctx& c) {
  if (c.n == 0) return;
  k_unpack<<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.pos.get(), perm_of(c), int(c.n),
                                                     c.xyz_stage.get());
  ++c.launches;
}

void unpack_forces(Ctx& c) {
  if (c.n == 0) return;
  c.forces_user.reserve(3 * std::size_t(c.n));
  k_permute3<true><<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.forces.get(), perm_of(c),
                                                             int(c.n), c.forces_user.get());
  ++c.launches;
}

void pack_velocities(Ctx& c) {
  if (c.n == 0) return;
  k_permute3<false><<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.xyz_stage.get(), perm_of(c),
                                                              int(c.n), c.vel.get());
  ++c.launches;
}

void unpack_velocities(Ctx& c) {
  if (c.n == 0) return;
  k_permute3<true><<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.vel.get(), perm_of(c), int(c.n),
                                                             c.xyz_stage.get());
  ++c.launches;
}

void unsort(Ctx& c) {
  c.near_ok = false;   // slots change: the near list no longer describes them
  c.center_slots = -1;   // (identity order: no slot-class truncation of the launches)
  if (!c.sorted || c.n == 0) {
    c.sorted = false;
    return;
  }
  const std::size_t n = std::size_t(c.n);
  c.tmp4.reserve(n);
  c.tmp3.reserve(3 * n);
  const int* perm = c.perm.get();
  k_unsort_pos<<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.pos.get(), perm, int(c.n),
                                                         c.tmp4.get());
  TSF_CUDA(cudaMemcpyAsync(c.pos.get(), c.tmp4.get(), n * sizeof(double4),
                           cudaMemcpyDeviceToDevice, c.stream));
  k_permute3<true><<<blocks_for(c.n), kBlock, 0, c.stream>>>(c.vel.get(), perm, int(c.n),
                                                             c.tmp3.get());
  TSF_CUDA(cudaMemcpyAsync(c.vel.get(), c.tmp3.get(), 3 * n * sizeof(double),
                           cudaMemcpyDeviceToDevice, c.stream));
  c.launches += 2;
  c.sorted = false;
  c.forces_current = false;
  refresh_shadow(c);
}

int center_limit(const Ctx& c) {   // user atoms below it are owned (all unless decomposed)
  const std::int64_t centers = c.n_owned >= 0 ? std::min<std::int64_t>(c.n_owned, c.n) : c.n;
  return int(c.n_energy >= 0 ? std::min<std::int64_t>(c.n_energy, centers) : centers);
}

void md_kick(Ctx& c, double dt, bool drift, int kicks, bool check_rebuild, int seg_step) {
  if (c.n == 0) return;
  const bool check = drift && check_rebuild;
  if (check) TSF_CUDA(cudaMemsetAsync(c.flags.get() + kFlagMoved, 0, sizeof(int), c.stream));
  k_kick<<<blocks_for(c.n), kBlock, 0, c.stream>>>(
      c.pos.get(), c.posf.get(), c.flags.get() + 5, c.vel.get(), c.forces.get(), int(c.n),
      masses_of(c), dt, drift ? 1 : 0, kicks, c.box, c.pos_ref.get(), 0.25 * c.skin * c.skin,
      check ? c.flags.get() + kFlagMoved : nullptr, c.sorted ? c.perm.get() : nullptr, center_limit(c),
      disp_ref(c), seg_step >= 0 ? c.flags.get() : nullptr, seg_step);
  ++c.launches;
}

void md_kinetic(Ctx& c) {
  constexpr int kParts = 296;
  c.partials.reserve(std::size_t(kParts) * kRedWidth);
  k_ke_partial<<<kParts, 256, 0, c.stream>>>(c.pos.get(), c.vel.get(), int(c.n), masses_of(c),
                                             c.partials.get(), c.sorted ? c.perm.get() : nullptr,
                                             center_limit(c));
  k_ke_final<<<1, 256, 0, c.stream>>>(c.partials.get(), kParts, c.result.get() + 7);
  c.launches += 2;
}

}  // namespace tsf
