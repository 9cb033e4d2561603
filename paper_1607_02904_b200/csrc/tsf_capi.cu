// extern "C" boundary (include/tersoff_b200.h) over the device context.
//
// Error behaviour follows the reference: ConfigError / ParseError -> 2,
// NumericError -> 3 (proj/include/tmd/error.hpp:9-21, tools/main.cpp:241-256);
// CUDA failures -> 4.  Messages are kept per context and per thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tersoff_b200.h"
#include "tsf_context.hpp"

struct tsf_params {
  tsf::Params p;
};
struct tsf_ctx {
  tsf::Ctx c;
};

namespace tsf {

// Host-side generators (tsf_generators.cpp).
void diamond_lattice(int nx, int ny, int nz, double a0, std::int32_t sid, double* xyz,
                     std::int32_t* species, double* box);
void perturbed_lattice(const Params& p, int cells, double jitter, std::uint64_t seed,
                       double* xyz, std::int32_t* species, double* masses, double* box);
void maxwell_boltzmann(std::int64_t n, const std::int32_t* species, const double* masses,
                       double temperature, std::uint64_t seed, double* v);
// Device math diagnostics (tsf_force.cu).
void math_probe(const Params& p, int fn, std::int64_t n, const double* x, double* out);
// On-disk snapshots (tsf_snapshot.cpp).
void snapshot_write(const char* path, std::int64_t n, const double* xyz,
                    const std::int32_t* species, int ns, const double* masses, const double* box,
                    const std::uint8_t* periodic, const double* vel, std::uint32_t flags,
                    std::uint8_t* sha_out);
void snapshot_info(const char* path, std::int64_t* n, int* ns, std::uint32_t* flags,
                   std::uint8_t* sha_out);
void snapshot_read(const char* path, double* xyz, std::int32_t* species, double* masses,
                   double* box, std::uint8_t* periodic, double* vel);

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(cudaGetErrorString(e)) + " (" + what + ")");
}

template <typename T>
void DevBuf<T>::reserve(std::size_t n) {
  if (n <= cap) return;
  release();
  TSF_CUDA(cudaMalloc(reinterpret_cast<void**>(&ptr), n * sizeof(T)));
  cap = n;
}

template <typename T>
void DevBuf<T>::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
}

template struct DevBuf<double>;
template struct DevBuf<double4>;
template struct DevBuf<float4>;
template struct DevBuf<int>;
template struct DevBuf<unsigned char>;
template struct DevBuf<unsigned long long>;
template struct DevBuf<unsigned>;
template struct DevBuf<Row<double>>;
template struct DevBuf<Row<float>>;
template struct DevBuf<long long>;

void ensure_pinned(Ctx& c, std::size_t doubles) {
  if (doubles <= c.pinned_cap) return;
  if (c.pinned) cudaFreeHost(c.pinned);
  c.pinned = nullptr;
  c.pinned_cap = 0;
  TSF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c.pinned), doubles * sizeof(double),
                         cudaHostAllocDefault));
  c.pinned_cap = doubles;
}

}  // namespace tsf

namespace {

using tsf::Ctx;
constexpr int kMaxListSpecies = 1 << 20;  // list-only contexts accept any species id

thread_local std::string g_err;

template <typename F>
int guard(Ctx* c, F&& f) {
  int rc = TSF_OK;
  try {
    if (c) tsf::check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
    f();
  } catch (const tsf::ConfigError& e) {
    g_err = e.what();
    rc = TSF_ERR_CONFIG;
  } catch (const tsf::ParseError& e) {
    g_err = e.what();
    rc = TSF_ERR_CONFIG;
  } catch (const tsf::NumericError& e) {
    g_err = e.what();
    rc = TSF_ERR_NUMERIC;
  } catch (const tsf::CudaError& e) {
    g_err = std::string("CUDA error: ") + e.what();
    rc = TSF_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    rc = TSF_ERR_INTERNAL;
  }
  if (rc != TSF_OK && c) c->err = g_err;
  return rc;
}

void check_species(const Ctx& c, std::int64_t n, const std::int32_t* species) {
  const int s = c.has_potential ? c.params.species_count() : kMaxListSpecies;
  for (std::int64_t a = 0; a < n; ++a)
    if (species[a] < 0 || species[a] >= s)
      throw tsf::ConfigError("atom " + std::to_string(a) + " has species id " +
                             std::to_string(species[a]) + " but the parameter table defines " +
                             std::to_string(s) + " species");
}

// Page-locked caller buffers go straight over PCIe; pageable ones through the
// context's pinned staging buffer.
bool is_pinned(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

void upload_xyz(Ctx& c, const double* xyz) {
  const std::size_t m = 3 * std::size_t(c.n);
  if (m == 0) return;
  const double* src = xyz;
  if (!is_pinned(xyz)) {
    tsf::ensure_pinned(c, m);
    std::memcpy(c.pinned, xyz, m * sizeof(double));
    src = c.pinned;
  }
  TSF_CUDA(cudaMemcpyAsync(c.xyz_stage.get(), src, m * sizeof(double), cudaMemcpyHostToDevice,
                           c.stream));
  TSF_CUDA(cudaMemsetAsync(c.flags.get() + 5, 0, sizeof(int), c.stream));  // |coord| max
  tsf::pack_positions(c);
  c.forces_current = false;
}

// Atom count and box of a set_system call: reallocation, list invalidation.
void set_geometry(Ctx& c, std::int64_t n, const double* box, const std::uint8_t* per) {
  bool geometry_changed = n != c.n;
  for (int ax = 0; ax < 3; ++ax) {
    geometry_changed |= c.box.len[ax] != box[ax] || c.box.per[ax] != int(per[ax] != 0);
    c.box.len[ax] = box[ax];
    c.box.per[ax] = per[ax] != 0;
    c.box.quarter[ax] = 0.25 * box[ax];
    c.boxf.len[ax] = float(box[ax]);
    c.boxf.half[ax] = 0.5f * float(box[ax]);
    c.boxf.per[ax] = c.box.per[ax];
    c.boxf.inv[ax] = c.box.per[ax] ? 1.0f / c.boxf.len[ax] : 0.0f;
  }
  if (n != c.n) {
    c.n = n;
    c.sorted = false;
    c.n_owned = -1;
    c.n_energy = -1;
    c.n_interior = -1;
    c.split_slots = -1;
    c.center_slots = -1;
    ++c.list_version;
    c.npad = int(std::max<std::int64_t>(32, (n + 31) / 32 * 32));
    const std::size_t nn = std::size_t(std::max<std::int64_t>(n, 1));
    c.pos.reserve(nn);
    c.posf.reserve(nn);
    c.species.reserve(nn);
    c.xyz_stage.reserve(3 * nn);
    c.forces.reserve(3 * nn);
    c.vel.reserve(3 * nn);
    TSF_CUDA(cudaMemsetAsync(c.vel.get(), 0, 3 * nn * sizeof(double), c.stream));
  }
  if (geometry_changed) {
    c.near_ok = false;
    c.skin_list.valid = false;
    c.short_list.valid = false;
    c.tiled = false;
  }
}

void set_system(Ctx& c, std::int64_t n, const double* xyz, const std::int32_t* species,
                const double* box, const std::uint8_t* per) {
  if (n < 0 || n > (std::int64_t(1) << 30)) throw tsf::ConfigError("atom count out of range");
  for (int ax = 0; ax < 3; ++ax)
    if (!(box[ax] > 0.0)) throw tsf::ConfigError("simulation box edges must be positive");
  if (!species) {
    // the resident species stay (repeat calls on the same system send only positions)
    if (n != c.n || !c.species_set)
      throw tsf::ConfigError("species may be NULL only when the context already holds the "
                             "species of n atoms");
    set_geometry(c, n, box, per);
    upload_xyz(c, xyz);
    return;
  }
  // page-locked species go straight to the device and are validated there (no
  // O(n) host pass per call); pageable ones are checked and cached on the host
  const bool sp_pinned = n > 0 && is_pinned(species);
  if (!sp_pinned) check_species(c, n, species);
  set_geometry(c, n, box, per);
  c.species_set = true;
  if (sp_pinned) {
    TSF_CUDA(cudaMemcpyAsync(c.species.get(), species, sizeof(int) * n, cudaMemcpyHostToDevice,
                             c.stream));
    tsf::validate_species(c, c.has_potential ? c.params.species_count() : kMaxListSpecies);
    c.host_species.clear();
  } else if (n > 0 && (c.host_species.size() != std::size_t(n) ||
                       std::memcmp(c.host_species.data(), species, sizeof(int) * n) != 0)) {
    // species change rarely: re-upload only when they differ from the last upload
    c.host_species.assign(species, species + n);
    TSF_CUDA(cudaMemcpyAsync(c.species.get(), c.host_species.data(), sizeof(int) * n,
                             cudaMemcpyHostToDevice, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
  }
  upload_xyz(c, xyz);
}

void download_forces(Ctx& c, double* forces) {
  const std::size_t m = 3 * std::size_t(c.n);
  if (m == 0) return;
  tsf::unpack_forces(c);  // slot order -> user order
  if (is_pinned(forces)) {
    TSF_CUDA(cudaMemcpyAsync(forces, c.forces_user.get(), m * sizeof(double),
                             cudaMemcpyDeviceToHost, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  tsf::ensure_pinned(c, m);
  TSF_CUDA(cudaMemcpyAsync(c.pinned, c.forces_user.get(), m * sizeof(double),
                           cudaMemcpyDeviceToHost, c.stream));
  TSF_CUDA(cudaStreamSynchronize(c.stream));
  std::memcpy(forces, c.pinned, m * sizeof(double));
}

void raise_device_errors(Ctx& c) {
  int f[24] = {0};
  TSF_CUDA(cudaMemcpyAsync(f, c.flags.get(), sizeof f, cudaMemcpyDeviceToHost, c.stream));
  TSF_CUDA(cudaStreamSynchronize(c.stream));
  if (f[tsf::kFlagFilterNaN]) {
    TSF_CUDA(cudaMemsetAsync(c.flags.get() + tsf::kFlagFilterNaN, 0, sizeof(int), c.stream));
    throw tsf::NumericError("non-finite pair term (a coordinate is NaN)");
  }
  if (f[7] & tsf::kErrBadSpecies) {
    TSF_CUDA(cudaMemsetAsync(c.flags.get() + 7, 0, sizeof(int), c.stream));
    c.host_species.clear();
    throw tsf::ConfigError("a species id lies outside the parameter table's species");
  }
  if (f[0] & tsf::kErrShortOverflow)
    throw tsf::ConfigError("an atom has more than 32 neighbours within r_cut_max");
  if (f[0] & tsf::kErrNonFinite) throw tsf::NumericError("non-finite pair term");
}

void finish(Ctx& c, double* energy, double* forces, double* virial) {
  if (!energy && !forces && !virial) return;
  double res[8];
  TSF_CUDA(cudaMemcpyAsync(res, c.result.get(), 7 * sizeof(double), cudaMemcpyDeviceToHost,
                           c.stream));
  if (forces) download_forces(c, forces);
  raise_device_errors(c);
  if (energy) *energy = res[0];
  if (virial)
    for (int q = 0; q < 6; ++q) virial[q] = res[1 + q];
}

void set_phase(Ctx& c, int lo, int hi, bool first, bool last) {
  c.phase_lo = lo;
  c.phase_hi = hi;
  c.phase_first = first;
  c.phase_last = last;
}

// One evaluation's device work: the short-list filter and the force launches.
void evaluate_launches(Ctx& c, tsf::Precision p, std::uint32_t flags) {
  set_phase(c, 0, int(c.n), true, true);
  c.phase_blocks = 0;
  c.mark(0);
  // The short list is rebuilt from the skin list on every evaluation, as the
  // reference does (kernels.hpp:187-188).  A filter fused into the force
  // kernel measured slower (profiles/r01): its gathers then sit
  // in the register-limited force kernel.  Pairs beyond every cutoff of their
  // species pair are dropped here as well: they add exact zeros in the
  // reference (the kernel tests the same exact r^2).
  // atomic mode: the filter launch also zeroes the force accumulator (the
  // f64/mixed double forces, or the f32 float partials)
  void* zf = nullptr;
  int zb = 0;
  if (!(flags & TSF_DETERMINISTIC) && c.n > 0) {
    if (p == tsf::Precision::F32) {
      c.fself.reserve(3 * std::size_t(c.n) * sizeof(float) / sizeof(double) + 1);
      zf = c.fself.get();
      zb = 4;
    } else {
      zf = c.forces.get();
      zb = 8;
    }
  }
  // the filter launch (none for an empty system) also zeroes flags[0..3]
  const bool zero_flags = c.n > 0;
  tsf::list_filter(c, (flags & TSF_NO_FILTER) ? tsf::FilterMode::Copy : tsf::FilterMode::Pair,
                   zf, zb, 0, -1, zero_flags);
  c.mark(1);
  tsf::compute(c, p, (zf ? (flags | tsf::kFlagForcesZeroed) : flags) |
                         (zero_flags ? tsf::kFlagFlagsZeroed : 0u));
  c.mark(4);
}

}  // namespace (reopened below)

namespace tsf {
int pdl_level() {
  static const int level = [] {
    const char* e = std::getenv("TSF_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return level;
}
}  // namespace tsf

namespace {

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TSF_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// A fresh capture goes into the slot's executable graph by cudaGraphExecUpdate
// when the topology is unchanged (after a list rebuild: the same launches with
// new parameters), else by a new instantiation — updates cost a fraction of an
// instantiation, and an MD run re-captures after every rebuild.
bool install_graph(cudaGraphExec_t& exec, cudaGraph_t g) {
  if (exec) {
    cudaGraphExecUpdateResultInfo info{};
    if (cudaGraphExecUpdate(exec, g, &info) == cudaSuccess) return true;
    cudaGetLastError();
    cudaGraphExecDestroy(exec);
    exec = nullptr;
  }
  return cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
}

// Replay slot `slot`'s graph while its key holds; capture it on the second
// eager run with the same key; else run eagerly.  `launches` must leave the
// same host state on every run with one key (restored on replay).
template <typename F>
void run_graphed(Ctx& c, int slot, bool graphable, const std::uint64_t* key, F&& launches) {
  Ctx::GraphSlot& s = c.graph[slot];
  if (graphable && s.exec && std::equal(key, key + 6, s.key)) {
    TSF_CUDA(cudaGraphLaunch(s.exec, c.stream));
    c.launches += s.launches;
    c.phase_blocks = s.phase_blocks;
    return;
  }
  if (!(graphable && std::equal(key, key + 6, s.warm))) {
    launches();
    std::copy(key, key + 6, s.warm);
    return;
  }
  const std::int64_t l0 = c.launches;
  const int pb0 = c.phase_blocks;
  cudaGraph_t g = nullptr;
  bool ok = cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    try {
      launches();
    } catch (...) {
      ok = false;
    }
    ok = cudaStreamEndCapture(c.stream, &g) == cudaSuccess && ok;
    ok = ok && install_graph(s.exec, g);
    if (g) cudaGraphDestroy(g);
  }
  if (ok) {
    s.launches = c.launches - l0;
    s.phase_blocks = c.phase_blocks;
    std::copy(key, key + 6, s.key);
    TSF_CUDA(cudaGraphLaunch(s.exec, c.stream));
  } else {   // capture refused: clear the sticky error and stay eager
    cudaGetLastError();
    if (s.exec) cudaGraphExecDestroy(s.exec);
    s.exec = nullptr;
    c.graphs_off = true;
    c.launches = l0;
    c.phase_blocks = pb0;
    launches();
  }
}

// Steady-state evaluations replay a CUDA graph of evaluate_launches: between
// list rebuilds every launch has the same configuration and arguments (device
// buffers, group width, grid sizes), so at small N — where ~10 launches and
// memsets per step, not the GPU, set the pace — one graph launch replaces
// them.  The key covers everything a launch's arguments depend on; a graph is
// captured on the second evaluation with a key (the first, eager one grows
// every buffer), never right after a rebuild (the filter then reads the
// short-count distribution back synchronously) and never while profiling.
void evaluate(Ctx& c, tsf::Precision p, std::uint32_t flags) {
  if (!c.has_potential)
    throw tsf::ConfigError("context was created without a parameter table (list-only)");
  if (!c.skin_list.valid)
    throw tsf::ConfigError(
        "no neighbor list: call tsf_build_neighbor_list or tsf_set_neighbor_list first");
  const int mode = int((flags & TSF_NO_FILTER) ? tsf::FilterMode::Copy : tsf::FilterMode::Pair);
  const bool steady = !c.short_max_stale && c.short_apply == mode;
  const std::uint64_t key[6] = {c.list_version, std::uint64_t(p),
                                flags | (c.speculative ? 0x80000000u : 0u), std::uint64_t(c.n),
                                std::uint64_t(c.n_owned),
                                std::uint64_t(reinterpret_cast<std::uintptr_t>(c.stream))};
  const bool graphable = graphs_enabled() && !c.graphs_off && !c.profile && steady && c.n > 0;
  run_graphed(c, 0, graphable, key, [&] { evaluate_launches(c, p, flags); });
  c.forces_current = true;
  if (c.profile) {
    TSF_CUDA(cudaEventSynchronize(c.ev[4]));
    for (int k = 0; k < 4; ++k) {
      float ms = 0;
      TSF_CUDA(cudaEventElapsedTime(&ms, c.ev[k], c.ev[k + 1]));
      c.stage_ms[k] += ms;
    }
    ++c.profiled_calls;
  }
}

}  // namespace

// Context operations for the other translation units (tsf_dd.cu: the domain
// decomposition drives a context with device-resident inputs).
namespace tsf {
void evaluate_ctx(Ctx& c, Precision p, std::uint32_t flags) { evaluate(c, p, flags); }
void raise_errors(Ctx& c) { raise_device_errors(c); }
// set_system with device arrays (positions AoS [n][3] user order, species)
void set_system_device(Ctx& c, std::int64_t n, const double* d_xyz, const int* d_species,
                       const double* box, const std::uint8_t* per) {
  if (n < 0 || n > (std::int64_t(1) << 30)) throw ConfigError("atom count out of range");
  for (int ax = 0; ax < 3; ++ax)
    if (!(box[ax] > 0.0)) throw ConfigError("simulation box edges must be positive");
  set_geometry(c, n, box, per);
  c.host_species.clear();
  c.species_set = true;
  if (n == 0) return;
  TSF_CUDA(cudaMemcpyAsync(c.species.get(), d_species, sizeof(int) * n, cudaMemcpyDeviceToDevice,
                           c.stream));
  validate_species(c, c.has_potential ? c.params.species_count() : kMaxListSpecies);
  TSF_CUDA(cudaMemcpyAsync(c.xyz_stage.get(), d_xyz, 3 * n * sizeof(double),
                           cudaMemcpyDeviceToDevice, c.stream));
  TSF_CUDA(cudaMemsetAsync(c.flags.get() + 5, 0, sizeof(int), c.stream));
  pack_positions(c);
  c.forces_current = false;
}
// velocities (AoS [n][3] user order) from device memory; masses per species
void set_velocities_device(Ctx& c, const double* d_vel, const double* masses) {
  const int s = c.params.species_count();
  for (int q = 0; q < s; ++q)
    if (!(masses[q] > 0.0)) throw ConfigError("species " + std::to_string(q) + " has non-positive mass");
  c.masses.assign(masses, masses + s);
  if (c.n == 0) return;
  TSF_CUDA(cudaMemcpyAsync(c.xyz_stage.get(), d_vel, 3 * c.n * sizeof(double),
                           cudaMemcpyDeviceToDevice, c.stream));
  pack_velocities(c);
}
// user-order positions / velocities of atoms [0, m) into device arrays
void get_state_device(Ctx& c, std::int64_t m, double* d_xyz, double* d_vel) {
  if (m <= 0) return;
  if (d_xyz) {
    unpack_positions(c);
    TSF_CUDA(cudaMemcpyAsync(d_xyz, c.xyz_stage.get(), 3 * m * sizeof(double),
                             cudaMemcpyDeviceToDevice, c.stream));
  }
  if (d_vel) {
    unpack_velocities(c);
    TSF_CUDA(cudaMemcpyAsync(d_vel, c.xyz_stage.get(), 3 * m * sizeof(double),
                             cudaMemcpyDeviceToDevice, c.stream));
  }
}
}  // namespace tsf

namespace {

// Would evaluate() replay its graph now (so it can be captured inside a
// larger graph as a child)?
bool evaluate_replays(Ctx& c, tsf::Precision p, std::uint32_t flags) {
  const int mode = int((flags & TSF_NO_FILTER) ? tsf::FilterMode::Copy : tsf::FilterMode::Pair);
  const bool steady = !c.short_max_stale && c.short_apply == mode;
  const std::uint64_t key[6] = {c.list_version, std::uint64_t(p),
                                flags | (c.speculative ? 0x80000000u : 0u), std::uint64_t(c.n),
                                std::uint64_t(c.n_owned),
                                std::uint64_t(reinterpret_cast<std::uintptr_t>(c.stream))};
  const Ctx::GraphSlot& g = c.graph[0];
  return graphs_enabled() && !c.graphs_off && !c.profile && steady && c.n > 0 && g.exec &&
         std::equal(key, key + 6, g.key);
}

// An MD segment: replayed from graph slot 3 while its key holds, captured at
// its first graphable run (segments repeat only within one list's life), else
// launched eagerly.
template <typename F>
void run_segment(Ctx& c, const std::uint64_t* key, bool graphable, F&& launches) {
  Ctx::GraphSlot& s = c.graph[3];
  if (graphable && s.exec && std::equal(key, key + 6, s.key)) {
    TSF_CUDA(cudaGraphLaunch(s.exec, c.stream));
    c.launches += s.launches;
    return;
  }
  if (!graphable) {
    launches();
    return;
  }
  const std::int64_t l0 = c.launches;
  cudaGraph_t g = nullptr;
  bool ok = cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    try {
      launches();
    } catch (...) {
      ok = false;
    }
    ok = cudaStreamEndCapture(c.stream, &g) == cudaSuccess && ok;
    ok = ok && install_graph(s.exec, g);
    if (g) cudaGraphDestroy(g);
  }
  if (ok) {
    s.launches = c.launches - l0;
    std::copy(key, key + 6, s.key);
    TSF_CUDA(cudaGraphLaunch(s.exec, c.stream));
  } else {
    cudaGetLastError();
    if (s.exec) cudaGraphExecDestroy(s.exec);
    s.exec = nullptr;
    c.graphs_off = true;
    c.launches = l0;
    launches();
  }
}

int compute_entry(tsf_ctx* ctx, tsf::Precision p, std::uint32_t flags, double* e, double* f,
                  double* w) {
  // outputs asked for without the virial: it is never formed.  (All three
  // NULL: the caller reads the device results, virial included.)
  if (!w && (e || f)) flags |= tsf::kFlagNoVirial;
  return guard(&ctx->c, [&] {
    evaluate(ctx->c, p, flags);
    finish(ctx->c, e, f, w);
  });
}

std::vector<int> download_ell(Ctx& c, const tsf::ListState& s, std::vector<int>& cnt) {
  cnt.assign(std::size_t(c.n), 0);
  std::vector<int> ell(std::size_t(s.cap) * c.npad);
  if (c.n == 0) return ell;
  TSF_CUDA(cudaMemcpyAsync(cnt.data(), s.cnt.get(), sizeof(int) * c.n, cudaMemcpyDeviceToHost,
                           c.stream));
  if (!ell.empty())
    TSF_CUDA(cudaMemcpyAsync(ell.data(), s.nbr.get(), sizeof(int) * ell.size(),
                             cudaMemcpyDeviceToHost, c.stream));
  TSF_CUDA(cudaStreamSynchronize(c.stream));
  return ell;
}

const tsf::ListState& list_for(Ctx& c, int which) {
  if (!c.skin_list.valid) throw tsf::ConfigError("no neighbor list has been built");
  if (which == TSF_LIST_SKIN) return c.skin_list;
  if (which != TSF_LIST_SHORT) throw tsf::ConfigError("unknown list selector");
  if (!c.has_potential) throw tsf::ConfigError("the short list needs a parameter table");
  tsf::list_filter(c, tsf::FilterMode::Cutoff);
  return c.short_list;
}

}  // namespace

extern "C" {

const char* tsf_error_message(void) { return g_err.c_str(); }
const char* tsf_last_error(const tsf_ctx* ctx) { return ctx ? ctx->c.err.c_str() : g_err.c_str(); }
const char* tsf_version(void) { return "paper_1607_02904_b200 0.1.0 (sm_100a)"; }

/* ---- parameters ---- */
int tsf_params_parse(const char* text, size_t len, const char* source_name, tsf_params** out) {
  return guard(nullptr, [&] {
    *out = new tsf_params{tsf::parse_params(std::string_view(text, len),
                                            source_name ? source_name : "<string>")};
  });
}
int tsf_params_load(const char* path, tsf_params** out) {
  return guard(nullptr, [&] { *out = new tsf_params{tsf::load_params(path)}; });
}
int tsf_params_builtin_silicon(tsf_params** out) {
  return guard(nullptr, [&] { *out = new tsf_params{tsf::builtin_silicon()}; });
}
void tsf_params_free(tsf_params* p) { delete p; }
int tsf_params_species_count(const tsf_params* p) { return p->p.species_count(); }
const char* tsf_params_species_name(const tsf_params* p, int s) {
  if (s < 0 || s >= p->p.species_count()) return nullptr;
  return p->p.species()[std::size_t(s)].c_str();
}
int tsf_params_species_id(const tsf_params* p, const char* name) {
  return p->p.species_id(name);
}
double tsf_params_r_cut_max(const tsf_params* p) { return p->p.r_cut_max(); }
int tsf_params_flat_rows(const tsf_params* p, double* rows, size_t cap) {
  const std::vector<double> r = p->p.flat_rows();
  if (cap < r.size()) {
    g_err = "row buffer too small";
    return TSF_ERR_CONFIG;
  }
  std::copy(r.begin(), r.end(), rows);
  return TSF_OK;
}
int64_t tsf_params_serialize(const tsf_params* p, char* buf, size_t cap) {
  const std::string s = p->p.serialize();
  if (buf && cap > 0) {
    const std::size_t m = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), m);
    buf[m] = '\0';
  }
  return int64_t(s.size());
}

/* ---- generators ---- */
int64_t tsf_diamond_lattice_size(int nx, int ny, int nz) {
  return int64_t(nx) * ny * nz * 8;
}
int tsf_make_diamond_lattice(int nx, int ny, int nz, double a0, int32_t species_id, double* xyz,
                             int32_t* species, double* box) {
  return guard(nullptr,
               [&] { tsf::diamond_lattice(nx, ny, nz, a0, species_id, xyz, species, box); });
}
int tsf_perturbed_lattice(const tsf_params* p, int cells, double jitter, uint64_t seed,
                          double* xyz, int32_t* species, double* masses, double* box) {
  return guard(nullptr, [&] {
    tsf::perturbed_lattice(p->p, cells, jitter, seed, xyz, species, masses, box);
  });
}
int tsf_init_velocities(int64_t n, const int32_t* species, const double* masses,
                        double temperature, uint64_t seed, double* vel) {
  return guard(nullptr,
               [&] { tsf::maxwell_boltzmann(n, species, masses, temperature, seed, vel); });
}

/* ---- diagnostics ---- */
int tsf_math_probe(const tsf_params* p, int fn, int64_t n, const double* x, double* out) {
  return guard(nullptr, [&] { tsf::math_probe(p->p, fn, n, x, out); });
}

/* ---- snapshots ---- */
int tsf_snapshot_write(const char* path, int64_t n, const double* xyz, const int32_t* species,
                       int nspecies, const double* masses, const double box[3],
                       const uint8_t periodic[3], const double* vel, uint32_t flags,
                       uint8_t sha256_out[32]) {
  return guard(nullptr, [&] {
    tsf::snapshot_write(path, n, xyz, species, nspecies, masses, box, periodic, vel, flags,
                        sha256_out);
  });
}
int tsf_snapshot_info(const char* path, int64_t* n, int* nspecies, uint32_t* flags,
                      uint8_t sha256_out[32]) {
  return guard(nullptr, [&] { tsf::snapshot_info(path, n, nspecies, flags, sha256_out); });
}
int tsf_snapshot_read(const char* path, double* xyz, int32_t* species, double* masses,
                      double box[3], uint8_t periodic[3], double* vel) {
  return guard(nullptr,
               [&] { tsf::snapshot_read(path, xyz, species, masses, box, periodic, vel); });
}

/* ---- context ---- */
int tsf_create(const tsf_params* p, int device, tsf_ctx** out) {
  *out = nullptr;
  tsf_ctx* ctx = nullptr;
  const int rc = guard(nullptr, [&] {
    int count = 0;
    tsf::check_cuda(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count)
      throw tsf::ConfigError("CUDA device " + std::to_string(device) + " not available (" +
                             std::to_string(count) + " visible)");
    tsf::check_cuda(cudaSetDevice(device), "cudaSetDevice");
    ctx = new tsf_ctx{tsf::Ctx(p ? p->p : tsf::builtin_silicon())};
    Ctx& c = ctx->c;
    c.has_potential = p != nullptr;
    c.device = device;
    TSF_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    c.own_stream = c.stream;
    c.flags.reserve(32);
    c.result.reserve(8);
    TSF_CUDA(cudaMemsetAsync(c.flags.get(), 0, 32 * sizeof(int), c.stream));
    TSF_CUDA(cudaMemsetAsync(c.result.get(), 0, 8 * sizeof(double), c.stream));
    tsf::upload_params(c);
    c.masses.assign(std::size_t(c.params.species_count()), 28.0855);
  });
  if (rc != TSF_OK) {
    if (ctx) tsf_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return TSF_OK;
}

void tsf_destroy(tsf_ctx* ctx) {
  if (!ctx) return;
  Ctx& c = ctx->c;
  cudaSetDevice(c.device);
  if (c.stream) cudaStreamSynchronize(c.stream);
  if (c.pinned) cudaFreeHost(c.pinned);
  c.pinned = nullptr;
  if (c.pinned_flag) cudaFreeHost(c.pinned_flag);
  if (c.flag_event) cudaEventDestroy(c.flag_event);
  for (auto& g : c.graph)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& e : c.ev)
    if (e) cudaEventDestroy(e);
  cudaStream_t s = c.own_stream;       // never destroy a caller's stream
  delete ctx;  // DevBufs free themselves
  if (s) cudaStreamDestroy(s);
}

int tsf_set_stream(tsf_ctx* ctx, void* stream) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    c.stream = stream ? static_cast<cudaStream_t>(stream) : c.own_stream;
  });
}

int tsf_set_centers(tsf_ctx* ctx, int64_t n_owned, int64_t n_centers) {
  return guard(&ctx->c, [&] {
    if (n_centers > ctx->c.n) throw tsf::ConfigError("center count exceeds the atom count");
    if (n_owned > n_centers) throw tsf::ConfigError("owned count exceeds the center count");
    ctx->c.n_owned = n_centers < 0 ? -1 : n_centers;
    ctx->c.n_energy = n_owned < 0 ? -1 : n_owned;
    ++ctx->c.list_version;
  });
}

int tsf_set_interior(tsf_ctx* ctx, int64_t n_interior) {
  return guard(&ctx->c, [&] {
    if (n_interior > ctx->c.n) throw tsf::ConfigError("interior count exceeds the atom count");
    ctx->c.n_interior = n_interior < 0 ? -1 : n_interior;
    ctx->c.split_slots = -1;     // takes effect with the next list build
    ++ctx->c.list_version;
  });
}

int tsf_compute_phase(tsf_ctx* ctx, int precision, uint32_t flags, int phase) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (precision < 0 || precision > 2) throw tsf::ConfigError("unknown precision selector");
    if (phase != 0 && phase != 1) throw tsf::ConfigError("phase must be 0 or 1");
    const tsf::Precision p = tsf::Precision(precision);
    const int mode = int((flags & TSF_NO_FILTER) ? tsf::FilterMode::Copy : tsf::FilterMode::Pair);
    if (phase == 0) {
      c.phase0_done = false;
      if (!c.has_potential || !c.skin_list.valid) return;   // phase 1 reports it
      const bool steady = !c.short_max_stale && c.short_apply == mode;
      if (c.split_slots < 0 || !steady || c.profile) return;   // phase 1 does it all
      const int split = int(c.split_slots);
      const std::uint64_t key[6] = {c.list_version, std::uint64_t(p), flags, std::uint64_t(c.n),
                                    std::uint64_t(split),
                                    std::uint64_t(reinterpret_cast<std::uintptr_t>(c.stream))};
      // graph-replayed like evaluate(): at 8 ranks a phase's dozen launches
      // set the pace of a 0.1 ms step (tools/rank_share.py)
      run_graphed(c, 1, graphs_enabled() && !c.graphs_off && c.n > 0, key, [&] {
        set_phase(c, 0, split, true, false);
        c.phase_blocks = 0;
        tsf::list_filter(c, tsf::FilterMode(mode), nullptr, 0, 0, split);
        tsf::compute(c, p, flags);
      });
      c.phase0_done = true;
      c.forces_current = false;
      return;
    }
    if (!c.phase0_done) {          // no split (or not steady): one full evaluation
      evaluate(c, p, flags);
      return;
    }
    const int split = int(c.split_slots);
    const std::uint64_t key[6] = {c.list_version, std::uint64_t(p), flags, std::uint64_t(c.n),
                                  std::uint64_t(split),
                                  std::uint64_t(reinterpret_cast<std::uintptr_t>(c.stream))};
    run_graphed(c, 2, graphs_enabled() && !c.graphs_off && c.n > 0, key, [&] {
      set_phase(c, split, int(c.n), false, true);
      tsf::list_filter(c, tsf::FilterMode(mode), nullptr, 0, split, int(c.n));
      tsf::compute(c, p, flags);
    });
    set_phase(c, 0, int(c.n), true, true);
    c.phase0_done = false;
    c.forces_current = true;
  });
}

int tsf_set_owned(tsf_ctx* ctx, int64_t n_owned) {
  return guard(&ctx->c, [&] {
    if (n_owned > ctx->c.n) throw tsf::ConfigError("owned count exceeds the atom count");
    ctx->c.n_owned = n_owned < 0 ? -1 : n_owned;
    ctx->c.n_energy = -1;
    ++ctx->c.list_version;
    ctx->c.forces_current = false;
  });
}

int tsf_gather_positions(tsf_ctx* ctx, const int32_t* d_idx, int64_t m, double* d_xyz) {
  return guard(&ctx->c, [&] { tsf::gather_positions(ctx->c, d_idx, m, d_xyz); });
}

int tsf_scatter_positions(tsf_ctx* ctx, int64_t lo, int64_t m, const double* d_xyz) {
  return guard(&ctx->c, [&] {
    if (lo < 0 || lo + m > ctx->c.n) throw tsf::ConfigError("position range out of bounds");
    tsf::scatter_positions(ctx->c, lo, m, d_xyz);
  });
}

int tsf_gather_forces(tsf_ctx* ctx, int64_t lo, int64_t m, double* d_f) {
  return guard(&ctx->c, [&] {
    if (lo < 0 || lo + m > ctx->c.n) throw tsf::ConfigError("force range out of bounds");
    tsf::gather_forces(ctx->c, lo, m, d_f);
  });
}

int tsf_add_forces(tsf_ctx* ctx, const int32_t* d_idx, int64_t m, const double* d_f) {
  return guard(&ctx->c, [&] { tsf::add_forces(ctx->c, d_idx, m, d_f); });
}

int tsf_results_device(tsf_ctx* ctx, double* d_ev, double* d_forces) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (d_ev)
      TSF_CUDA(cudaMemcpyAsync(d_ev, c.result.get(), 7 * sizeof(double),
                               cudaMemcpyDeviceToDevice, c.stream));
    if (d_forces && c.n > 0) {
      tsf::unpack_forces(c);
      TSF_CUDA(cudaMemcpyAsync(d_forces, c.forces_user.get(), 3 * c.n * sizeof(double),
                               cudaMemcpyDeviceToDevice, c.stream));
    }
  });
}

void* tsf_stream(tsf_ctx* ctx) { return ctx ? static_cast<void*>(ctx->c.stream) : nullptr; }

int tsf_profile_enable(tsf_ctx* ctx, int on) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (on && !c.ev[0])
      for (auto& e : c.ev) TSF_CUDA(cudaEventCreate(&e));
    c.profile = on != 0;
  });
}

int tsf_profile_read(tsf_ctx* ctx, double* ms, int64_t* calls, int reset) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    for (int k = 0; k < 4; ++k) ms[k] = c.stage_ms[k];
    if (calls) *calls = c.profiled_calls;
    if (reset) {
      for (double& v : c.stage_ms) v = 0;
      c.profiled_calls = 0;
    }
  });
}
int64_t tsf_launch_count(const tsf_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int64_t tsf_near_refreshes(tsf_ctx* ctx) {
  if (!ctx) return -1;
  int v = -1;
  const int rc = guard(&ctx->c, [&] {
    TSF_CUDA(cudaMemcpyAsync(&v, ctx->c.flags.get() + tsf::kFlagNearRefreshCount, sizeof(int),
                             cudaMemcpyDeviceToHost, ctx->c.stream));
    TSF_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
  return rc == TSF_OK ? v : -1;
}

int tsf_set_system(tsf_ctx* ctx, int64_t n, const double* xyz, const int32_t* species,
                   const double box[3], const uint8_t periodic[3]) {
  return guard(&ctx->c, [&] { set_system(ctx->c, n, xyz, species, box, periodic); });
}
int tsf_set_positions(tsf_ctx* ctx, const double* xyz) {
  return guard(&ctx->c, [&] { upload_xyz(ctx->c, xyz); });
}
int tsf_get_positions(tsf_ctx* ctx, double* xyz) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    const std::size_t m = 3 * std::size_t(c.n);
    if (m == 0) return;
    tsf::unpack_positions(c);
    tsf::ensure_pinned(c, m);
    TSF_CUDA(cudaMemcpyAsync(c.pinned, c.xyz_stage.get(), m * sizeof(double),
                             cudaMemcpyDeviceToHost, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    std::memcpy(xyz, c.pinned, m * sizeof(double));
  });
}

int tsf_build_neighbor_list(tsf_ctx* ctx, double cutoff, double skin) {
  return guard(&ctx->c, [&] { tsf::list_build(ctx->c, cutoff, skin); });
}

// Identity of an adopted list: a 4-lane multiply-xor hash over every word
// of (n, cutoff, skin, offsets, neighbors) — ~30 GB/s on the host, so the
// drop-in shim's per-call adoption of the same NeighborList (Engine::run
// passes it every step, engine.cpp:136-140) costs a scan instead of the
// CSR -> ELL conversion, the upload and a new graph key.
std::uint64_t list_identity(std::int64_t n, const int32_t* offsets, const int32_t* nbrs,
                            double cutoff, double skin) {
  constexpr std::uint64_t kMul = 0x9E3779B97F4A7C15ull;
  std::uint64_t h[4] = {std::uint64_t(n) ^ 0x243F6A8885A308D3ull, 0x13198A2E03707344ull,
                        0xA4093822299F31D0ull, 0x082EFA98EC4E6C89ull};
  std::uint64_t cb, sb;
  std::memcpy(&cb, &cutoff, 8);
  std::memcpy(&sb, &skin, 8);
  h[1] ^= cb;
  h[2] ^= sb;
  auto mix = [&](const int32_t* p, std::int64_t len) {
    std::int64_t i = 0;
    for (; i + 8 <= len; i += 8)
      for (int l = 0; l < 4; ++l) {
        std::uint64_t w;
        std::memcpy(&w, p + i + 2 * l, 8);
        h[l] = (h[l] ^ w) * kMul;
        h[l] ^= h[l] >> 29;
      }
    for (; i < len; ++i) h[0] = ((h[0] ^ std::uint32_t(p[i])) * kMul) ^ (h[0] >> 31);
  };
  mix(offsets, n + 1);
  mix(nbrs, offsets[n]);
  std::uint64_t r = h[0];
  for (int l = 1; l < 4; ++l) r = (r ^ (h[l] + kMul + (r << 6) + (r >> 2))) * kMul;
  return r ^ (r >> 32);
}

int tsf_set_neighbor_list(tsf_ctx* ctx, const int32_t* offsets, const int32_t* nbrs,
                          double cutoff, double skin) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (offsets[0] != 0) throw tsf::ConfigError("neighbor offsets must start at 0");
    const std::uint64_t id = list_identity(c.n, offsets, nbrs, cutoff, skin);
    if (c.adopted_valid && c.adopted_id == id && c.skin_list.valid && !c.sorted) {
      ++c.adoption_hits;   // the list already on the device: keep it, its graphs
      return;              // and its reference positions
    }
    c.adopted_valid = false;
    tsf::unsort(c);  // an external list speaks user indices: slot == user index
    c.short_list.valid = false;
    c.tiled = false;
    int mx = 0;
    for (std::int64_t a = 0; a < c.n; ++a) {
      const int len = offsets[a + 1] - offsets[a];
      if (len < 0) throw tsf::ConfigError("neighbor offsets must be non-decreasing");
      mx = std::max(mx, len);
    }
    // >= 16 entries: the filter reads the first 4 ELL4 rows unconditionally
    const int cap = std::max(16, (mx + 3) / 4 * 4);
    std::vector<int> ell(std::size_t(cap) * c.npad, 0), cnt(std::size_t(c.npad), 0);
    for (std::int64_t a = 0; a < c.n; ++a) {
      cnt[std::size_t(a)] = offsets[a + 1] - offsets[a];
      for (int s = offsets[a]; s < offsets[a + 1]; ++s) {
        const int b = nbrs[s];
        if (b < 0 || b >= c.n || b == a)
          throw tsf::ConfigError("neighbor index out of range in segment of atom " +
                                 std::to_string(a));
        ell[tsf::ell_at(s - offsets[a], int(a), c.npad)] = b;
      }
    }
    c.skin_list.cap = cap;
    c.skin_list.nbr.reserve(ell.size());
    c.skin_list.cnt.reserve(cnt.size());
    // ordered on the context's stream (a filter may still read the old list)
    // and complete before the pageable host vectors go out of scope
    TSF_CUDA(cudaMemcpyAsync(c.skin_list.nbr.get(), ell.data(), sizeof(int) * ell.size(),
                             cudaMemcpyHostToDevice, c.stream));
    TSF_CUDA(cudaMemcpyAsync(c.skin_list.cnt.get(), cnt.data(), sizeof(int) * cnt.size(),
                             cudaMemcpyHostToDevice, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    c.skin_list.max_count = mx;
    c.skin_list.valid = true;
    c.cutoff = cutoff;
    c.skin = skin;
    c.short_max_stale = true;
    c.split_slots = -1;          // an external list: slots follow user order
    c.center_slots = -1;
    ++c.list_version;
    tsf::snapshot_reference_positions(c);
    c.adopted_id = id;
    c.adopted_valid = true;
  });
}

int tsf_needs_rebuild(tsf_ctx* ctx, int* out) {
  return guard(&ctx->c, [&] { *out = tsf::list_needs_rebuild(ctx->c) ? 1 : 0; });
}

int64_t tsf_neighbor_entries(tsf_ctx* ctx, int which) {
  int64_t total = -1;
  const int rc = guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    const tsf::ListState& s = list_for(c, which);
    std::vector<int> cnt(std::size_t(c.n));
    if (c.n > 0) {
      TSF_CUDA(cudaMemcpyAsync(cnt.data(), s.cnt.get(), sizeof(int) * c.n,
                               cudaMemcpyDeviceToHost, c.stream));
      TSF_CUDA(cudaStreamSynchronize(c.stream));
    }
    total = 0;
    for (int v : cnt) total += v;
  });
  return rc == TSF_OK ? total : -int64_t(rc);
}

int tsf_export_neighbors(tsf_ctx* ctx, int which, int32_t* offsets, int32_t* nbrs, int64_t cap) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    const tsf::ListState& s = list_for(c, which);
    std::vector<int> cnt;
    const std::vector<int> ell = download_ell(c, s, cnt);
    // slot space -> user indices; segments ascending by user index
    // (neighbor.cpp:114; the filter keeps that order, neighbor.cpp:143-152)
    std::vector<int> perm(std::size_t(c.n)), slot_of(std::size_t(c.n));
    if (c.sorted && c.n > 0) {
      TSF_CUDA(cudaMemcpyAsync(perm.data(), c.perm.get(), sizeof(int) * c.n,
                               cudaMemcpyDeviceToHost, c.stream));
      TSF_CUDA(cudaStreamSynchronize(c.stream));
    } else {
      for (std::int64_t q = 0; q < c.n; ++q) perm[std::size_t(q)] = int(q);
    }
    for (std::int64_t q = 0; q < c.n; ++q) slot_of[std::size_t(perm[std::size_t(q)])] = int(q);
    std::int64_t w = 0;
    offsets[0] = 0;
    for (std::int64_t u = 0; u < c.n; ++u) {
      const int a = slot_of[std::size_t(u)];
      const int m = cnt[std::size_t(a)];
      if (w + m > cap) throw tsf::ConfigError("neighbor export buffer too small");
      for (int q = 0; q < m; ++q) nbrs[w + q] = perm[std::size_t(ell[tsf::ell_at(q, a, c.npad)])];
      std::sort(nbrs + w, nbrs + w + m);
      w += m;
      offsets[u + 1] = int32_t(w);
    }
  });
}

int tsf_compute_f64(tsf_ctx* ctx, uint32_t flags, double* e, double* f, double* w) {
  return compute_entry(ctx, tsf::Precision::F64, flags, e, f, w);
}
int tsf_compute_mixed(tsf_ctx* ctx, uint32_t flags, double* e, double* f, double* w) {
  return compute_entry(ctx, tsf::Precision::Mixed, flags, e, f, w);
}
int tsf_compute_f32(tsf_ctx* ctx, uint32_t flags, double* e, double* f, double* w) {
  return compute_entry(ctx, tsf::Precision::F32, flags, e, f, w);
}

int tsf_evaluate_forces(tsf_ctx* ctx, int precision, int64_t n, const double* xyz,
                        const int32_t* species, const double box[3], const uint8_t periodic[3],
                        double skin, uint32_t flags, double* energy, double* forces,
                        double* virial) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (precision < 0 || precision > 2) throw tsf::ConfigError("unknown precision selector");
    set_system(c, n, xyz, species, box, periodic);
    if (!c.skin_list.valid || c.skin != skin || c.cutoff != c.params.r_cut_max() ||
        tsf::list_needs_rebuild(c))
      tsf::list_build(c, c.params.r_cut_max(), skin);
    evaluate(c, tsf::Precision(precision), virial ? flags : flags | tsf::kFlagNoVirial);
    finish(c, energy, forces, virial);
  });
}

/* ---- MD ---- */
int tsf_md_set_state(tsf_ctx* ctx, const double* vel, const double* masses) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    const int s = c.params.species_count();
    for (int q = 0; q < s; ++q)
      if (!(masses[q] > 0.0))
        throw tsf::ConfigError("species " + std::to_string(q) + " has non-positive mass");
    c.masses.assign(masses, masses + s);
    const std::size_t m = 3 * std::size_t(c.n);
    if (m == 0) return;
    tsf::ensure_pinned(c, m);
    std::memcpy(c.pinned, vel, m * sizeof(double));
    TSF_CUDA(cudaMemcpyAsync(c.xyz_stage.get(), c.pinned, m * sizeof(double),
                             cudaMemcpyHostToDevice, c.stream));
    tsf::pack_velocities(c);
    TSF_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int tsf_md_get_state(tsf_ctx* ctx, double* xyz, double* vel) {
  const int rc = xyz ? tsf_get_positions(ctx, xyz) : TSF_OK;
  if (rc != TSF_OK || !vel) return rc;
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    const std::size_t m = 3 * std::size_t(c.n);
    if (m == 0) return;
    tsf::ensure_pinned(c, m);
    tsf::unpack_velocities(c);
    TSF_CUDA(cudaMemcpyAsync(c.pinned, c.xyz_stage.get(), m * sizeof(double),
                             cudaMemcpyDeviceToHost, c.stream));
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    std::memcpy(vel, c.pinned, m * sizeof(double));
  });
}

int tsf_md_scale_velocities(tsf_ctx* ctx, double factor) {
  return guard(&ctx->c, [&] {
    if (!(factor >= 0.0)) throw tsf::ConfigError("velocity scale must be non-negative");
    tsf::md_scale_velocities(ctx->c, factor);
  });
}

int tsf_md_kick(tsf_ctx* ctx, double dt, int drift, int kicks, int* moved) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (!(dt > 0.0)) throw tsf::ConfigError("dt must be positive");
    if (kicks != 1 && kicks != 2) throw tsf::ConfigError("kicks must be 1 or 2");
    if (c.masses.empty()) throw tsf::ConfigError("call tsf_md_set_state before tsf_md_kick");
    const bool check = drift && moved && c.skin_list.valid;
    tsf::md_kick(c, dt, drift != 0, kicks, check);
    if (drift) c.forces_current = false;
    if (moved) {
      int f = 0;
      if (check)
        TSF_CUDA(cudaMemcpyAsync(&f, c.flags.get() + tsf::kFlagMoved, sizeof(int), cudaMemcpyDeviceToHost,
                                 c.stream));
      TSF_CUDA(cudaStreamSynchronize(c.stream));
      *moved = check ? f : 1;   // no list: a build is due anyway
    }
  });
}

int tsf_md_kinetic(tsf_ctx* ctx, double* ke) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (c.masses.empty()) throw tsf::ConfigError("call tsf_md_set_state before tsf_md_kinetic");
    double v = 0.0;
    if (c.n > 0) {
      tsf::md_kinetic(c);
      TSF_CUDA(cudaMemcpyAsync(&v, c.result.get() + 7, sizeof(double), cudaMemcpyDeviceToHost,
                               c.stream));
      TSF_CUDA(cudaStreamSynchronize(c.stream));
    }
    *ke = v;
  });
}

int tsf_md_run(tsf_ctx* ctx, int precision, int64_t steps, double dt, uint32_t flags,
               int thermo_every, double* thermo, int64_t cap, int64_t* nsamples,
               int64_t* rebuilds) {
  return guard(&ctx->c, [&] {
    Ctx& c = ctx->c;
    if (precision < 0 || precision > 2) throw tsf::ConfigError("unknown precision selector");
    if (steps < 0) throw tsf::ConfigError("steps must be non-negative");
    if (!(dt > 0.0)) throw tsf::ConfigError("dt must be positive");
    if (thermo_every < 1) throw tsf::ConfigError("thermo interval must be at least 1");
    if (!c.skin_list.valid)
      throw tsf::ConfigError("no neighbor list: build one before running dynamics");
    const tsf::Precision p = tsf::Precision(precision);
    flags |= tsf::kFlagNoVirial;   // thermo samples read energies only
    std::int64_t ns = 0, nreb = 0;
    auto sample = [&](std::int64_t step) {
      tsf::md_kinetic(c);
      double res[8];
      TSF_CUDA(cudaMemcpyAsync(res, c.result.get(), 8 * sizeof(double), cudaMemcpyDeviceToHost,
                               c.stream));
      raise_device_errors(c);
      if (thermo && ns < cap) {
        thermo[3 * ns] = double(step);
        thermo[3 * ns + 1] = res[0];
        thermo[3 * ns + 2] = res[7];
      }
      ++ns;
    };
    if (!c.forces_current) evaluate(c, p, flags);
    sample(0);
    // velocity Verlet (engine.cpp:142-172).  The closing half-kick of a step
    // is deferred into the next step's opening kick + drift (one pass over
    // the atoms instead of two) unless a sample needs full-step velocities.
    // Speculative: the evaluation is queued behind the kick before the host
    // knows the kick's needs_rebuild result; only the 4-byte flag is awaited
    // (an event right after the kick), so the GPU runs step s's evaluation
    // while the host decides and queues step s+1.  A stale list (a rebuild
    // step, every ~20 steps at 1600 K) makes that evaluation's launches return
    // at once; the step is then rebuilt and evaluated again — the reference's
    // rebuild schedule and results (neighbor.cpp:134-141, engine.cpp:174-199).
    if (!c.pinned_flag)
      TSF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c.pinned_flag), 64,
                             cudaHostAllocDefault));
    if (!c.flag_event) TSF_CUDA(cudaEventCreateWithFlags(&c.flag_event, cudaEventDisableTiming));
    struct Spec {
      Ctx& c;
      explicit Spec(Ctx& cc) : c(cc) { c.speculative = !c.profile; }
      ~Spec() { c.speculative = false; }
    } spec(c);
    auto clear_moved = [&] {
      TSF_CUDA(cudaMemsetAsync(c.flags.get() + tsf::kFlagMoved, 0, sizeof(int), c.stream));
      TSF_CUDA(cudaMemsetAsync(c.flags.get() + tsf::kFlagMovedAny, 0, 2 * sizeof(int), c.stream));
    };
    clear_moved();
    // Multi-step segments: up to TSF_MD_SEGMENT steps (default 8, never past
    // a thermo sample) are queued — and, once the evaluation replays from its
    // graph, captured and replayed as ONE graph — before the host looks at
    // the flags.  A kick that moves an atom past skin/2 records its step;
    // every later launch of the segment returns at once (k_reduce folds the
    // step's flag into kFlagMovedAny, which the next kick reads), so the
    // state stops at that step: the host rebuilds, re-evaluates it and
    // resumes after it.
    const char* seg_env = std::getenv("TSF_MD_SEGMENT");
    const int seg_max = std::max(1, seg_env ? std::atoi(seg_env) : 8);
    bool kick_pending = false;
    for (std::int64_t s = 1; s <= steps;) {
      const std::int64_t sample_at =
          std::min<std::int64_t>(steps, (s + thermo_every - 1) / thermo_every * thermo_every);
      const std::int64_t e = std::min<std::int64_t>(sample_at, s + seg_max - 1);
      const int first_kicks = kick_pending ? 2 : 1;
      auto segment = [&] {
        for (std::int64_t t = s; t <= e; ++t) {
          tsf::md_kick(c, dt, true, t == s ? first_kicks : 2, /*check_rebuild=*/true, int(t - s));
          evaluate(c, p, flags);
        }
      };
      const std::uint64_t key[6] = {
          c.list_version, std::uint64_t(p) | (std::uint64_t(e - s + 1) << 8) |
                              (std::uint64_t(first_kicks) << 24),
          flags | 0x80000000u, std::uint64_t(c.n), std::uint64_t(c.n_owned),
          std::uint64_t(reinterpret_cast<std::uintptr_t>(c.stream))};
      if (c.seg_dt != dt && c.graph[3].exec) {   // the kick nodes carry dt
        TSF_CUDA(cudaGraphExecDestroy(c.graph[3].exec));
        c.graph[3].exec = nullptr;
      }
      c.seg_dt = dt;
      run_segment(c, key, c.speculative && evaluate_replays(c, p, flags), segment);
      TSF_CUDA(cudaMemcpyAsync(c.pinned_flag, c.flags.get() + tsf::kFlagMovedAny,
                               2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      TSF_CUDA(cudaEventRecord(c.flag_event, c.stream));
      TSF_CUDA(cudaEventSynchronize(c.flag_event));
      std::int64_t done = e;
      if (c.pinned_flag[0]) {
        // the segment stopped after the kick of step s + pinned_flag[1]
        done = s + c.pinned_flag[1];
        clear_moved();
        tsf::list_build(c, c.cutoff, c.skin);
        ++nreb;
        evaluate(c, p, flags);
      }
      kick_pending = true;
      s = done + 1;
      if (done == sample_at) {
        tsf::md_kick(c, dt, false);
        sample(done);
        kick_pending = false;
      }
    }
    if (nsamples) *nsamples = ns;
    if (rebuilds) *rebuilds = nreb;
  });
}

}  // extern "C"
