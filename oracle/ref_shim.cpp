// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (/root/reference/proj),
// compiled from the reference sources where they lie by oracle/Makefile into
// oracle/_ref/libtmdref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, as the checker
// and as the timed CPU baseline ("kind": "reference").
//
// Each entry point forwards to the reference's own public API:
//   tmdref_params_*        -> parse_param_text / ParamTable      (params.hpp:40-75)
//   tmdref_system_*        -> AtomSystem / SimulationBox          (system.hpp:14-27, box.hpp:11-24)
//   tmdref_list_*          -> build_neighbor_list, needs_rebuild, filter_all_segments
//                                                                 (neighbor.hpp:31-54)
//   tmdref_compute_ref     -> compute_ref                          (potential_ref.hpp:51-52)
//   tmdref_evaluate        -> evaluate_forces                      (potential_opt.hpp:105-106)
//   tmdref_diamond_lattice / tmdref_perturbed_lattice / tmdref_init_velocities
//                          -> engine.hpp:54-60, verify.hpp:24-25
//   tmdref_run_nve         -> Engine::run                          (engine.hpp:63-93)
//
// Return codes mirror the reference CLI (tools/main.cpp:241-256):
// 0 ok, 2 config/parse error, 3 numeric error, 1 anything else.

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tmd/engine.hpp"
#include "tmd/error.hpp"
#include "tmd/neighbor.hpp"
#include "tmd/params.hpp"
#include "tmd/potential_opt.hpp"
#include "tmd/potential_ref.hpp"
#include "tmd/system.hpp"
#include "tmd/verify.hpp"

using namespace tmd;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void copy_vec3(const std::vector<Vec3>& v, double* out) {
  for (std::size_t a = 0; a < v.size(); ++a) {
    out[3 * a + 0] = v[a].x;
    out[3 * a + 1] = v[a].y;
    out[3 * a + 2] = v[a].z;
  }
}

}  // namespace

extern "C" {

const char* tmdref_last_error() { return g_err.c_str(); }

/* ---- parameters ---- */
int tmdref_params_parse(const char* text, ParamTable** out) {
  return guarded([&] { *out = new ParamTable(parse_param_text(text, "<string>")); });
}
int tmdref_params_builtin_silicon(ParamTable** out) {
  return guarded([&] { *out = new ParamTable(builtin_silicon()); });
}
double tmdref_params_r_cut_max(const ParamTable* p) { return p->r_cut_max(); }
int tmdref_params_species_count(const ParamTable* p) { return p->species_count(); }
void tmdref_params_free(ParamTable* p) { delete p; }

/* ---- systems ---- */
int tmdref_system_new(int64_t n, const double* xyz, const int32_t* species,
                      int nmass, const double* masses, const double* box,
                      const uint8_t* periodic, AtomSystem** out) {
  return guarded([&] {
    auto* s = new AtomSystem;
    s->positions.resize(std::size_t(n));
    for (int64_t a = 0; a < n; ++a)
      s->positions[std::size_t(a)] = {xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]};
    s->velocities.assign(std::size_t(n), Vec3{});
    s->forces.assign(std::size_t(n), Vec3{});
    s->species.assign(species, species + n);
    s->species_masses.assign(masses, masses + nmass);
    s->box = {box[0], box[1], box[2], periodic[0] != 0, periodic[1] != 0,
              periodic[2] != 0};
    *out = s;
  });
}
void tmdref_system_free(AtomSystem* s) { delete s; }
int64_t tmdref_system_size(const AtomSystem* s) { return int64_t(s->size()); }
void tmdref_system_get(const AtomSystem* s, double* xyz, double* vel,
                       int32_t* species, double* box, uint8_t* periodic) {
  if (xyz) copy_vec3(s->positions, xyz);
  if (vel) copy_vec3(s->velocities, vel);
  if (species) std::memcpy(species, s->species.data(), s->species.size() * 4);
  if (box) {
    box[0] = s->box.lx;
    box[1] = s->box.ly;
    box[2] = s->box.lz;
  }
  if (periodic) {
    periodic[0] = s->box.periodic_x;
    periodic[1] = s->box.periodic_y;
    periodic[2] = s->box.periodic_z;
  }
}
void tmdref_system_set_positions(AtomSystem* s, const double* xyz) {
  for (std::size_t a = 0; a < s->size(); ++a)
    s->positions[a] = {xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]};
}
void tmdref_system_set_velocities(AtomSystem* s, const double* v) {
  for (std::size_t a = 0; a < s->size(); ++a)
    s->velocities[a] = {v[3 * a], v[3 * a + 1], v[3 * a + 2]};
}

/* ---- generators ---- */
int tmdref_diamond_lattice(int nx, int ny, int nz, double a0, int32_t species_id,
                           double mass, AtomSystem** out) {
  return guarded([&] {
    *out = new AtomSystem(make_diamond_lattice(nx, ny, nz, a0, species_id, mass));
  });
}
int tmdref_perturbed_lattice(const ParamTable* p, int cells, double jitter,
                             uint64_t seed, AtomSystem** out) {
  return guarded([&] { *out = new AtomSystem(perturbed_lattice(*p, cells, jitter, seed)); });
}
int tmdref_init_velocities(AtomSystem* s, double temperature, uint64_t seed) {
  return guarded([&] { init_velocities(*s, temperature, seed); });
}

/* ---- neighbor lists ---- */
int tmdref_list_build(const AtomSystem* s, double cutoff, double skin, NeighborList** out) {
  return guarded([&] { *out = new NeighborList(build_neighbor_list(*s, cutoff, skin)); });
}
void tmdref_list_free(NeighborList* l) { delete l; }
int64_t tmdref_list_entries(const NeighborList* l) { return int64_t(l->neighbors.size()); }
void tmdref_list_export(const NeighborList* l, int32_t* offsets, int32_t* nbrs) {
  std::memcpy(offsets, l->offsets.data(), l->offsets.size() * 4);
  std::memcpy(nbrs, l->neighbors.data(), l->neighbors.size() * 4);
}
int tmdref_needs_rebuild(const NeighborList* l, const AtomSystem* s) {
  return needs_rebuild(*l, *s) ? 1 : 0;
}
// Short list (paper Sec. 4.4 filter): writes offsets (n+1) and returns the
// entry count; nbrs may be null to query the size.
int64_t tmdref_filter(const NeighborList* l, const AtomSystem* s, double r_cut_max,
                      int apply, int32_t* offsets, int32_t* nbrs) {
  const PackedSegments p = filter_all_segments(*l, *s, r_cut_max, apply != 0);
  if (offsets) std::memcpy(offsets, p.offsets.data(), p.offsets.size() * 4);
  if (nbrs) std::memcpy(nbrs, p.indices.data(), p.indices.size() * 4);
  return int64_t(p.indices.size());
}

/* ---- force evaluation ---- */
int tmdref_compute_ref(const AtomSystem* s, const NeighborList* l, const ParamTable* p,
                       double* energy, double* forces) {
  return guarded([&] {
    const EnergyForces ef = compute_ref(*s, *l, *p);
    *energy = ef.energy;
    if (forces) copy_vec3(ef.forces, forces);
  });
}
int tmdref_evaluate(const AtomSystem* s, const NeighborList* l, const ParamTable* p,
                    const char* scheme, const char* precision, int width, int k_max,
                    int workers, int filter, double* energy, double* forces) {
  return guarded([&] {
    ForceOptions o;
    o.scheme = scheme_from_string(scheme);
    o.precision = precision_from_string(precision);
    o.width = width;
    o.k_max = k_max;
    o.workers = workers;
    o.filter = filter != 0;
    const EnergyForces ef = evaluate_forces(*s, *l, *p, o);
    *energy = ef.energy;
    if (forces) copy_vec3(ef.forces, forces);
  });
}
int tmdref_fd_forces(const AtomSystem* s, const NeighborList* l, const ParamTable* p,
                     double h, double* forces) {
  return guarded([&] { copy_vec3(fd_force_oracle(*s, *l, *p, h), forces); });
}

/* ---- NVE engine (caller of the path; used for the cfg-2 CPU baseline) ---- */
int tmdref_run_nve(const AtomSystem* s, const ParamTable* p, long steps, double dt,
                   double skin, const char* scheme, const char* precision, int width,
                   int workers, int thermo_every, double* wall_seconds,
                   double* etot_first, double* etot_last, int* rebuilds,
                   AtomSystem** final_state) {
  return guarded([&] {
    RunConfig cfg;
    cfg.steps = steps;
    cfg.dt = dt;
    cfg.skin = skin;
    cfg.scheme = scheme_from_string(scheme);
    cfg.precision = precision_from_string(precision);
    cfg.width = width;
    cfg.workers = workers;
    cfg.thermo_every = thermo_every;
    Engine engine(*s, *p, cfg);
    const RunReport rep = engine.run();
    *wall_seconds = rep.wall_seconds;
    *etot_first = rep.samples.front().etot_ev;
    *etot_last = rep.samples.back().etot_ev;
    *rebuilds = engine.neighbor_rebuilds();
    if (final_state) *final_state = new AtomSystem(engine.system());
  });
}

}  // extern "C"
