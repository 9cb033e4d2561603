// Drop-in B200 `tmd::evaluate_forces` for the reference.
//
// Link-time replacement of evaluate_forces (proj/include/tmd/potential_opt.hpp:105-106,
// proj/src/potential_opt.cpp:104-138): build the reference with
// potential_opt.cpp compiled as `-Devaluate_forces=evaluate_forces_cpu` and
// link this file and libtersoff_b200.so (oracle/Makefile target `refverify`
// does exactly that).  Every caller — Engine::compute_forces
// (engine.cpp:136-140), the verification battery (verify.cpp), the CLI and the
// Python module — then runs on the GPU without a source change.
//
// Semantics kept from the reference:
//   * the option checks and error messages of potential_opt.cpp:106-121;
//   * Scheme::Ref and Scheme::ScalarOpt are the reference's exact CPU schemes
//     (compute_ref / compute_opt_scalar) and stay on the CPU;
//   * V1 / V2 / V3 / Auto run on the B200 in the requested precision
//     (OptD/Ref -> f64, OptM -> mixed, OptS -> f32), deterministic scatter —
//     re-evaluations are bitwise identical, as verify.cpp's determinism check
//     requires; `filter` maps to TSF_NO_FILTER; width / k_max / workers have
//     no GPU meaning beyond their validation.
#include <cstdint>
#include <memory>
#include <string>

#include "../include/tersoff_b200.h"
#include "tmd/error.hpp"
#include "tmd/params.hpp"
#include "tmd/potential_opt.hpp"
#include "tmd/potential_ref.hpp"

namespace tmd {

EnergyForces evaluate_forces_cpu(const AtomSystem& sys, const NeighborList& list,
                                 const ParamTable& params, const ForceOptions& opt);

namespace {

// One device context per thread, re-created when the parameter table changes
// (the reference's evaluate_forces is re-entrant; a context is not).
struct GpuContext {
  tsf_params* params = nullptr;
  tsf_ctx* ctx = nullptr;
  std::string table;
  ~GpuContext() { reset(); }
  void reset() {
    if (ctx) tsf_destroy(ctx);
    if (params) tsf_params_free(params);
    ctx = nullptr;
    params = nullptr;
  }
};

void check(int rc, const tsf_ctx* ctx) {
  if (rc == TSF_OK) return;
  const std::string msg = tsf_last_error(ctx);
  if (rc == TSF_ERR_NUMERIC) throw NumericError(msg);
  throw ConfigError(msg);
}

tsf_ctx* context_for(const ParamTable& params) {
  thread_local GpuContext g;
  std::string text = serialize_param_table(params);
  if (!g.ctx || g.table != text) {
    g.reset();
    if (tsf_params_parse(text.data(), text.size(), "<ParamTable>", &g.params) != TSF_OK)
      throw ParseError(tsf_error_message());
    if (tsf_create(g.params, /*device=*/0, &g.ctx) != TSF_OK)
      throw ConfigError(tsf_error_message());
    g.table = std::move(text);
  }
  return g.ctx;
}

}  // namespace

EnergyForces evaluate_forces(const AtomSystem& sys, const NeighborList& list,
                             const ParamTable& params, const ForceOptions& opt) {
  // option handling of potential_opt.cpp:106-121
  if (opt.k_max < 0) throw ConfigError("k_max must be non-negative");
  if (opt.workers < 1) throw ConfigError("worker count must be at least 1");
  const int width = opt.width > 0 ? opt.width : default_width(opt.precision);
  Scheme scheme = opt.scheme;
  if (opt.precision == PrecisionMode::Ref && scheme == Scheme::Auto) scheme = Scheme::Ref;
  if (scheme == Scheme::Auto) scheme = select_scheme(width, opt.precision);
  if (scheme == Scheme::Ref || scheme == Scheme::ScalarOpt)
    return evaluate_forces_cpu(sys, list, params, opt);   // the exact CPU schemes
  const int eff_width = scheme == Scheme::V3 ? 1 : width;
  if (eff_width != 1 && eff_width != 4 && eff_width != 8 && eff_width != 16)
    throw ConfigError("unsupported backend width " + std::to_string(width) +
                      " (supported: 1, 4, 8, 16)");

  tsf_ctx* ctx = context_for(params);
  const std::size_t n = sys.size();
  const double box[3] = {sys.box.lx, sys.box.ly, sys.box.lz};
  const std::uint8_t per[3] = {std::uint8_t(sys.box.periodic_x), std::uint8_t(sys.box.periodic_y),
                               std::uint8_t(sys.box.periodic_z)};
  EnergyForces out;
  out.forces.resize(n);
  // std::vector<Vec3> is AoS double[n][3] (vec3.hpp), the C-ABI's layout
  const double* xyz = n ? &sys.positions[0].x : nullptr;
  check(tsf_set_system(ctx, std::int64_t(n), xyz, sys.species.data(), box, per), ctx);
  check(tsf_set_neighbor_list(ctx, list.offsets.data(), list.neighbors.data(),
                              list.build_cutoff - list.skin, list.skin),
        ctx);
  const std::uint32_t flags = TSF_DETERMINISTIC | (opt.filter ? 0u : TSF_NO_FILTER);
  double* f = n ? &out.forces[0].x : nullptr;
  switch (opt.precision) {
    case PrecisionMode::OptS: check(tsf_compute_f32(ctx, flags, &out.energy, f, nullptr), ctx); break;
    case PrecisionMode::OptM: check(tsf_compute_mixed(ctx, flags, &out.energy, f, nullptr), ctx); break;
    default: check(tsf_compute_f64(ctx, flags, &out.energy, f, nullptr), ctx); break;
  }
  return out;
}

}  // namespace tmd
