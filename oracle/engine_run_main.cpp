// TEST / MEASUREMENT INFRASTRUCTURE ONLY.  tmd::Engine::run (engine.cpp:174-199)
// on BASELINE cfg 2 — 20x20x10 Si cells (32,000 atoms), init_velocities(1600 K,
// seed 12345), dt 1 fs, skin 1 A, rebuild check every step — built twice by
// oracle/Makefile from the unmodified reference sources:
//   engine_run_cpu   the stock evaluate_forces (potential_opt.cpp), all host threads
//   engine_run_b200  the same Engine with integration/potential_b200.cpp as
//                    evaluate_forces: every force pass runs on the B200
// Prints one JSON line: steps, wall seconds of the step loop, atom-steps/s,
// ns/day, Etot at step 0 and at the end, rebuilds.
//   engine_run_{cpu,b200} [steps] [precision opt-d|opt-m|opt-s] [workers]
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>

#include "tmd/engine.hpp"
#include "tmd/params.hpp"

int main(int argc, char** argv) {
  const long steps = argc > 1 ? std::atol(argv[1]) : 100;
  const std::string prec = argc > 2 ? argv[2] : "opt-d";
  const int workers = argc > 3 ? std::atoi(argv[3])
                               : int(std::max(1u, std::thread::hardware_concurrency()));
  tmd::AtomSystem sys = tmd::make_diamond_lattice(20, 20, 10, 5.431, 0, 28.0855);
  tmd::init_velocities(sys, 1600.0, 12345);
  tmd::RunConfig cfg;
  cfg.steps = steps;
  cfg.dt = 0.001;
  cfg.skin = 1.0;
  cfg.workers = workers;
  cfg.thermo_every = 10;
  cfg.precision = prec == "opt-m"   ? tmd::PrecisionMode::OptM
                  : prec == "opt-s" ? tmd::PrecisionMode::OptS
                                    : tmd::PrecisionMode::OptD;
  tmd::Engine engine(sys, tmd::builtin_silicon(), cfg);
  const tmd::RunReport rep = engine.run();
  const double n = double(sys.size());
  std::printf(
      "{\"steps\": %ld, \"natoms\": %.0f, \"precision\": \"%s\", \"workers\": %d, "
      "\"wall_s\": %.6f, \"atom_steps_per_s\": %.6e, \"ns_per_day\": %.4f, "
      "\"etot_first\": %.17g, \"etot_last\": %.17g, \"rebuilds\": %d}\n",
      steps, n, prec.c_str(), workers, rep.wall_seconds,
      rep.wall_seconds > 0 ? n * double(steps) / rep.wall_seconds : 0.0, rep.ns_per_day,
      rep.samples.front().etot_ev, rep.samples.back().etot_ev, engine.neighbor_rebuilds());
  return 0;
}
