/* tersoff_b200.h — C-ABI of the B200-native Tersoff force/energy path.
 *
 * Drop-in boundary for the reference's force path
 *   tmd::evaluate_forces(const AtomSystem&, const NeighborList&,
 *                        const ParamTable&, const ForceOptions&) -> EnergyForces
 *   (/root/reference/proj/include/tmd/potential_opt.hpp:105-106,
 *    /root/reference/proj/src/potential_opt.cpp:104-138)
 * and the neighbor-list routines it consumes
 *   (/root/reference/proj/include/tmd/neighbor.hpp:31-54).
 *
 * Plain pointers and sizes only.  Host arrays are owned by the caller.
 * Positions/forces are AoS double[n][3] exactly like std::vector<Vec3>
 * (vec3.hpp:9-37); species are int32 (system.hpp:19).
 *
 * Return codes mirror the reference's error taxonomy and CLI exit codes
 * (error.hpp:9-21, tools/main.cpp:241-256):
 *   TSF_OK 0, TSF_ERR_CONFIG 2 (ConfigError/ParseError), TSF_ERR_NUMERIC 3
 *   (NumericError), plus TSF_ERR_CUDA 4 and TSF_ERR_INTERNAL 1.
 * The message of the last failure is available through tsf_last_error(ctx)
 * or, for calls without a context, tsf_error_message().
 *
 * Threading: one CUDA stream per context; a context must not be used from
 * two threads at once.  Distinct contexts are independent.
 */
#ifndef TERSOFF_B200_H
#define TERSOFF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSF_OK 0
#define TSF_ERR_INTERNAL 1
#define TSF_ERR_CONFIG 2
#define TSF_ERR_NUMERIC 3
#define TSF_ERR_CUDA 4

/* compute flags */
#define TSF_DETERMINISTIC 0x1u /* slot buffers + reverse gather: bitwise reproducible  */
#define TSF_NO_FILTER 0x2u     /* ForceOptions::filter = false (potential_opt.hpp:35) */
#define TSF_NO_VIRIAL 0x4u     /* the virial is not formed (result[1..6] stay zero)     */

/* neighbor-list selectors for tsf_export_neighbors */
#define TSF_LIST_SKIN 0  /* NeighborList (neighbor.hpp:15-27)              */
#define TSF_LIST_SHORT 1 /* filter_all_segments output (neighbor.hpp:46-54) */

typedef struct tsf_params tsf_params;
typedef struct tsf_ctx tsf_ctx;

/* ---- errors ------------------------------------------------------------ */
const char* tsf_error_message(void);          /* thread-local, context-free calls */
const char* tsf_last_error(const tsf_ctx* ctx);
const char* tsf_version(void);

/* ---- parameter table (host only; no GPU needed) -------------------------
 * Replaces parse_param_text / load_param_file / builtin_silicon /
 * serialize_param_table (params.hpp:62-75, params.cpp:119-234). */
int tsf_params_parse(const char* text, size_t len, const char* source_name, tsf_params** out);
int tsf_params_load(const char* path, tsf_params** out);
int tsf_params_builtin_silicon(tsf_params** out);
void tsf_params_free(tsf_params* p);
int tsf_params_species_count(const tsf_params* p);
const char* tsf_params_species_name(const tsf_params* p, int species);
int tsf_params_species_id(const tsf_params* p, const char* name); /* -1 when unknown */
double tsf_params_r_cut_max(const tsf_params* p);
/* FlatParams<double> rows (params.hpp:88-115): S^3 rows of 16 doubles. */
int tsf_params_flat_rows(const tsf_params* p, double* rows, size_t cap);
/* round-trip-exact text; returns the length (excluding NUL), writes at most cap bytes. */
int64_t tsf_params_serialize(const tsf_params* p, char* buf, size_t cap);

/* ---- synthetic inputs (host) --------------------------------------------
 * make_diamond_lattice (engine.hpp:54-55, engine.cpp:28-58),
 * perturbed_lattice (verify.hpp:24-25, verify.cpp:83-104),
 * init_velocities (engine.hpp:60, engine.cpp:64-116); bit-identical. */
int64_t tsf_diamond_lattice_size(int nx, int ny, int nz);
int tsf_make_diamond_lattice(int nx, int ny, int nz, double a0, int32_t species_id,
                             double* xyz, int32_t* species, double* box);
int tsf_perturbed_lattice(const tsf_params* p, int cells, double jitter, uint64_t seed,
                          double* xyz, int32_t* species, double* masses /* S */, double* box);
int tsf_init_velocities(int64_t n, const int32_t* species, const double* masses,
                        double temperature, uint64_t seed, double* vel);

/* ---- on-disk snapshots (fixtures for thermal and liquid states) ---------
 * SURVEY.md 8f row 4; the reference regenerates fixtures from seeds
 * (engine.cpp:28-116, verify.cpp:83-104) and has no file format.  Layout in
 * csrc/tsf_snapshot.cpp: header, masses, coordinates (float64, or float32
 * with TSF_SNAP_F32_COORDS — the stored state is then the float32-rounded
 * one), uint8 species, optional velocities, SHA-256 trailer of every byte
 * before it.  Readers verify the checksum (TSF_ERR_CONFIG on mismatch). */
#define TSF_SNAP_F32_COORDS 0x1u
#define TSF_SNAP_VELOCITIES 0x2u
int tsf_snapshot_write(const char* path, int64_t n, const double* xyz, const int32_t* species,
                       int nspecies, const double* masses, const double box[3],
                       const uint8_t periodic[3], const double* vel /* NULL unless flagged */,
                       uint32_t flags, uint8_t sha256_out[32] /* may be NULL */);
int tsf_snapshot_info(const char* path, int64_t* n, int* nspecies, uint32_t* flags,
                      uint8_t sha256_out[32] /* may be NULL */);
/* any output may be NULL; vel is zero-filled when the file has none */
int tsf_snapshot_read(const char* path, double* xyz, int32_t* species, double* masses,
                      double box[3], uint8_t periodic[3], double* vel);

/* ---- device context -------------------------------------------------- */
/* p may be NULL: a list-only context (neighbor lists and rebuild checks, no
 * force evaluation), for build_neighbor_list, which takes no parameters. */
int tsf_create(const tsf_params* p, int device, tsf_ctx** out);
void tsf_destroy(tsf_ctx* ctx);
void* tsf_stream(tsf_ctx* ctx); /* the context's cudaStream_t */

/* AtomSystem upload (system.hpp:14-27): positions, species, box.  Species ids
 * must lie in [0, S).  Invalidates the neighbor list when n changes. */
int tsf_set_system(tsf_ctx* ctx, int64_t n, const double* xyz, const int32_t* species,
                   const double box[3], const uint8_t periodic[3]);
int tsf_set_positions(tsf_ctx* ctx, const double* xyz);
int tsf_get_positions(tsf_ctx* ctx, double* xyz);

/* build_neighbor_list (neighbor.hpp:31, neighbor.cpp:37-132) on the device. */
int tsf_build_neighbor_list(tsf_ctx* ctx, double cutoff, double skin);
/* Adopt an externally built NeighborList (CSR offsets[n+1], neighbors). */
int tsf_set_neighbor_list(tsf_ctx* ctx, const int32_t* offsets, const int32_t* nbrs,
                          double cutoff, double skin);
/* needs_rebuild (neighbor.hpp:35, neighbor.cpp:134-141): *out = 0/1. */
int tsf_needs_rebuild(tsf_ctx* ctx, int* out);
/* Entry count of a list (TSF_LIST_SKIN or TSF_LIST_SHORT; the short list is
 * refreshed from the current positions, as filter_all_segments does). */
int64_t tsf_neighbor_entries(tsf_ctx* ctx, int which);
int tsf_export_neighbors(tsf_ctx* ctx, int which, int32_t* offsets, int32_t* nbrs, int64_t cap);

/* ---- force evaluation (evaluate_forces), precision fixed per symbol -----
 * f64:   double compute, double accumulation          (PrecisionMode::OptD)
 * mixed: float compute, double accumulation           (PrecisionMode::OptM)
 * f32:   float compute, float per-atom accumulation    (PrecisionMode::OptS)
 * Any of energy / forces (n*3) / virial (6: xx yy zz xy xz yz) may be NULL;
 * results then stay on the device and the call does not synchronize.  A NULL
 * virial next to a non-NULL energy or forces skips the virial's arithmetic
 * (the device copy, tsf_results_device, then holds zeros for it); with all
 * three NULL everything is formed for tsf_results_device.  tsf_md_run and
 * tsf_evaluate_forces with a NULL virial skip it likewise. */
int tsf_compute_f64(tsf_ctx* ctx, uint32_t flags, double* energy, double* forces, double* virial);
int tsf_compute_mixed(tsf_ctx* ctx, uint32_t flags, double* energy, double* forces, double* virial);
int tsf_compute_f32(tsf_ctx* ctx, uint32_t flags, double* energy, double* forces, double* virial);

/* One-shot drop-in: upload positions (and species/box), build the list when
 * it is missing or stale, evaluate, download.  precision: 0 f64, 1 mixed, 2 f32.
 * species may be NULL on a repeat call with the same n: the resident species
 * stay (tsf_set_system accepts NULL species likewise). */
int tsf_evaluate_forces(tsf_ctx* ctx, int precision, int64_t n, const double* xyz,
                        const int32_t* species, const double box[3], const uint8_t periodic[3],
                        double skin, uint32_t flags, double* energy, double* forces,
                        double* virial);

/* Diagnostics: the device math on n host values x (current device), out[2n]:
 * fn 0 exp (constant-bank polynomial), 1 log (same), 2 libdevice exp, 3
 * libdevice log (out[2q] = f(x[q])); 4 bond order b, db/dzeta at zeta = x[q]
 * in double, 5 in float, 6 the reference's pow form in double (row (0,0,0)
 * of p; out[2q] = b, out[2q+1] = db); 7 the double bond order's path at
 * zeta = x[q] (out[2q] = 1 for the series, out[2q+1] = ln u); 8 the cutoff
 * ramp's sin(pi x), cos(pi x) for |x| <= 1/2, 9 libdevice sincospi. */
int tsf_math_probe(const tsf_params* p, int fn, int64_t n, const double* x, double* out);

/* Kernel launches issued by this context since creation (evidence counter). */
int64_t tsf_launch_count(const tsf_ctx* ctx);

/* Near-list refreshes since creation (the filter rewrote both near lists from
 * the skin list mid-life); synchronizes.  -1 on error. */
int64_t tsf_near_refreshes(tsf_ctx* ctx);

/* Per-stage CUDA-event timing of every evaluation while enabled (adds one
 * stream synchronization per evaluation).  ms[4] accumulates: filter, launch
 * setup, main force kernel, overflow + reductions + scatter gather. */
int tsf_profile_enable(tsf_ctx* ctx, int on);
int tsf_profile_read(tsf_ctx* ctx, double* ms, int64_t* calls, int reset);

/* ---- spatial domain decomposition support ----------------
 * A rank's context holds its owned atoms as user indices [0, n_owned) and
 * ghost copies after them, all in the global frame and global box.  Only
 * owned atoms act as central atoms (energy, virial, and the (i,j,k) terms
 * they own); forces land on owned and ghost atoms alike and the caller sends
 * the ghost part back to the owners.  Pointers marked d_ are device pointers
 * on the context's device; all work is ordered on the context's stream. */
/* NULL: back to the context's own (non-blocking) stream — pass a real
 * stream, not the legacy default stream's 0, to share ordering with a caller */
int tsf_set_stream(tsf_ctx* ctx, void* stream);
int tsf_set_owned(tsf_ctx* ctx, int64_t n_owned);  /* default: all atoms */
/* Ghost centers: user atoms [0, n_owned) are owned (energy, virial, MD);
 * [n_owned, n_centers) are ghosts that still act as centers, so that every
 * term putting force on an owned atom is evaluated locally and no reverse
 * force exchange is needed (their energy is their owner's).  n_owned <=
 * n_centers <= n; tsf_set_owned(n) is tsf_set_centers(n, n). */
int tsf_set_centers(tsf_ctx* ctx, int64_t n_owned, int64_t n_centers);
/* Overlap of the halo exchange with compute: user atoms [0, n_interior) are
 * owned atoms with no ghost within cutoff + skin (the caller's geometry); the
 * next list build gives them slots [0, n_interior).  Then an evaluation may
 * be split: tsf_compute_phase(.., 0) filters and computes those centres — no
 * ghost position is read, so it can run while the ghosts are in flight — and
 * tsf_compute_phase(.., 1) the rest, the tier launches and the reductions.
 * Phase 0 does nothing (and phase 1 a whole evaluation) when the list has no
 * split or the first evaluation after a build is due.  -1: off. */
int tsf_set_interior(tsf_ctx* ctx, int64_t n_interior);
int tsf_compute_phase(tsf_ctx* ctx, int precision, uint32_t flags, int phase);
/* d_xyz[m][3] = positions of user atoms d_idx[0..m) */
int tsf_gather_positions(tsf_ctx* ctx, const int32_t* d_idx, int64_t m, double* d_xyz);
/* positions of user atoms [lo, lo+m) = d_xyz[m][3] (ghost refresh) */
int tsf_scatter_positions(tsf_ctx* ctx, int64_t lo, int64_t m, const double* d_xyz);
/* d_f[m][3] = current forces of user atoms [lo, lo+m) (ghost forces) */
int tsf_gather_forces(tsf_ctx* ctx, int64_t lo, int64_t m, double* d_f);
/* forces of user atoms d_idx[0..m) += d_f[m][3] (reverse communication) */
int tsf_add_forces(tsf_ctx* ctx, const int32_t* d_idx, int64_t m, const double* d_f);
/* device copies of the latest results: d_out[0] energy, [1..6] virial; forces[n][3] user order */
int tsf_results_device(tsf_ctx* ctx, double* d_energy_virial, double* d_forces);

/* ---- spatial domain decomposition in C++  ----------------
 * One rank per GPU, x slabs of equal width (periodic x, slabs wider than two
 * ghost reaches), global frame and global box.  Each rank's context holds
 * [owned (sorted by global id) | ghosts]; ghost selection, the per-step ghost
 * position exchange, the reverse ghost-force exchange, atom migration at
 * rebuilds and the velocity-Verlet loop run on the device; the host only
 * sizes buffers at rebuilds.  Transports: NCCL (libnccl.so.2 loaded at run
 * time; rank 0 makes the unique id, the caller distributes it) or LOCAL —
 * several ranks of one process, each driven by its own host thread, sharing
 * a group (tests and per-rank projections on one GPU).
 * TSF_DD_GHOST_CENTERS: ghosts within two halos, the first layer also acts as
 * centres — one exchange per step, no reverse force exchange.
 * Errors: the return codes above; messages via tsf_dd_error_message(). */
typedef struct tsf_dd tsf_dd;
typedef struct tsf_dd_group tsf_dd_group;
#define TSF_DD_GHOST_CENTERS 0x1u
const char* tsf_dd_error_message(void);
int tsf_dd_nccl_unique_id(uint8_t* id /* 128 bytes */);
int tsf_dd_create_nccl(tsf_ctx* ctx, int world, int rank, const uint8_t* id, double cutoff,
                       double skin, const double box[3], const uint8_t periodic[3],
                       const double* masses /* S, may be NULL */, uint32_t mode, tsf_dd** out);
int tsf_dd_group_create(int world, tsf_dd_group** out);
void tsf_dd_group_destroy(tsf_dd_group* group);
int tsf_dd_create_local(tsf_ctx* ctx, tsf_dd_group* group, int rank, double cutoff, double skin,
                        const double box[3], const uint8_t periodic[3], const double* masses,
                        uint32_t mode, tsf_dd** out);
void tsf_dd_destroy(tsf_dd* dd);
/* this rank's owned atoms (host arrays, any order); vel may be NULL */
int tsf_dd_setup(tsf_dd* dd, int64_t n_owned, const int64_t* gid, const double* xyz,
                 const int32_t* species, const double* vel);
/* forward ghost exchange, evaluation, reverse exchange, energy/virial allreduce */
int tsf_dd_evaluate(tsf_dd* dd, int precision, uint32_t flags);
/* migration + ghost re-selection + list build now (collective) */
int tsf_dd_rebuild(tsf_dd* dd);
/* distributed NVE: as tsf_md_run; thermo samples are global (summed over ranks) */
int tsf_dd_md_run(tsf_dd* dd, int precision, int64_t steps, double dt, uint32_t flags,
                  int thermo_every, double* thermo, int64_t cap, int64_t* nsamples,
                  int64_t* rebuilds);
/* new positions of this rank's owned atoms (host, gid order as returned by
 * tsf_dd_results); ghosts follow at the next evaluation's exchange */
int tsf_dd_set_positions(tsf_dd* dd, const double* xyz);
/* counts[8]: owned, centres, local atoms, sent left, sent right, rebuilds,
 * atoms received by migration, ghost-centre mode */
int tsf_dd_counts(tsf_dd* dd, int64_t* counts);
/* global energy + virial (7), and this rank's owned atoms in gid order:
 * gid[n_owned], positions, forces, velocities (any pointer may be NULL) */
int tsf_dd_results(tsf_dd* dd, double* energy_virial, int64_t* gid, double* xyz, double* forces,
                   double* vel);

/* ---- GPU-resident velocity-Verlet NVE (engine.cpp:142-199) ------------- */
int tsf_md_set_state(tsf_ctx* ctx, const double* vel, const double* masses /* S */);
int tsf_md_get_state(tsf_ctx* ctx, double* xyz, double* vel);
/* Runs `steps` steps; precision as above.  Thermo every thermo_every steps
 * (and after the last): up to cap samples of (step, pe, ke) written to
 * thermo[3*s..]; *nsamples receives the count; *rebuilds the rebuild count. */
int tsf_md_run(tsf_ctx* ctx, int precision, int64_t steps, double dt, uint32_t flags,
               int thermo_every, double* thermo, int64_t cap, int64_t* nsamples,
               int64_t* rebuilds);
/* v *= factor for every atom (velocity-rescaling thermostat for fixture
 * generation, e.g. the liquid-Si melt of SURVEY.md 8d cfg 5). */
int tsf_md_scale_velocities(tsf_ctx* ctx, double factor);
/* One velocity-Verlet piece for drivers that interleave communication (the
 * slab decomposition's distributed NVE): v += F dt/(2 m mvv2e), `kicks` (1
 * or 2) times in a row, then with drift != 0 x += v dt, wrap, and the
 * needs_rebuild test (neighbor.cpp:134-141) on the new positions, whose
 * result goes to *moved when moved != NULL (engine.cpp:142-172).  Owned atoms
 * only (tsf_set_owned); ghosts are refreshed by the exchange. */
int tsf_md_kick(tsf_ctx* ctx, double dt, int drift, int kicks, int* moved);
/* Kinetic energy of the owned atoms, eV (system.cpp:16-21). */
int tsf_md_kinetic(tsf_ctx* ctx, double* ke);

#ifdef __cplusplus
}
#endif
#endif /* TERSOFF_B200_H */
