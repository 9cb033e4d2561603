// Device context behind the C-ABI: one CUDA stream, device-resident system,
// neighbor lists, force buffers and reduction scratch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "tsf_device.cuh"
#include "tsf_math.cuh"
#include "tsf_params.hpp"

namespace tsf {

// Growable device buffer.
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  std::size_t cap = 0;
  void reserve(std::size_t n);   // discards contents when it grows
  void release();
  ~DevBuf() { release(); }
  T* get() const { return ptr; }
};

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check_cuda(cudaError_t e, const char* what);
#define TSF_CUDA(call) ::tsf::check_cuda((call), #call)

// Launch with programmatic stream serialization (see griddep_wait): the
// kernel must begin with griddep_wait().
// TSF_PDL=0: plain launches (A/B runs).  Only the force chain (main -> tiers
// -> reduction) uses it: letting the main launch in behind the filter as well
// made the 2M-atom mixed/single step 15% slower (its blocks take the filter's
// last-wave slots), tools/ab.py.
int pdl_level();

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t stream,
                Args&&... args) {
  if (pdl_level() == 0) {
    kernel<<<grid, block, 0, stream>>>(std::forward<Args>(args)...);
    TSF_CUDA(cudaGetLastError());
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TSF_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Per-step reduction slots (energy + 6 virial components) per block.
constexpr int kRedWidth = 8;
// flags[] words outside the force path's [0..17]: the needs_rebuild result of
// the position writers (kick, k_needs_rebuild) — its own word, so the
// filter's per-evaluation zeroing of [0..3] cannot race a speculative
// readback (tsf_md_run) — and a word that stays zero (the "skip" pointer of
// non-speculative evaluations)
constexpr int kFlagMoved = 18;
constexpr int kFlagZero = 19;
// NaN distances seen by a force-path filter (its own word: the filter's block 0
// zeroes flags[0..3] while other blocks run); cleared when raised
constexpr int kFlagFilterNaN = 20;
// tsf_md_run's multi-step segments: the "moved" flag of any earlier step of
// the segment (folded in by k_reduce, so it never changes during a kick) and
// the step whose kick first set it
constexpr int kFlagMovedAny = 21;
constexpr int kFlagMovedStep = 22;
// a filter launch refreshed the near lists (their displacement maximum,
// flags[10], restarts: k_reduce clears both once every launch has read it)
constexpr int kFlagNearRefresh = 23;
constexpr int kFlagNearRefreshCount = 24;   // cumulative (tsf_near_refreshes)
// a force-path filter saw a short count over 4 (set once, check before store;
// cleared by k_reduce): an idle packed tier launch exits without scanning
constexpr int kFlagOver4 = 25;

struct ListState {
  int cap = 0;                 // ELL slots per atom
  DevBuf<int> nbr;             // [cap * npad]
  DevBuf<int> cnt;             // [npad]
  int max_count = 0;           // host copy, from the last build / filter
  int over4 = 0, over8 = 0;    // atoms with more than 4 / 8 entries (short list)
  bool valid = false;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  Params params;
  bool has_potential = true;   // false: list-only context (tsf_create with NULL params)
  bool hoist_ramp = true;
  std::string err;
  std::int64_t launches = 0;

  // parameters on the device
  DevBuf<Row<double>> rows_f64;
  DevBuf<Row<float>> rows_f32;
  DevBuf<double> cutsq;        // S^3, exact doubles for the cutoff tests

  // system
  std::int64_t n = 0;
  int npad = 0;
  Box box{};
  // Atoms live in HBM in cell-sorted order ("slots"), re-sorted at every list
  // build with the key (cell, user index); perm maps slot -> user index.  The
  // user order is restored only at the I/O boundary (pack / unpack / forces).
  DevBuf<int> species;         // [n] user order
  std::vector<int> host_species;  // last uploaded species ids
  DevBuf<int> perm;            // [n] slot -> user index
  DevBuf<int> inv;             // [n] user index -> slot
  bool sorted = false;         // false: perm is the identity (slot == user index)
  std::int64_t n_owned = -1;   // user atoms [0, n_owned) are centers; -1: all
  std::int64_t n_interior = -1; // user atoms [0, n_interior) are interior owned atoms (no
                               // ghost in their skin list): list builds give them slots
                               // [0, n_interior) for the two-phase evaluation; -1: off
  std::int64_t n_energy = -1;  // user atoms [0, n_energy) are owned: they count energy and
                               // virial and are integrated by MD; -1: the centers
  cudaStream_t own_stream = nullptr;
  DevBuf<double4> pos;         // [n] slot order {x, y, z, species}
  DevBuf<float4> posf;         // [n] slot order float shadow for the cutoff pre-tests
  BoxF boxf{};
  DevBuf<double4> pos_ref;     // positions at the last list build (needs_rebuild)
  // Near lists (k_filter): our own list builds also keep, per atom, the skin
  // entries that lay within near_cut[q] = r_cut_max + h_q at the build
  // (h_0 = s/4, h_1 = s/2, s the list's reach past every cutoff), in skin
  // order.  Every position writer keeps the largest squared displacement since
  // the build in flags[10]; while 2 |d|max < h_q an entry outside near list q
  // is provably outside every cutoff, so the filter reads the smallest near
  // list still valid instead of the skin list (crystalline Si: 4 entries
  // instead of 16).  near_ok: pos_ref and the near lists describe the current
  // slots (our build, not an external list).
  ListState near_list[2];
  double near_cut[2] = {0, 0};  // 0: no near lists
  float near_t[2] = {0, 0};     // list q valid while |d|max^2 < near_t[q] = ((h_q - mu) / 2)^2
  int near_pre[2] = {4, 4};     // ELL4 blocks the filter requests up front from list q
  bool near_ok = false;
  // Near-list refresh: when both near lists go stale mid-life, the force
  // path's filter reads the skin list and writes both near lists afresh from
  // the current positions; near_d0[s] keeps slot s's displacement since the
  // build at that moment, so displacements are tracked from the refresh
  // without a second position read (DispRef).
  DevBuf<float4> near_d0;
  DevBuf<double> xyz_stage;    // AoS staging for H2D / D2H, user order
  DevBuf<double> forces;       // [n][3] slot order (accumulation, MD)
  DevBuf<double> forces_user;  // [n][3] user order (download)
  DevBuf<double4> tmp4;        // re-sort scratch
  DevBuf<double> tmp3;
  DevBuf<int> tmp_i;
  DevBuf<unsigned> sort_keys, sort_keys_out;   // cell ids, indexed by user atom
  DevBuf<int> sort_vals, sort_vals_out;
  double* pinned = nullptr;    // pinned host staging, pinned_cap doubles
  std::size_t pinned_cap = 0;

  // neighbor lists
  double cutoff = 0, skin = 0;
  ListState skin_list, short_list;
  bool short_max_stale = true; // re-read the largest short count after the next filter
  int short_apply = -1;        // filter mode of the current short list
  DevBuf<int> cell_of, cell_count, cell_start, cell_fill, binned;
  CellGrid grid{};             // cell grid of the last build
  bool tiled = false;          // slots are cell-sorted for `grid` (our own build)
  DevBuf<unsigned char> scan_tmp;

  // force scratch
  DevBuf<double> px, py, pz;   // deterministic slot buffers [cap * npad]
  DevBuf<double> fself;        // [n][3]
  DevBuf<double> atom_ev;      // deterministic tier launches: [n][8] energy + virial
  DevBuf<double> partials;     // [blocks][kRedWidth]
  DevBuf<double> result;       // energy + virial (7), reduced
  DevBuf<int> flags;           // [0] error bits, [1..3] tier queue counts (force path;
                               // [2] doubles as the rebuild flag and [3] as the largest
                               // skin count, both read synchronously in their own calls),
                               // [3] largest skin count, [4] largest short count,
                               // [5] |coord| max bits, [6] max cell occupancy,
                               // [7] species error, [8]/[9] atoms with > 4 / > 8 short entries,
                               // [10] squared displacement max since the list build (float bits),
                               // [11..16] atoms with > 4 / > 8 / > 12 entries in near list
                               // 0 / 1 (list build)
  DevBuf<int> overflow;        // [3n] tier queues (G = 8, 16, 32 inputs)

  // slot range and position of the current compute() call in a two-phase
  // evaluation (tsf_compute_phase); a plain evaluation is [0, n), first+last
  int phase_lo = 0, phase_hi = 0;
  bool phase_first = true, phase_last = true;
  int phase_blocks = 0;                // partial blocks written by earlier phases
  std::int64_t split_slots = -1;       // interior slots [0, split) of the current list
  std::int64_t center_slots = -1;      // list built with centres first: slots [0, this) hold
                                       // every centre, non-centre ghosts follow (else -1)
  bool phase0_done = false;            // phase 0 ran; phase 1 completes the evaluation

  // CUDA graph of the steady-state evaluation (filter + force launches),
  // replayed while its key holds; see evaluate() in tsf_capi.cu
  std::uint64_t list_version = 0;      // bumped by every list / centre-set change
  // tsf_md_run's speculative step: the evaluation is queued behind the kick
  // before its rebuild flag is known; its filter and force launches return at
  // once when flags[kFlagMoved] is set (the step is then re-evaluated after
  // the rebuild), so the GPU never waits for the host between steps
  bool speculative = false;
  bool filter_marks_over4 = false;   // the last filter launch raised flags[kFlagOver4]
  bool main_packed = false;          // the last force evaluation's main launch was packed
  int* pinned_flag = nullptr;          // page-locked host word for the flag readback
  cudaEvent_t flag_event = nullptr;
  // identity of the externally supplied list on the device (tsf_set_neighbor_list)
  std::uint64_t adopted_id = 0;
  bool adopted_valid = false;          // cleared by every device-side list build
  std::int64_t adoption_hits = 0;      // adoptions that found the same list resident
  // (slot 0: a whole evaluation; 1 and 2: the two phases of a split one)
  struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    std::uint64_t key[6] = {};         // key of exec
    std::uint64_t warm[6] = {};        // key of the last eager run
    std::int64_t launches = 0;         // kernels per replay
    int phase_blocks = 0;              // host state the launches leave behind
  };
  GraphSlot graph[4];   // 0 evaluation, 1-2 split phases, 3 MD segment
  double seg_dt = 0;    // time step baked into graph[3]'s kick nodes
  bool species_set = false;   // species of the current n atoms are on the device
  bool graphs_off = false;             // capture failed once: stay eager

  // MD state
  DevBuf<double> vel;          // [n][3]
  std::vector<double> masses;  // per species
  bool forces_current = false; // forces/result match the current positions

  // optional per-stage CUDA-event timing of evaluate():
  // [0] filter, [1] memsets/launch setup, [2] main force kernel, [3] overflow +
  // reduction + gather/convert
  bool profile = false;
  cudaEvent_t ev[5] = {};
  double stage_ms[4] = {0, 0, 0, 0};
  std::int64_t profiled_calls = 0;
  void mark(int k) {
    if (profile) TSF_CUDA(cudaEventRecord(ev[k], stream));
  }

  explicit Ctx(Params p) : params(std::move(p)) {}
};

// ---- kernels (tsf_neighbor.cu) ----
void list_build(Ctx& c, double cutoff, double skin);
// Short list from the skin list: a verbatim copy (filter off), the
// reference's r_cut_max test (exports), or the per species-pair bounds the
// force path uses (PairBounds; identical to Cutoff for one species).
enum class FilterMode { Copy = 0, Cutoff = 1, Pair = 2 };
// zero_forces: optional [n][3] accumulator (zero_bytes = 8 double / 4 float)
// the filter zeroes for the atomic-mode force kernel
// lo / hi: the slot range (two-phase evaluation); hi < 0: all atoms
// zero_flags: the filter launch also zeroes flags[0..3] (kFlagFlagsZeroed)
void list_filter(Ctx& c, FilterMode mode, void* zero_forces = nullptr, int zero_bytes = 0,
                 int lo = 0, int hi = -1, bool zero_flags = false);
bool list_needs_rebuild(Ctx& c);
void snapshot_reference_positions(Ctx& c);

// ---- kernels (tsf_force.cu) ----
enum class Precision { F64 = 0, Mixed = 1, F32 = 2 };
// compute() flag (internal, above the public TSF_* bits): the atomic-mode
// force accumulator was zeroed by the filter launch
constexpr std::uint32_t kFlagForcesZeroed = 1u << 16;
// the filter launch zeroed flags[0..3] (error bits and tier queue counts)
constexpr std::uint32_t kFlagFlagsZeroed = 1u << 17;
// no caller reads this evaluation's virial (result[1..6] are left zero)
constexpr std::uint32_t kFlagNoVirial = 0x4u;   // = TSF_NO_VIRIAL (include/tersoff_b200.h)
void compute(Ctx& c, Precision prec, std::uint32_t flags);
void upload_params(Ctx& c);

// ---- kernels (tsf_md.cu) ----
// error bits in flags[0]
constexpr int kErrShortOverflow = 1;   // an atom has more than 32 short neighbours
constexpr int kErrNonFinite = 2;       // non-finite pair term
constexpr int kErrBadSpecies = 4;      // species id out of range (device-side check)

void validate_species(Ctx& c, int nspecies);   // sets kErrBadSpecies in flags[0]

void pack_positions(Ctx& c);           // xyz_stage + species (user order) -> pos (slots)
void unpack_positions(Ctx& c);         // pos (slots) -> xyz_stage (user order)
void unpack_forces(Ctx& c);            // forces (slots) -> forces_user
void unsort(Ctx& c);                   // back to slot == user index (external lists)
// decomposition support (device pointers, user indices)
void gather_positions(Ctx& c, const int* d_idx, std::int64_t m, double* d_xyz);
void scatter_positions(Ctx& c, std::int64_t lo, std::int64_t m, const double* d_xyz);
void gather_forces(Ctx& c, std::int64_t lo, std::int64_t m, double* d_f);
void add_forces(Ctx& c, const int* d_idx, std::int64_t m, const double* d_f);
void refresh_shadow(Ctx& c);           // posf = float(pos)
void pack_velocities(Ctx& c);          // xyz_stage (user order velocities) -> vel (slots)
void unpack_velocities(Ctx& c);        // vel (slots) -> xyz_stage (user order)
// v += F dt/(2 m mvv2e), `kicks` (1 or 2) times in a row [; x += v dt, wrap
// [; the needs_rebuild test on the new positions -> flags[2]]]
void md_kick(Ctx& c, double dt, bool drift, int kicks = 1, bool check_rebuild = false,
             int seg_step = -1);   // seg_step >= 0: a segment step (skips once a step moved)
void md_kinetic(Ctx& c);               // KE -> result[7] (device)
void md_scale_velocities(Ctx& c, double factor);

void ensure_pinned(Ctx& c, std::size_t doubles);

}  // namespace tsf
