// Device context behind the C-ABI: one CUDA stream, device-resident system,
// neighbor lists, force buffers and reduction scratch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
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

// Per-step reduction slots (energy + 6 virial components) per block.
constexpr int kRedWidth = 8;

struct ListState {
  int cap = 0;                 // ELL slots per atom
  DevBuf<int> nbr;             // [cap * npad]
  DevBuf<int> cnt;             // [npad]
  int max_count = 0;           // host copy, from the last build / filter
  bool valid = false;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  Params params;
  bool has_potential = true;   // false: list-only context (tsf_create with NULL params)
  bool hoist_ramp = true;
  bool fuse_filter = true;     // filter inside the force kernel (env TSF_FUSE_FILTER=0: separate)
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
  DevBuf<int> species;         // [n]
  std::vector<int> host_species;  // last uploaded species ids
  DevBuf<double4> pos;         // {x, y, z, species}
  DevBuf<double4> pos_ref;     // positions at the last list build (needs_rebuild)
  DevBuf<double> xyz_stage;    // AoS staging for H2D / D2H
  DevBuf<double> forces;       // [n][3]
  double* pinned = nullptr;    // pinned host staging, pinned_cap doubles
  std::size_t pinned_cap = 0;

  // neighbor lists
  double cutoff = 0, skin = 0;
  ListState skin_list, short_list;
  bool short_max_stale = true; // re-read the largest short count after the next filter
  int short_apply = -1;        // filter mode of the current short list
  DevBuf<int> cell_of, cell_count, cell_start, cell_fill, binned;
  DevBuf<unsigned char> scan_tmp;

  // force scratch
  DevBuf<double> px, py, pz;   // deterministic slot buffers [cap * npad]
  DevBuf<double> fself;        // [n][3]
  DevBuf<double> partials;     // [blocks][kRedWidth]
  DevBuf<double> result;       // energy + virial (7), reduced
  DevBuf<int> flags;           // [0] error bits, [1] overflow count, [2] rebuild flag,
                               // [3] largest skin count, [4] largest short count
  DevBuf<int> overflow;        // atoms with more short neighbors than the group width

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
void list_filter(Ctx& c, double r_cut_max, bool apply);
bool list_needs_rebuild(Ctx& c);
void snapshot_reference_positions(Ctx& c);

// ---- kernels (tsf_force.cu) ----
enum class Precision { F64 = 0, Mixed = 1, F32 = 2 };
void compute(Ctx& c, Precision prec, std::uint32_t flags);
void upload_params(Ctx& c);

// ---- kernels (tsf_md.cu) ----
// error bits in flags[0]
constexpr int kErrShortOverflow = 1;   // an atom has more than 32 short neighbours
constexpr int kErrNonFinite = 2;       // non-finite pair term

void pack_positions(Ctx& c);           // xyz_stage + species -> pos
void unpack_positions(Ctx& c);         // pos -> xyz_stage
void md_kick(Ctx& c, double dt, bool drift);   // v += F dt/(2 m mvv2e) [; x += v dt, wrap]
void md_kinetic(Ctx& c);               // KE -> result[7] (device)

void ensure_pinned(Ctx& c, std::size_t doubles);

}  // namespace tsf
