// Spatial domain decomposition behind the C-ABI: x slabs, one
// rank per GPU, ghost-atom halo exchange, reverse ghost forces, atom migration
// at rebuilds and the distributed velocity-Verlet loop — all bookkeeping on
// the device, the host only sizes buffers.
//
// The reference has no distribution; this is the multi-GPU form
// of the paper's LAMMPS runs (Fig. 9).  Everything stays in the
// GLOBAL frame and the global periodic box: ghosts keep their owners' wrapped
// coordinates, so every displacement is the reference's minimum image bit for
// bit and a rank's lists are the global lists restricted to its atoms.
//
// Local layout of a rank's context (user order):
//   classic       [owned | ghosts from left | ghosts from right]
//   ghost centres [owned | layer-1 from left | layer-1 from right |
//                  layer-2 from left | layer-2 from right]
// Owned atoms are sorted by global id (deterministic layouts for any rank
// count).  Only owned atoms carry energy and virial; classic mode evaluates
// centres on owned atoms only and sends the forces its terms put on ghosts
// back to their owners (Newton's third law across the face); ghost-centre mode
// also evaluates the layer-1 ghosts (within one halo), so every term that
// puts force on an owned atom is evaluated locally — one exchange per step.
//
// Transports: NCCL (libnccl.so.2 loaded at run time — the library has no link
// dependency on it), or LOCAL: several ranks in one process, one context and
// one host thread each, messages moved by device-to-device copies ordered
// with CUDA events (stream waits only: no kernel ever waits on another rank).
// The local transport runs the multi-rank path on one GPU (tests, per-rank
// projections); NCCL runs it across the GPUs of a box.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tersoff_b200.h"
#include "tsf_context.hpp"

namespace tsf {

void evaluate_ctx(Ctx& c, Precision p, std::uint32_t flags);
void raise_errors(Ctx& c);
void set_system_device(Ctx& c, std::int64_t n, const double* d_xyz, const int* d_species,
                       const double* box, const std::uint8_t* per);
void set_velocities_device(Ctx& c, const double* d_vel, const double* masses);
void get_state_device(Ctx& c, std::int64_t m, double* d_xyz, double* d_vel);
void check_cuda(cudaError_t e, const char* what);

namespace {

int nblk(std::int64_t n, int b = 256) { return int(std::max<std::int64_t>(1, (n + b - 1) / b)); }

// ---------------------------------------------------------------------------
// transports
// ---------------------------------------------------------------------------
struct Msg {
  void* ptr;
  std::size_t bytes;
  int peer;
};

class Transport {
 public:
  virtual ~Transport() = default;
  // matched per (sender, receiver) pair in issue order; zero-byte messages
  // are legal and move nothing
  virtual void exchange(cudaStream_t s, const std::vector<Msg>& sends,
                        const std::vector<Msg>& recvs) = 0;
  // in place, every rank ends with the maximum
  virtual void allreduce_max_int(cudaStream_t s, int* d_val) = 0;
  // d_out[q] = sum over ranks of d_in[q], summed in rank order on every rank
  virtual void allreduce_sum(cudaStream_t s, const double* d_in, double* d_out, int count) = 0;
  int rank = 0, world = 1;
};

// ---- NCCL, resolved with dlopen ----
struct NcclApi {
  void* lib = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // TSF_NCCL_LIB, else a libnccl the process already loaded (torch's, so one
    // NCCL instance serves both), else the system's libnccl.so.2
    std::string path;
    if (const char* e = std::getenv("TSF_NCCL_LIB")) path = e;
    if (path.empty()) {
      if (std::FILE* f = std::fopen("/proc/self/maps", "r")) {
        char line[4096];
        while (std::fgets(line, sizeof line, f)) {
          const char* p = std::strstr(line, "/");
          if (p && std::strstr(p, "libnccl.so")) {
            path = p;
            while (!path.empty() && (path.back() == '\n' || path.back() == ' ')) path.pop_back();
            break;
          }
        }
        std::fclose(f);
      }
    }
    if (!path.empty()) a.lib = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if (!a.lib) a.lib = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
    if (!a.lib) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.lib, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.lib, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.lib, "ncclCommDestroy"));
    a.send = reinterpret_cast<decltype(a.send)>(dlsym(a.lib, "ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(a.lib, "ncclRecv"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(a.lib, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(a.lib, "ncclGroupEnd"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.lib, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.lib, "ncclGetErrorString"));
    return a;
  }();
  if (!api.lib || !api.send || !api.recv || !api.all_reduce || !api.comm_init_rank)
    throw ConfigError("NCCL transport unavailable: cannot load libnccl.so.2");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CudaError(std::string("NCCL ") + what + ": " +
                    (nccl().error_string ? nccl().error_string(r) : "error"));
}

class NcclTransport final : public Transport {
 public:
  NcclTransport(int world_, int rank_, const std::uint8_t* id) {
    world = world_;
    rank = rank_;
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    nccl_check(nccl().comm_init_rank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm_) nccl().comm_destroy(comm_);
  }
  void exchange(cudaStream_t s, const std::vector<Msg>& sends,
                const std::vector<Msg>& recvs) override {
    const NcclApi& a = nccl();
    nccl_check(a.group_start(), "ncclGroupStart");
    for (const Msg& m : sends)
      if (m.bytes) nccl_check(a.send(m.ptr, m.bytes, ncclUint8, m.peer, comm_, s), "ncclSend");
    for (const Msg& m : recvs)
      if (m.bytes) nccl_check(a.recv(m.ptr, m.bytes, ncclUint8, m.peer, comm_, s), "ncclRecv");
    nccl_check(a.group_end(), "ncclGroupEnd");
  }
  void allreduce_max_int(cudaStream_t s, int* d_val) override {
    nccl_check(nccl().all_reduce(d_val, d_val, 1, ncclInt32, ncclMax, comm_, s), "ncclAllReduce");
  }
  void allreduce_sum(cudaStream_t s, const double* d_in, double* d_out, int count) override {
    nccl_check(nccl().all_reduce(d_in, d_out, std::size_t(count), ncclFloat64, ncclSum, comm_, s),
               "ncclAllReduce");
  }

 private:
  ncclComm_t comm_ = nullptr;
};

// ---- in-process ranks ----
struct LocalGroup {
  explicit LocalGroup(int w) : world(w), box(std::size_t(w)) {}
  struct Posted {
    const void* ptr;
    std::size_t bytes;
    int dst;
  };
  struct Box {
    std::vector<Posted> out;
    cudaEvent_t ready = nullptr, consumed = nullptr;
    const void* red_ptr = nullptr;
  };
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
  int world;
  std::vector<Box> box;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
};

__global__ void k_max_of(const int* __restrict__ v, int m, int* __restrict__ out) {
  int r = v[0];
  for (int q = 1; q < m; ++q) r = max(r, v[q]);
  *out = r;
}

__global__ void k_sum_rows(const double* __restrict__ v, int m, int count,
                           double* __restrict__ out) {
  const int q = threadIdx.x;
  if (q >= count) return;
  double s = 0;
  for (int r = 0; r < m; ++r) s += v[r * count + q];
  out[q] = s;
}

class LocalTransport final : public Transport {
 public:
  LocalTransport(std::shared_ptr<LocalGroup> g, int rank_) : g_(std::move(g)) {
    world = g_->world;
    rank = rank_;
    LocalGroup::Box& b = g_->box[std::size_t(rank)];
    TSF_CUDA(cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming));
    TSF_CUDA(cudaEventCreateWithFlags(&b.consumed, cudaEventDisableTiming));
    scratch_.reserve(std::size_t(world) * 8);
  }
  ~LocalTransport() override {
    LocalGroup::Box& b = g_->box[std::size_t(rank)];
    if (b.ready) cudaEventDestroy(b.ready);
    if (b.consumed) cudaEventDestroy(b.consumed);
  }
  void exchange(cudaStream_t s, const std::vector<Msg>& sends,
                const std::vector<Msg>& recvs) override {
    LocalGroup::Box& me = g_->box[std::size_t(rank)];
    me.out.clear();
    for (const Msg& m : sends) me.out.push_back({m.ptr, m.bytes, m.peer});
    TSF_CUDA(cudaEventRecord(me.ready, s));
    g_->barrier();
    // pull every message addressed to me, per sender in issue order
    std::vector<std::size_t> next(std::size_t(world), 0);
    for (const Msg& m : recvs) {
      LocalGroup::Box& src = g_->box[std::size_t(m.peer)];
      std::size_t& k = next[std::size_t(m.peer)];
      while (k < src.out.size() && src.out[k].dst != rank) ++k;
      if (k >= src.out.size()) throw ConfigError("local transport: unmatched receive");
      const LocalGroup::Posted& p = src.out[k++];
      if (p.bytes != m.bytes) throw ConfigError("local transport: message size mismatch");
      if (m.bytes) {
        TSF_CUDA(cudaStreamWaitEvent(s, src.ready, 0));
        TSF_CUDA(cudaMemcpyAsync(m.ptr, p.ptr, m.bytes, cudaMemcpyDeviceToDevice, s));
      }
    }
    TSF_CUDA(cudaEventRecord(me.consumed, s));
    g_->barrier();
    // my later writes to the send buffers wait for the receivers' copies
    for (const Msg& m : sends)
      TSF_CUDA(cudaStreamWaitEvent(s, g_->box[std::size_t(m.peer)].consumed, 0));
    g_->barrier();
  }
  void allreduce_max_int(cudaStream_t s, int* d_val) override {
    gather(s, d_val, sizeof(int));
    k_max_of<<<1, 1, 0, s>>>(reinterpret_cast<const int*>(scratch_.get()), world, d_val);
    finish(s);
  }
  void allreduce_sum(cudaStream_t s, const double* d_in, double* d_out, int count) override {
    if (count > 8) throw ConfigError("local transport: allreduce of more than 8 values");
    gather(s, d_in, sizeof(double) * std::size_t(count));
    k_sum_rows<<<1, 32, 0, s>>>(scratch_.get(), world, count, d_out);
    finish(s);
  }

 private:
  // scratch[r] = rank r's value (rows of `bytes`)
  void gather(cudaStream_t s, const void* d_in, std::size_t bytes) {
    LocalGroup::Box& me = g_->box[std::size_t(rank)];
    me.red_ptr = d_in;
    TSF_CUDA(cudaEventRecord(me.ready, s));
    g_->barrier();
    for (int r = 0; r < world; ++r) {
      LocalGroup::Box& src = g_->box[std::size_t(r)];
      TSF_CUDA(cudaStreamWaitEvent(s, src.ready, 0));
      TSF_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(scratch_.get()) + r * bytes, src.red_ptr,
                               bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  void finish(cudaStream_t s) {
    TSF_CUDA(cudaEventRecord(g_->box[std::size_t(rank)].consumed, s));
    g_->barrier();
    for (int r = 0; r < world; ++r)
      TSF_CUDA(cudaStreamWaitEvent(s, g_->box[std::size_t(r)].consumed, 0));
    g_->barrier();
  }
  std::shared_ptr<LocalGroup> g_;
  DevBuf<double> scratch_;
};

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// wrapped distance from the slab faces: d_left = mod(x - lo, L), d_right = mod(hi - x, L)
__device__ __forceinline__ double dmod(double v, double L) {
  v = fmod(v, L);
  return v < 0 ? v + L : v;
}

// per owned atom: send flags {left L1, left L2, right L1, right L2} (classic
// mode uses the L1 pair with reach = halo)
__global__ void k_send_flags(const double* __restrict__ xyz, int n, double L, double lo,
                             double hi, double halo, double reach, int ghost_centers,
                             unsigned char* __restrict__ fl) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double x = xyz[3 * a];
  const double dl = dmod(x - lo, L), dr = dmod(hi - x, L);
  const bool l1 = dl <= halo, r1 = dr <= halo;
  const bool l2 = ghost_centers && !l1 && dl <= reach;
  const bool r2 = ghost_centers && !r1 && dr <= reach;
  fl[a] = l1;
  fl[n + a] = l2;
  fl[2 * n + a] = r1;
  fl[3 * n + a] = r2;
}

// ghost payload rows: gid, species, x, y, z
__global__ void k_pack_ghosts(const int* __restrict__ idx, int m, const long long* __restrict__ gid,
                              const int* __restrict__ sp, const double* __restrict__ xyz,
                              double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const int a = idx[q];
  double* o = out + 5 * std::size_t(q);
  o[0] = double(gid[a]);
  o[1] = double(sp[a]);
  o[2] = xyz[3 * a];
  o[3] = xyz[3 * a + 1];
  o[4] = xyz[3 * a + 2];
}

// received ghost rows -> local arrays at [lo, lo + m)
__global__ void k_unpack_ghosts(const double* __restrict__ in, int m, int lo,
                                long long* __restrict__ gid, int* __restrict__ sp,
                                double* __restrict__ xyz) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const double* r = in + 5 * std::size_t(q);
  const int a = lo + q;
  gid[a] = (long long)(r[0]);
  sp[a] = int(r[1]);
  xyz[3 * a] = r[2];
  xyz[3 * a + 1] = r[3];
  xyz[3 * a + 2] = r[4];
}

// owner of each owned atom after a step: flags {stay, to left, to right}; an
// atom farther than one slab sets *err
__global__ void k_owner_flags(const double* __restrict__ xyz, int n, double L, double width,
                              int world, int rank, unsigned char* __restrict__ fl,
                              int* __restrict__ err) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double x = dmod(xyz[3 * a], L);
  const int o = min(int(x / width), world - 1);
  const int left = (rank - 1 + world) % world, right = (rank + 1) % world;
  const bool stay = o == rank, to_l = !stay && o == left, to_r = !stay && !to_l && o == right;
  fl[a] = stay;
  fl[n + a] = to_l;
  fl[2 * n + a] = to_r;
  if (!(stay || to_l || to_r)) atomicOr(err, 1);
}

// migration payload rows: gid, species, x, y, z, vx, vy, vz
__global__ void k_pack_movers(const int* __restrict__ idx, int m, const long long* __restrict__ gid,
                              const int* __restrict__ sp, const double* __restrict__ xyz,
                              const double* __restrict__ vel, double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const int a = idx[q];
  double* o = out + 8 * std::size_t(q);
  o[0] = double(gid[a]);
  o[1] = double(sp[a]);
  for (int d = 0; d < 3; ++d) {
    o[2 + d] = xyz[3 * a + d];
    o[5 + d] = vel[3 * a + d];
  }
}

// new owned set: rows [0, ns) from the kept atoms (idx into the old arrays),
// rows [ns, ns + m) from the arrivals' payload
__global__ void k_assemble_owned(const int* __restrict__ keep, int ns, const double* __restrict__ arr,
                                 int m, const long long* __restrict__ gid0,
                                 const int* __restrict__ sp0, const double* __restrict__ xyz0,
                                 const double* __restrict__ vel0,
                                 unsigned long long* __restrict__ key, int* __restrict__ val,
                                 int* __restrict__ sp, double* __restrict__ xyz,
                                 double* __restrict__ vel) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ns + m) return;
  if (q < ns) {
    const int a = keep[q];
    key[q] = (unsigned long long)gid0[a];
    sp[q] = sp0[a];
    for (int d = 0; d < 3; ++d) {
      xyz[3 * q + d] = xyz0[3 * a + d];
      vel[3 * q + d] = vel0[3 * a + d];
    }
  } else {
    const double* r = arr + 8 * std::size_t(q - ns);
    key[q] = (unsigned long long)(long long)(r[0]);
    sp[q] = int(r[1]);
    for (int d = 0; d < 3; ++d) {
      xyz[3 * q + d] = r[2 + d];
      vel[3 * q + d] = r[5 + d];
    }
  }
  val[q] = q;
}

// apply a permutation: out row q = in row perm[q] (AoS triples, ints, gids)
__global__ void k_permute_owned(const int* __restrict__ perm,
                                const unsigned long long* __restrict__ key_sorted, int n,
                                const int* __restrict__ sp, const double* __restrict__ xyz,
                                const double* __restrict__ vel, long long* __restrict__ gid_o,
                                int* __restrict__ sp_o, double* __restrict__ xyz_o,
                                double* __restrict__ vel_o) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int a = perm[q];
  gid_o[q] = (long long)key_sorted[q];
  sp_o[q] = sp[a];
  for (int d = 0; d < 3; ++d) {
    xyz_o[3 * q + d] = xyz[3 * a + d];
    vel_o[3 * q + d] = vel[3 * a + d];
  }
}

__global__ void k_iota(int* __restrict__ v, int n) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) v[q] = q;
}

__global__ void k_copy_rows3(const double* __restrict__ in, int n, double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < 3 * n) out[q] = in[q];
}

}  // namespace

// ---------------------------------------------------------------------------
// one rank of the decomposition
// ---------------------------------------------------------------------------
struct DomainDecomposition {
  Ctx* c = nullptr;
  std::unique_ptr<Transport> tr;
  int rank = 0, world = 1, left = 0, right = 0;
  bool ghost_centers = false;
  double box[3] = {0, 0, 0};
  std::uint8_t per[3] = {1, 1, 1};
  double cutoff = 0, skin = 0, halo = 0, reach = 0;
  std::vector<double> masses;
  bool has_vel = false;
  // owned atoms (sorted by gid) and the local arrays [owned | ghosts]
  std::int64_t n_own = 0, n_loc = 0, n_ctr = 0;
  std::int64_t nl1 = 0, nl2 = 0, nr1 = 0, nr2 = 0;        // sent left / right, by layer
  std::int64_t gl1 = 0, gr1 = 0, gl2 = 0, gr2 = 0;        // ghosts received, by block
  DevBuf<long long> gid;            // [n_loc]
  DevBuf<int> sp;                   // [n_loc]
  DevBuf<double> xyz, vel;          // [n_loc][3] (vel: owned rows)
  DevBuf<int> send_idx;             // [to left L1 | L2 | to right L1 | L2]
  DevBuf<double> pos_send, ghost_in, f_ghost, f_to, payload_out, payload_in;
  DevBuf<unsigned char> flags_u8, cub_tmp;
  DevBuf<int> sel_count, idx_tmp, err;
  DevBuf<unsigned long long> key, key_out;
  DevBuf<int> val, val_out, sp_tmp;
  DevBuf<long long> gid_tmp;
  DevBuf<double> xyz_tmp, vel_tmp;
  DevBuf<double> ev_global;         // [7]: energy + virial summed over ranks
  std::int64_t rebuilds = 0, migrated = 0;

  cudaStream_t s() const { return c->stream; }

  // stable compaction of the indices [0, n) with flag fl[q]; count -> host
  std::int64_t select(const unsigned char* fl, int n, int* out) {
    if (n == 0) return 0;
    idx_tmp.reserve(std::size_t(n));
    k_iota<<<nblk(n), 256, 0, s()>>>(idx_tmp.get(), n);
    std::size_t tb = 0;
    TSF_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx_tmp.get(), fl, out, sel_count.get(), n,
                                        s()));
    cub_tmp.reserve(tb);
    TSF_CUDA(cub::DeviceSelect::Flagged(cub_tmp.get(), tb, idx_tmp.get(), fl, out,
                                        sel_count.get(), n, s()));
    int h = 0;
    TSF_CUDA(cudaMemcpyAsync(&h, sel_count.get(), sizeof(int), cudaMemcpyDeviceToHost, s()));
    TSF_CUDA(cudaStreamSynchronize(s()));
    return h;
  }

  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs) {
    tr->exchange(s(), sends, recvs);
  }

  // sizes in elements of T exchanged with the two neighbours: to-left /
  // to-right in, from-left / from-right out (host ints through a device buffer)
  void swap_counts(const std::int64_t* to_l, const std::int64_t* to_r, int k,
                   std::int64_t* from_l, std::int64_t* from_r) {
    DevBuf<long long> b;
    b.reserve(4 * std::size_t(k));
    std::vector<long long> h(4 * std::size_t(k), 0);
    for (int q = 0; q < k; ++q) {
      h[std::size_t(q)] = to_l[q];
      h[std::size_t(k + q)] = to_r[q];
    }
    TSF_CUDA(cudaMemcpyAsync(b.get(), h.data(), sizeof(long long) * 2 * k, cudaMemcpyHostToDevice,
                             s()));
    const std::size_t bytes = sizeof(long long) * std::size_t(k);
    exchange({{b.get(), bytes, left}, {b.get() + k, bytes, right}},
             {{b.get() + 3 * k, bytes, right}, {b.get() + 2 * k, bytes, left}});
    TSF_CUDA(cudaMemcpyAsync(h.data(), b.get(), sizeof(long long) * 4 * k,
                             cudaMemcpyDeviceToHost, s()));
    TSF_CUDA(cudaStreamSynchronize(s()));
    for (int q = 0; q < k; ++q) {
      from_l[q] = h[std::size_t(2 * k + q)];
      from_r[q] = h[std::size_t(3 * k + q)];
    }
  }

  // Ghost selection, ghost payload exchange, context load and list build from
  // the owned arrays (gid-sorted, rows [0, n_own) of gid / sp / xyz / vel).
  void rebuild_local() {
    const double L = box[0], width = L / world;
    const double lo = rank * width, hi = (rank + 1) * width;
    const int n = int(n_own);
    nl1 = nl2 = nr1 = nr2 = gl1 = gr1 = gl2 = gr2 = 0;
    send_idx.reserve(4 * std::size_t(std::max(n, 1)));
    if (world > 1) {
      flags_u8.reserve(4 * std::size_t(std::max(n, 1)));
      if (n > 0)
        k_send_flags<<<nblk(n), 256, 0, s()>>>(xyz.get(), n, L, lo, hi, halo, reach,
                                               ghost_centers ? 1 : 0, flags_u8.get());
      int* out = send_idx.get();
      nl1 = select(flags_u8.get(), n, out);
      nl2 = select(flags_u8.get() + n, n, out + nl1);
      nr1 = select(flags_u8.get() + 2 * n, n, out + nl1 + nl2);
      nr2 = select(flags_u8.get() + 3 * n, n, out + nl1 + nl2 + nr1);
      const std::int64_t to_l[2] = {nl1, nl2}, to_r[2] = {nr1, nr2};
      std::int64_t fl[2], fr[2];
      swap_counts(to_l, to_r, 2, fl, fr);
      gl1 = fl[0];
      gl2 = fl[1];
      gr1 = fr[0];
      gr2 = fr[1];
    }
    const std::int64_t nsend = nl1 + nl2 + nr1 + nr2, nghost = gl1 + gr1 + gl2 + gr2;
    n_loc = n_own + nghost;
    n_ctr = n_own + (ghost_centers ? gl1 + gr1 : 0);
    // local arrays grow to hold the ghosts (owned rows stay in place)
    auto grow = [&](auto& buf, std::size_t per_atom) {
      if (buf.cap < per_atom * std::size_t(std::max<std::int64_t>(n_loc, 1))) {
        using T = std::remove_reference_t<decltype(*buf.get())>;
        DevBuf<T> nb;
        nb.reserve(per_atom * std::size_t(std::max<std::int64_t>(n_loc, 1)));
        if (n_own > 0)
          TSF_CUDA(cudaMemcpyAsync(nb.get(), buf.get(), sizeof(T) * per_atom * n_own,
                                   cudaMemcpyDeviceToDevice, s()));
        std::swap(buf.ptr, nb.ptr);
        std::swap(buf.cap, nb.cap);
        TSF_CUDA(cudaStreamSynchronize(s()));   // the old buffer is freed here
      }
    };
    grow(gid, 1);
    grow(sp, 1);
    grow(xyz, 3);
    grow(vel, 3);
    if (nghost > 0) {
      payload_out.reserve(5 * std::size_t(nsend) + 1);
      payload_in.reserve(5 * std::size_t(nghost) + 1);
      if (nsend > 0)
        k_pack_ghosts<<<nblk(nsend), 256, 0, s()>>>(send_idx.get(), int(nsend), gid.get(),
                                                     sp.get(), xyz.get(), payload_out.get());
    }
    if (world > 1) {
      // sender: [to left L1 | L2 | to right L1 | L2]; receiver blocks
      // [L1 left | L1 right | L2 left | L2 right] (classic: L2 blocks empty)
      double* po = payload_out.get();
      double* pi = payload_in.get();
      const std::size_t row = 5 * sizeof(double);
      exchange({{po, row * nl1, left}, {po + 5 * nl1, row * nl2, left},
                {po + 5 * (nl1 + nl2), row * nr1, right},
                {po + 5 * (nl1 + nl2 + nr1), row * nr2, right}},
               {{pi + 5 * gl1, row * gr1, right}, {pi + 5 * (gl1 + gr1 + gl2), row * gr2, right},
                {pi, row * gl1, left}, {pi + 5 * (gl1 + gr1), row * gl2, left}});
      if (nghost > 0)
        k_unpack_ghosts<<<nblk(nghost), 256, 0, s()>>>(payload_in.get(), int(nghost), int(n_own),
                                                        gid.get(), sp.get(), xyz.get());
    }
    if (n_loc > n_own)
      TSF_CUDA(cudaMemsetAsync(vel.get() + 3 * n_own, 0, sizeof(double) * 3 * (n_loc - n_own),
                               s()));
    set_system_device(*c, n_loc, xyz.get(), sp.get(), box, per);
    c->n_owned = n_ctr;           // centres
    c->n_energy = n_own;          // energy, virial, integration
    c->n_interior = -1;
    c->split_slots = -1;
    ++c->list_version;
    if (has_vel) set_velocities_device(*c, vel.get(), masses.data());
    list_build(*c, cutoff, skin);
    // per-step buffers
    pos_send.reserve(3 * std::size_t(nsend) + 1);
    ghost_in.reserve(3 * std::size_t(nghost) + 1);
    f_ghost.reserve(3 * std::size_t(nghost) + 1);
    f_to.reserve(3 * std::size_t(nsend) + 1);
  }

  // ghost positions from their owners (every step)
  void forward() {
    if (world == 1) return;
    const std::int64_t nsend = nl1 + nl2 + nr1 + nr2;
    gather_positions(*c, send_idx.get(), nsend, pos_send.get());
    double* po = pos_send.get();
    double* gi = ghost_in.get();
    const std::size_t row = 3 * sizeof(double);
    exchange({{po, row * nl1, left}, {po + 3 * nl1, row * nl2, left},
              {po + 3 * (nl1 + nl2), row * nr1, right},
              {po + 3 * (nl1 + nl2 + nr1), row * nr2, right}},
             {{gi + 3 * gl1, row * gr1, right}, {gi + 3 * (gl1 + gr1 + gl2), row * gr2, right},
              {gi, row * gl1, left}, {gi + 3 * (gl1 + gr1), row * gl2, left}});
    scatter_positions(*c, n_own, n_loc - n_own, ghost_in.get());
  }

  // forces the owned centres' terms put on ghosts go home (classic mode)
  void reverse() {
    if (world == 1 || ghost_centers) return;
    const std::int64_t ng = n_loc - n_own;
    gather_forces(*c, n_own, ng, f_ghost.get());
    double* fg = f_ghost.get();
    double* ft = f_to.get();
    const std::size_t row = 3 * sizeof(double);
    // my left ghosts are the left rank's to-right list, my right ghosts its to-left
    exchange({{fg + 3 * gl1, row * gr1, right}, {fg, row * gl1, left}},
             {{ft, row * nl1, left}, {ft + 3 * nl1, row * nr1, right}});
    add_forces(*c, send_idx.get(), nl1 + nr1, f_to.get());
  }

  void evaluate(Precision p, std::uint32_t flags) {
    forward();
    evaluate_ctx(*c, p, flags);
    reverse();
    ev_global.reserve(8);
    tr->allreduce_sum(s(), c->result.get(), ev_global.get(), 7);
  }

  // owned positions + velocities out of the context (gid order rows)
  void pull_owned() {
    xyz.reserve(3 * std::size_t(std::max<std::int64_t>(n_loc, 1)));
    vel.reserve(3 * std::size_t(std::max<std::int64_t>(n_loc, 1)));
    get_state_device(*c, n_own, xyz.get(), has_vel ? vel.get() : nullptr);
  }

  // atoms that left the slab go to their new owner with species and velocity
  void migrate() {
    pull_owned();
    const int n = int(n_own);
    std::int64_t ns = n, ml = 0, mr = 0;
    int* keep = nullptr;
    std::int64_t from_l = 0, from_r = 0;
    if (world > 1) {
      flags_u8.reserve(3 * std::size_t(std::max(n, 1)));
      err.reserve(1);
      TSF_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(int), s()));
      if (n > 0)
        k_owner_flags<<<nblk(n), 256, 0, s()>>>(xyz.get(), n, box[0], box[0] / world, world,
                                                rank, flags_u8.get(), err.get());
      send_idx.reserve(3 * std::size_t(std::max(n, 1)));
      keep = send_idx.get();
      ns = select(flags_u8.get(), n, keep);
      ml = select(flags_u8.get() + n, n, keep + ns);
      mr = select(flags_u8.get() + 2 * n, n, keep + ns + ml);
      int e = 0;
      TSF_CUDA(cudaMemcpyAsync(&e, err.get(), sizeof(int), cudaMemcpyDeviceToHost, s()));
      TSF_CUDA(cudaStreamSynchronize(s()));
      if (e) throw ConfigError("an atom moved farther than one slab between list builds");
      swap_counts(&ml, &mr, 1, &from_l, &from_r);
    }
    const std::int64_t arrivals = from_l + from_r;
    payload_out.reserve(8 * std::size_t(ml + mr) + 1);
    payload_in.reserve(8 * std::size_t(arrivals) + 1);
    if (world > 1) {
      if (ml + mr > 0)
        k_pack_movers<<<nblk(ml + mr), 256, 0, s()>>>(keep + ns, int(ml + mr), gid.get(),
                                                      sp.get(), xyz.get(), vel.get(),
                                                      payload_out.get());
      const std::size_t row = 8 * sizeof(double);
      exchange({{payload_out.get(), row * ml, left}, {payload_out.get() + 8 * ml, row * mr, right}},
               {{payload_in.get() + 8 * from_l, row * from_r, right},
                {payload_in.get(), row * from_l, left}});
    } else {
      send_idx.reserve(std::size_t(std::max(n, 1)));
      keep = send_idx.get();
      if (n > 0) k_iota<<<nblk(n), 256, 0, s()>>>(keep, n);
    }
    migrated += arrivals;
    const std::int64_t m = ns + arrivals;
    const std::size_t mm = std::size_t(std::max<std::int64_t>(m, 1));
    key.reserve(mm);
    key_out.reserve(mm);
    val.reserve(mm);
    val_out.reserve(mm);
    sp_tmp.reserve(mm);
    xyz_tmp.reserve(3 * mm);
    vel_tmp.reserve(3 * mm);
    if (m > 0)
      k_assemble_owned<<<nblk(m), 256, 0, s()>>>(keep, int(ns), payload_in.get(), int(arrivals),
                                                 gid.get(), sp.get(), xyz.get(), vel.get(),
                                                 key.get(), val.get(), sp_tmp.get(),
                                                 xyz_tmp.get(), vel_tmp.get());
    set_owned_sorted(m);
  }

  // rows [0, m) of key / val / sp_tmp / xyz_tmp / vel_tmp, sorted by gid into
  // the owned arrays
  void set_owned_sorted(std::int64_t m) {
    n_own = m;
    const std::size_t mm = std::size_t(std::max<std::int64_t>(m, 1));
    gid.reserve(mm);
    sp.reserve(mm);
    xyz.reserve(3 * mm);
    vel.reserve(3 * mm);
    if (m > 0) {
      std::size_t tb = 0;
      TSF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.get(), key_out.get(), val.get(),
                                               val_out.get(), int(m), 0, 64, s()));
      cub_tmp.reserve(tb);
      TSF_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp.get(), tb, key.get(), key_out.get(),
                                               val.get(), val_out.get(), int(m), 0, 64, s()));
      k_permute_owned<<<nblk(m), 256, 0, s()>>>(val_out.get(), key_out.get(), int(m), sp_tmp.get(),
                                                xyz_tmp.get(), vel_tmp.get(), gid.get(), sp.get(),
                                                xyz.get(), vel.get());
    }
    rebuild_local();
  }

  // host arrays of this rank's owned atoms (any order)
  void setup(std::int64_t n, const std::int64_t* hgid, const double* hxyz, const std::int32_t* hsp,
             const double* hvel) {
    const std::size_t mm = std::size_t(std::max<std::int64_t>(n, 1));
    key.reserve(mm);
    key_out.reserve(mm);
    val.reserve(mm);
    val_out.reserve(mm);
    sp_tmp.reserve(mm);
    xyz_tmp.reserve(3 * mm);
    vel_tmp.reserve(3 * mm);
    std::vector<unsigned long long> k(mm, 0);
    std::vector<int> v(mm, 0);
    for (std::int64_t q = 0; q < n; ++q) {
      if (hgid[q] < 0) throw ConfigError("global atom ids must be non-negative");
      k[std::size_t(q)] = (unsigned long long)hgid[q];
      v[std::size_t(q)] = int(q);
    }
    if (n > 0) {
      TSF_CUDA(cudaMemcpyAsync(key.get(), k.data(), sizeof(unsigned long long) * n,
                               cudaMemcpyHostToDevice, s()));
      TSF_CUDA(cudaMemcpyAsync(val.get(), v.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s()));
      TSF_CUDA(cudaMemcpyAsync(sp_tmp.get(), hsp, sizeof(int) * n, cudaMemcpyHostToDevice, s()));
      TSF_CUDA(cudaMemcpyAsync(xyz_tmp.get(), hxyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice,
                               s()));
      if (hvel)
        TSF_CUDA(cudaMemcpyAsync(vel_tmp.get(), hvel, sizeof(double) * 3 * n,
                                 cudaMemcpyHostToDevice, s()));
      else
        TSF_CUDA(cudaMemsetAsync(vel_tmp.get(), 0, sizeof(double) * 3 * n, s()));
      TSF_CUDA(cudaStreamSynchronize(s()));
    }
    set_owned_sorted(n);
  }

  // velocity Verlet across the slabs (tsf_md_run's loop, engine.cpp:142-199):
  // the rebuild decision is the OR over ranks of the reference's
  // needs_rebuild test (a device allreduce the speculative evaluation reads);
  // at a rebuild atoms migrate and ghosts and lists are rebuilt.
  void md_run(Precision p, std::int64_t steps, double dt, std::uint32_t flags, int thermo_every,
              double* thermo, std::int64_t cap, std::int64_t* nsamples, std::int64_t* nreb) {
    if (!has_vel) throw ConfigError("set velocities before running dynamics");
    std::int64_t ns = 0, rb = 0;
    DevBuf<double> ke_loc, ke_glob;
    ke_loc.reserve(2);
    ke_glob.reserve(2);
    auto sample = [&](std::int64_t step) {
      md_kinetic(*c);
      TSF_CUDA(cudaMemcpyAsync(ke_loc.get(), c->result.get() + 7, sizeof(double),
                               cudaMemcpyDeviceToDevice, s()));
      tr->allreduce_sum(s(), ke_loc.get(), ke_glob.get(), 1);
      double pe = 0, ke = 0;
      TSF_CUDA(cudaMemcpyAsync(&pe, ev_global.get(), sizeof(double), cudaMemcpyDeviceToHost, s()));
      TSF_CUDA(cudaMemcpyAsync(&ke, ke_glob.get(), sizeof(double), cudaMemcpyDeviceToHost, s()));
      raise_errors(*c);
      if (thermo && ns < cap) {
        thermo[3 * ns] = double(step);
        thermo[3 * ns + 1] = pe;
        thermo[3 * ns + 2] = ke;
      }
      ++ns;
    };
    if (!c->pinned_flag)
      TSF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->pinned_flag), 64, cudaHostAllocDefault));
    if (!c->flag_event)
      TSF_CUDA(cudaEventCreateWithFlags(&c->flag_event, cudaEventDisableTiming));
    TSF_CUDA(cudaMemsetAsync(c->flags.get() + kFlagMoved, 0, sizeof(int), s()));
    TSF_CUDA(cudaMemsetAsync(c->flags.get() + kFlagMovedAny, 0, 2 * sizeof(int), s()));
    if (!c->forces_current) evaluate(p, flags);
    sample(0);
    struct Spec {
      Ctx& c;
      explicit Spec(Ctx& cc) : c(cc) { c.speculative = !c.profile; }
      ~Spec() { c.speculative = false; }
    } spec(*c);
    bool kick_pending = false;
    for (std::int64_t st = 1; st <= steps; ++st) {
      md_kick(*c, dt, true, kick_pending ? 2 : 1, /*check_rebuild=*/true);
      tr->allreduce_max_int(s(), c->flags.get() + kFlagMoved);
      TSF_CUDA(cudaMemcpyAsync(c->pinned_flag, c->flags.get() + kFlagMoved, sizeof(int),
                               cudaMemcpyDeviceToHost, s()));
      TSF_CUDA(cudaEventRecord(c->flag_event, s()));
      if (c->speculative) evaluate(p, flags);
      TSF_CUDA(cudaEventSynchronize(c->flag_event));
      if (*c->pinned_flag) {
        TSF_CUDA(cudaMemsetAsync(c->flags.get() + kFlagMoved, 0, sizeof(int), s()));
        TSF_CUDA(cudaMemsetAsync(c->flags.get() + kFlagMovedAny, 0, 2 * sizeof(int), s()));
        migrate();
        ++rb;
        ++rebuilds;
        evaluate(p, flags);
      } else if (!c->speculative) {
        evaluate(p, flags);
      }
      if (st % thermo_every == 0 || st == steps) {
        md_kick(*c, dt, false);
        sample(st);
        kick_pending = false;
      } else {
        kick_pending = true;
      }
    }
    if (nsamples) *nsamples = ns;
    if (nreb) *nreb = rb;
  }
};

}  // namespace tsf

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
struct tsf_ctx {
  tsf::Ctx c;
};
struct tsf_dd {
  tsf::DomainDecomposition d;
};
struct tsf_dd_group {
  std::shared_ptr<tsf::LocalGroup> g;
};

namespace {
thread_local std::string g_dd_err;

template <typename F>
int dd_guard(tsf_dd* dd, F&& f) {
  int rc = TSF_OK;
  try {
    if (dd) tsf::check_cuda(cudaSetDevice(dd->d.c->device), "cudaSetDevice");
    f();
  } catch (const tsf::ConfigError& e) {
    g_dd_err = e.what();
    rc = TSF_ERR_CONFIG;
  } catch (const tsf::ParseError& e) {
    g_dd_err = e.what();
    rc = TSF_ERR_CONFIG;
  } catch (const tsf::NumericError& e) {
    g_dd_err = e.what();
    rc = TSF_ERR_NUMERIC;
  } catch (const tsf::CudaError& e) {
    g_dd_err = std::string("CUDA error: ") + e.what();
    rc = TSF_ERR_CUDA;
  } catch (const std::exception& e) {
    g_dd_err = e.what();
    rc = TSF_ERR_INTERNAL;
  }
  return rc;
}

int dd_create(tsf_ctx* ctx, std::unique_ptr<tsf::Transport> tr, double cutoff, double skin,
              const double box[3], const uint8_t periodic[3], const double* masses,
              uint32_t mode, tsf_dd** out) {
  tsf::DomainDecomposition& d = (*out = new tsf_dd)->d;
  d.c = &ctx->c;
  d.tr = std::move(tr);
  d.world = d.tr->world;
  d.rank = d.tr->rank;
  d.left = (d.rank - 1 + d.world) % d.world;
  d.right = (d.rank + 1) % d.world;
  d.ghost_centers = (mode & TSF_DD_GHOST_CENTERS) != 0;
  for (int q = 0; q < 3; ++q) {
    d.box[q] = box[q];
    d.per[q] = periodic[q] ? 1 : 0;
  }
  d.cutoff = cutoff;
  d.skin = skin;
  d.halo = cutoff + skin;
  d.reach = d.ghost_centers ? 2.0 * d.halo : d.halo;
  if (!ctx->c.has_potential) throw tsf::ConfigError("the decomposition needs a context with a parameter table");
  if (masses) d.masses.assign(masses, masses + ctx->c.params.species_count());
  if (d.world > 1) {
    if (!d.per[0]) throw tsf::ConfigError("slab decomposition needs a periodic x axis");
    if (!(box[0] / d.world > 2.0 * d.reach))
      throw tsf::ConfigError(std::to_string(d.world) + " slabs of " +
                             std::to_string(box[0] / d.world) + " A are not wider than 2 x " +
                             std::to_string(d.reach) + " A");
  }
  d.sel_count.reserve(1);
  return TSF_OK;
}
}  // namespace

extern "C" {

const char* tsf_dd_error_message(void) { return g_dd_err.c_str(); }

int tsf_dd_nccl_unique_id(uint8_t* id) {
  return dd_guard(nullptr, [&] {
    ncclUniqueId uid;
    tsf::nccl_check(tsf::nccl().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(id, uid.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int tsf_dd_create_nccl(tsf_ctx* ctx, int world, int rank, const uint8_t* id, double cutoff,
                       double skin, const double box[3], const uint8_t periodic[3],
                       const double* masses, uint32_t mode, tsf_dd** out) {
  *out = nullptr;
  const int rc = dd_guard(nullptr, [&] {
    tsf::check_cuda(cudaSetDevice(ctx->c.device), "cudaSetDevice");
    if (world < 1 || rank < 0 || rank >= world) throw tsf::ConfigError("bad rank / world size");
    dd_create(ctx, std::make_unique<tsf::NcclTransport>(world, rank, id), cutoff, skin, box,
              periodic, masses, mode, out);
  });
  if (rc != TSF_OK && *out) {
    delete *out;
    *out = nullptr;
  }
  return rc;
}

int tsf_dd_group_create(int world, tsf_dd_group** out) {
  *out = nullptr;
  return dd_guard(nullptr, [&] {
    if (world < 1) throw tsf::ConfigError("bad world size");
    *out = new tsf_dd_group{std::make_shared<tsf::LocalGroup>(world)};
  });
}

void tsf_dd_group_destroy(tsf_dd_group* g) { delete g; }

int tsf_dd_create_local(tsf_ctx* ctx, tsf_dd_group* group, int rank, double cutoff, double skin,
                        const double box[3], const uint8_t periodic[3], const double* masses,
                        uint32_t mode, tsf_dd** out) {
  *out = nullptr;
  const int rc = dd_guard(nullptr, [&] {
    tsf::check_cuda(cudaSetDevice(ctx->c.device), "cudaSetDevice");
    if (rank < 0 || rank >= group->g->world) throw tsf::ConfigError("bad rank");
    auto t = std::make_unique<tsf::LocalTransport>(group->g, rank);
    dd_create(ctx, std::move(t), cutoff, skin, box, periodic, masses, mode, out);
  });
  if (rc != TSF_OK && *out) {
    delete *out;
    *out = nullptr;
  }
  return rc;
}

void tsf_dd_destroy(tsf_dd* dd) {
  if (!dd) return;
  cudaSetDevice(dd->d.c->device);
  cudaStreamSynchronize(dd->d.c->stream);
  delete dd;
}

int tsf_dd_setup(tsf_dd* dd, int64_t n_owned, const int64_t* gid, const double* xyz,
                 const int32_t* species, const double* vel) {
  return dd_guard(dd, [&] {
    tsf::DomainDecomposition& d = dd->d;
    if (vel && d.masses.empty()) throw tsf::ConfigError("velocities need species masses");
    d.has_vel = vel != nullptr;
    d.setup(n_owned, gid, xyz, species, vel);
  });
}

int tsf_dd_evaluate(tsf_dd* dd, int precision, uint32_t flags) {
  return dd_guard(dd, [&] {
    if (precision < 0 || precision > 2) throw tsf::ConfigError("unknown precision selector");
    dd->d.evaluate(tsf::Precision(precision), flags);
  });
}

int tsf_dd_rebuild(tsf_dd* dd) {
  return dd_guard(dd, [&] {
    dd->d.migrate();
    ++dd->d.rebuilds;
  });
}

int tsf_dd_md_run(tsf_dd* dd, int precision, int64_t steps, double dt, uint32_t flags,
                  int thermo_every, double* thermo, int64_t cap, int64_t* nsamples,
                  int64_t* rebuilds) {
  return dd_guard(dd, [&] {
    if (precision < 0 || precision > 2) throw tsf::ConfigError("unknown precision selector");
    if (steps < 0) throw tsf::ConfigError("steps must be non-negative");
    if (!(dt > 0.0)) throw tsf::ConfigError("dt must be positive");
    if (thermo_every < 1) throw tsf::ConfigError("thermo interval must be at least 1");
    dd->d.md_run(tsf::Precision(precision), steps, dt, flags, thermo_every, thermo, cap,
                 nsamples, rebuilds);
  });
}

int tsf_dd_set_positions(tsf_dd* dd, const double* xyz) {
  return dd_guard(dd, [&] {
    tsf::DomainDecomposition& d = dd->d;
    tsf::Ctx& c = *d.c;
    const std::int64_t n = d.n_own;
    if (n == 0) return;
    d.xyz_tmp.reserve(3 * std::size_t(n));
    TSF_CUDA(cudaMemcpyAsync(d.xyz_tmp.get(), xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice,
                             c.stream));
    tsf::scatter_positions(c, 0, n, d.xyz_tmp.get());
    TSF_CUDA(cudaStreamSynchronize(c.stream));   // pageable caller memory
  });
}

int tsf_dd_counts(tsf_dd* dd, int64_t* counts) {
  return dd_guard(dd, [&] {
    const tsf::DomainDecomposition& d = dd->d;
    const int64_t v[8] = {d.n_own, d.n_ctr, d.n_loc, d.nl1 + d.nl2, d.nr1 + d.nr2, d.rebuilds,
                          d.migrated, d.ghost_centers ? 1 : 0};
    std::memcpy(counts, v, sizeof v);
  });
}

int tsf_dd_results(tsf_dd* dd, double* energy_virial, int64_t* gid, double* xyz, double* forces,
                   double* vel) {
  return dd_guard(dd, [&] {
    tsf::DomainDecomposition& d = dd->d;
    tsf::Ctx& c = *d.c;
    const std::int64_t n = d.n_own;
    if (energy_virial) {
      TSF_CUDA(cudaMemcpyAsync(energy_virial, d.ev_global.get(), 7 * sizeof(double),
                               cudaMemcpyDeviceToHost, c.stream));
    }
    if (gid && n > 0)
      TSF_CUDA(cudaMemcpyAsync(gid, d.gid.get(), sizeof(long long) * n, cudaMemcpyDeviceToHost,
                               c.stream));
    std::vector<double> tmp;
    if ((xyz || vel) && n > 0) {
      d.pull_owned();
      if (xyz)
        TSF_CUDA(cudaMemcpyAsync(xyz, d.xyz.get(), sizeof(double) * 3 * n, cudaMemcpyDeviceToHost,
                                 c.stream));
      if (vel && d.has_vel)
        TSF_CUDA(cudaMemcpyAsync(vel, d.vel.get(), sizeof(double) * 3 * n, cudaMemcpyDeviceToHost,
                                 c.stream));
    }
    if (forces && n > 0) {
      tsf::unpack_forces(c);
      TSF_CUDA(cudaMemcpyAsync(forces, c.forces_user.get(), sizeof(double) * 3 * n,
                               cudaMemcpyDeviceToHost, c.stream));
    }
    TSF_CUDA(cudaStreamSynchronize(c.stream));
    tsf::raise_errors(c);
  });
}

}  // extern "C"
