// On-disk snapshots: the fixture format for thermalised and liquid states
// (SURVEY.md 8f row 4).  The reference has no snapshot file — its fixtures are
// regenerated from seeds (make_diamond_lattice engine.cpp:28-58,
// init_velocities engine.cpp:64-116, perturbed_lattice verify.cpp:83-104) —
// which is impossible for a melted state: a liquid comes from thousands of MD
// steps whose bits depend on the force kernel.  So the state is stored once
// and every consumer (GPU path, CPU oracle, the reference's own CPU arm)
// evaluates the same bytes.
//
// Layout (little-endian, no padding between sections):
//   0   char     magic[8]      "TSFSNAP1"
//   8   uint32   flags         TSF_SNAP_F32_COORDS | TSF_SNAP_VELOCITIES
//   12  int32    nspecies      1..255
//   16  int64    n
//   24  double   box[3]
//   48  uint8    periodic[3], 5 zero bytes
//   56  double   masses[nspecies]
//       coords   n*3 float64, or n*3 float32 with TSF_SNAP_F32_COORDS
//       uint8    species[n]
//       double   vel[n*3]      only with TSF_SNAP_VELOCITIES
//       uint8    sha256[32]    of every byte before it
// With F32 coordinates the stored state IS the float32-rounded one (exactly
// representable in double): a reader returns those values widened, bit for
// bit, whatever wrote them.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tersoff_b200.h"
#include "tsf_params.hpp"

namespace tsf {

// ---- SHA-256 (FIPS 180-4) ---------------------------------------------------
namespace {

constexpr std::uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

inline std::uint32_t rotr(std::uint32_t x, int s) { return (x >> s) | (x << (32 - s)); }

class Sha256 {
 public:
  void update(const void* data, std::size_t len) {
    const auto* p = static_cast<const std::uint8_t*>(data);
    total_ += len;
    if (fill_) {
      const std::size_t take = std::min<std::size_t>(64 - fill_, len);
      std::memcpy(buf_ + fill_, p, take);
      fill_ += take;
      p += take;
      len -= take;
      if (fill_ == 64) {
        block(buf_);
        fill_ = 0;
      }
    }
    for (; len >= 64; p += 64, len -= 64) block(p);
    if (len) {
      std::memcpy(buf_, p, len);
      fill_ = len;
    }
  }
  void finish(std::uint8_t out[32]) {
    const std::uint64_t bits = std::uint64_t(total_) * 8;
    const std::uint8_t one = 0x80, zero = 0;
    update(&one, 1);
    while (fill_ != 56) update(&zero, 1);
    std::uint8_t be[8];
    for (int i = 0; i < 8; ++i) be[i] = std::uint8_t(bits >> (56 - 8 * i));
    update(be, 8);
    for (int i = 0; i < 8; ++i)
      for (int b = 0; b < 4; ++b) out[4 * i + b] = std::uint8_t(h_[i] >> (24 - 8 * b));
  }

 private:
  void block(const std::uint8_t* p) {
    std::uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = std::uint32_t(p[4 * i]) << 24 | std::uint32_t(p[4 * i + 1]) << 16 |
             std::uint32_t(p[4 * i + 2]) << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const std::uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const std::uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    std::uint32_t a = h_[0], b = h_[1], c = h_[2], d = h_[3], e = h_[4], f = h_[5], g = h_[6],
                  h = h_[7];
    for (int i = 0; i < 64; ++i) {
      const std::uint32_t t1 =
          h + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + kK[i] + w[i];
      const std::uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      h = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h_[0] += a, h_[1] += b, h_[2] += c, h_[3] += d, h_[4] += e, h_[5] += f, h_[6] += g,
        h_[7] += h;
  }

  std::uint32_t h_[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                         0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  std::uint8_t buf_[64];
  std::size_t fill_ = 0;
  std::size_t total_ = 0;
};

constexpr char kMagic[8] = {'T', 'S', 'F', 'S', 'N', 'A', 'P', '1'};
constexpr std::size_t kHeader = 56;

struct File {
  std::FILE* f;
  explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

// Whole-file read + checksum verification; returns the payload (checksum stripped).
std::vector<std::uint8_t> read_verified(const char* path) {
  File fh(path, "rb");
  if (!fh.f) throw ConfigError(std::string("cannot open snapshot '") + path + "'");
  std::vector<std::uint8_t> buf;
  std::uint8_t chunk[1 << 16];
  for (std::size_t got; (got = std::fread(chunk, 1, sizeof chunk, fh.f)) > 0;)
    buf.insert(buf.end(), chunk, chunk + got);
  if (buf.size() < kHeader + 32 || std::memcmp(buf.data(), kMagic, 8) != 0)
    throw ParseError(std::string("'") + path + "' is not a TSFSNAP1 snapshot");
  std::uint8_t sha[32];
  Sha256 h;
  h.update(buf.data(), buf.size() - 32);
  h.finish(sha);
  if (std::memcmp(sha, buf.data() + buf.size() - 32, 32) != 0)
    throw ParseError(std::string("snapshot '") + path + "' fails its SHA-256 check");
  buf.resize(buf.size() - 32);
  return buf;
}

struct Header {
  std::uint32_t flags;
  std::int32_t ns;
  std::int64_t n;
  double box[3];
  std::uint8_t per[3];
};

Header parse_header(const std::vector<std::uint8_t>& b) {
  Header h{};
  std::memcpy(&h.flags, b.data() + 8, 4);
  std::memcpy(&h.ns, b.data() + 12, 4);
  std::memcpy(&h.n, b.data() + 16, 8);
  std::memcpy(h.box, b.data() + 24, 24);
  std::memcpy(h.per, b.data() + 48, 3);
  if (h.flags & ~std::uint32_t(TSF_SNAP_F32_COORDS | TSF_SNAP_VELOCITIES))
    throw ParseError("snapshot has unknown flags");
  if (h.ns < 1 || h.ns > 255 || h.n < 0) throw ParseError("snapshot header is corrupt");
  const std::size_t cw = (h.flags & TSF_SNAP_F32_COORDS) ? 4 : 8;
  const std::size_t want = kHeader + 8 * std::size_t(h.ns) + 3 * cw * std::size_t(h.n) +
                           std::size_t(h.n) +
                           ((h.flags & TSF_SNAP_VELOCITIES) ? 24 * std::size_t(h.n) : 0);
  if (b.size() != want) throw ParseError("snapshot size does not match its header");
  return h;
}

}  // namespace

void snapshot_sha256(const void* data, std::size_t len, std::uint8_t out[32]) {
  Sha256 h;
  h.update(data, len);
  h.finish(out);
}

void snapshot_write(const char* path, std::int64_t n, const double* xyz,
                    const std::int32_t* species, int ns, const double* masses, const double* box,
                    const std::uint8_t* periodic, const double* vel, std::uint32_t flags,
                    std::uint8_t* sha_out) {
  if (n < 0) throw ConfigError("atom count must be non-negative");
  if (ns < 1 || ns > 255) throw ConfigError("snapshots hold 1..255 species");
  if (flags & ~std::uint32_t(TSF_SNAP_F32_COORDS | TSF_SNAP_VELOCITIES))
    throw ConfigError("unknown snapshot flags");
  if ((flags & TSF_SNAP_VELOCITIES) && !vel)
    throw ConfigError("TSF_SNAP_VELOCITIES needs a velocity array");
  std::vector<std::uint8_t> b(kHeader, 0);
  std::memcpy(b.data(), kMagic, 8);
  const std::int32_t ns32 = ns;
  std::memcpy(b.data() + 8, &flags, 4);
  std::memcpy(b.data() + 12, &ns32, 4);
  std::memcpy(b.data() + 16, &n, 8);
  std::memcpy(b.data() + 24, box, 24);
  for (int d = 0; d < 3; ++d) b[48 + d] = periodic[d] ? 1 : 0;
  auto put = [&](const void* p, std::size_t len) {
    const auto* q = static_cast<const std::uint8_t*>(p);
    b.insert(b.end(), q, q + len);
  };
  put(masses, 8 * std::size_t(ns));
  for (int s = 0; s < ns; ++s)
    if (!(masses[s] > 0.0) || !std::isfinite(masses[s]))
      throw ConfigError("species masses must be positive and finite");
  for (std::int64_t i = 0; i < 3 * n; ++i)
    if (!std::isfinite(xyz[i])) throw ConfigError("non-finite coordinate");
  if (flags & TSF_SNAP_F32_COORDS) {
    std::vector<float> f(3 * std::size_t(n));
    for (std::size_t i = 0; i < f.size(); ++i) f[i] = float(xyz[i]);
    put(f.data(), 4 * f.size());
  } else {
    put(xyz, 24 * std::size_t(n));
  }
  for (std::int64_t a = 0; a < n; ++a) {
    if (species[a] < 0 || species[a] >= ns)
      throw ConfigError("atom " + std::to_string(a) + " has species id " +
                        std::to_string(species[a]) + " outside [0, " + std::to_string(ns) + ")");
    b.push_back(std::uint8_t(species[a]));
  }
  if (flags & TSF_SNAP_VELOCITIES) put(vel, 24 * std::size_t(n));
  std::uint8_t sha[32];
  snapshot_sha256(b.data(), b.size(), sha);
  put(sha, 32);
  File fh(path, "wb");
  if (!fh.f) throw ConfigError(std::string("cannot create snapshot '") + path + "'");
  if (std::fwrite(b.data(), 1, b.size(), fh.f) != b.size())
    throw ConfigError(std::string("short write to '") + path + "'");
  if (sha_out) std::memcpy(sha_out, sha, 32);
}

void snapshot_info(const char* path, std::int64_t* n, int* ns, std::uint32_t* flags,
                   std::uint8_t* sha_out) {
  const auto b = read_verified(path);
  const Header h = parse_header(b);
  if (n) *n = h.n;
  if (ns) *ns = h.ns;
  if (flags) *flags = h.flags;
  if (sha_out) {
    File fh(path, "rb");
    std::fseek(fh.f, -32, SEEK_END);
    if (std::fread(sha_out, 1, 32, fh.f) != 32) throw ParseError("cannot re-read checksum");
  }
}

void snapshot_read(const char* path, double* xyz, std::int32_t* species, double* masses,
                   double* box, std::uint8_t* periodic, double* vel) {
  const auto b = read_verified(path);
  const Header h = parse_header(b);
  const std::size_t n = std::size_t(h.n);
  std::size_t at = kHeader;
  if (masses) std::memcpy(masses, b.data() + at, 8 * std::size_t(h.ns));
  at += 8 * std::size_t(h.ns);
  if (h.flags & TSF_SNAP_F32_COORDS) {
    for (std::size_t i = 0; i < 3 * n; ++i) {
      float f;
      std::memcpy(&f, b.data() + at + 4 * i, 4);
      if (xyz) xyz[i] = double(f);
    }
    at += 12 * n;
  } else {
    if (xyz) std::memcpy(xyz, b.data() + at, 24 * n);
    at += 24 * n;
  }
  for (std::size_t a = 0; a < n; ++a) {
    if (b[at + a] >= h.ns) throw ParseError("snapshot species id out of range");
    if (species) species[a] = b[at + a];
  }
  at += n;
  if (vel) {
    if (h.flags & TSF_SNAP_VELOCITIES)
      std::memcpy(vel, b.data() + at, 24 * n);
    else
      std::memset(vel, 0, 24 * n);
  }
  if (box) std::memcpy(box, h.box, 24);
  if (periodic) std::memcpy(periodic, h.per, 3);
}

}  // namespace tsf
