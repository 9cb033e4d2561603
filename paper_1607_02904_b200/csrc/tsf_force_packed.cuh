// Packed lane groups: the paper's vector repacking (the
// reference's V2 per-lane traversal, kernels.hpp:304-494) as a warp layout.
//
// k_force gives every central atom a power-of-two group of G lanes, so an
// atom with 5 short neighbours idles 3 lanes of a G = 8 group, and an
// irregular system (3C-SiC: 45% of the atoms over 4; the 3000 K liquid: 2..13)
// either idles lanes or leaves atoms to wider launches.  Here a warp takes a
// chunk of 32 atoms — consecutive slots (main launch), or, behind a G-wide
// main launch, the next 32 atoms over G of its own slot range (tier launch:
// found by scanning the counts, no queue) — sorts them by count, scans the
// counts and packs their neighbour slots back to back: a pack is the longest
// run of atoms whose slots fit in 32 lanes, segment heads come from a ballot,
// every lane finds its atom through its segment head, and the rotation scheme
// of k_force runs inside each segment with its own length n_i (partner
// k = slot (l + t) mod n_i, stopping at the pack's largest count).  The
// k-gradients of the first kCacheRot rotations stay in registers; later
// rotations are recomputed in the scatter pass.  F_i is a segmented sum
// through shared memory.  Nothing is queued: any count up to 32 is served.
#pragma once

namespace tsf {
namespace {

#ifndef TSF_PACKED_CACHE_F64
#define TSF_PACKED_CACHE_F64 5
#endif
#ifndef TSF_PACKED_CACHE_F32
#define TSF_PACKED_CACHE_F32 7
#endif
#ifndef TSF_PACKED_AHEAD
#define TSF_PACKED_AHEAD 1
#endif
template <typename R>
constexpr int kPackedCacheRot =
    std::is_same<R, double>::value ? TSF_PACKED_CACHE_F64 : TSF_PACKED_CACHE_F32;
#ifndef TSF_PACKED_MINB_F64
#define TSF_PACKED_MINB_F64 4
#endif
#ifndef TSF_PACKED_MINB_F32
#define TSF_PACKED_MINB_F32 5
#endif
template <typename R>
constexpr int kPackedMinBlocks =
    std::is_same<R, double>::value ? TSF_PACKED_MINB_F64 : TSF_PACKED_MINB_F32;

// The packed kernel's shared memory (also embedded in k_force when the tier
// is merged into the G = 4 main launch).
template <typename R, typename Acc, int SPEC, bool DET, bool OVF>
struct PackedShared {
  static constexpr int kRows = kMaxSpecies * kMaxSpecies * kMaxSpecies;
  Row<R> srow[SPEC == kSingle ? 1 : kRows];
  double scut[SPEC == kSingle ? 1 : kRows];
  Stage<R> st;
  double s_r2[SPEC == kGeneric ? kBlock : 1];
  Acc s_seg[(OVF && DET) ? 7 : 3][kBlock];   // segmented sums
  int s_buf[OVF ? kBlock / 32 : 1][128];     // scanning tier: slots, counts
};

// The packed lane groups' work of one block (main: chunks of consecutive
// slots; OVF: the atoms over the main width, found by scanning the counts),
// accumulating energy and virial into e_acc / w_acc.
template <typename R, typename Acc, int SPEC, bool DET, bool OVF, bool FOREIGN, bool VIR>
__device__ __forceinline__ void packed_work(const ForceArgs<R>& a,
                                            PackedShared<R, Acc, SPEC, DET, OVF>& sh, Acc& e_acc,
                                            Acc (&w_acc)[6]) {
  constexpr int kC = kPackedCacheRot<R>;
  // next-pack lookahead (below): float liquid -4%, single -5%; the FP64
  // kernels spill with it (SiC f64 +4%) and keep the plain order
  constexpr bool kAhead = TSF_PACKED_AHEAD && !std::is_same<R, double>::value;
  auto& srow = sh.srow;
  auto& scut = sh.scut;
  auto& st = sh.st;
  auto& s_r2 = sh.s_r2;
  auto& s_seg = sh.s_seg;
  auto& s_buf = sh.s_buf;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wbase = tid - lane;

  const int ns = a.ns;
  const Row<R>* rows = static_cast<const Row<R>*>(a.rows);
  const Row<R>& row0 = a.row0;
  const double cut0 = a.cut0;
  if (SPEC != kSingle) {
    for (int q = tid; q < ns * ns * ns; q += blockDim.x) {
      srow[q] = rows[q];
      scut[q] = a.cutsq[q];
    }
    __syncthreads();
  }
  const int last = a.n_all - 1;
  const bool has_ghosts = a.center_limit < a.n_owned;
  const bool has_foreign = FOREIGN && a.energy_limit < a.center_limit;
  const int nwarps = gridDim.x * (kBlock / 32);
  const int warp = blockIdx.x * (kBlock / 32) + tid / 32;

  // One chunk: this lane's atom i (slot) with short count n (0: none) and its
  // ghost-centre bit; the warp sorts, scans and packs the chunk's slots.
  auto chunk_body = [&](int i, int n, int fgn) {
    if constexpr (OVF) {
      // the chunk's neighbour positions, one lane per atom, before the packs
      // walk them serially
      if (n > 0) {
        const int4 e = *reinterpret_cast<const int4*>(a.nbr + ell_at(0, i, a.npad));
        prefetch_l2(&a.pos[min(max(e.x, 0), last)]);
        prefetch_l2(&a.pos[min(max(e.y, 0), last)]);
        prefetch_l2(&a.pos[min(max(e.z, 0), last)]);
        prefetch_l2(&a.pos[min(max(e.w, 0), last)]);
        for (int q = 4; q < n; ++q) prefetch_l2(&a.pos[min(max(a.nbr[ell_at(q, i, a.npad)], 0), last)]);
      }
    }
    {
      // order the chunk's atoms by count (bitonic, key (n, lane): unique, so
      // deterministic): a pack then holds atoms of similar counts, and its
      // rotations stop at a largest count that fits most of its lanes
      int key = (n << 5) | lane;
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          const int other = __shfl_xor_sync(kFull, key, jj);
          const bool up = (lane & k) == 0, lower = (lane & jj) == 0;
          key = (lower == up) ? min(key, other) : max(key, other);
        }
      const int src = key & 31;
      i = __shfl_sync(kFull, i, src);
      n = __shfl_sync(kFull, n, src);
      fgn = __shfl_sync(kFull, fgn, src);
    }
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const int excl = incl - n;
    const int total = __shfl_sync(kFull, incl, 31);

    // Pack p's lane map without shared memory: the chunk is sorted by count,
    // so its zero-count atoms come first and pack p's atoms are the next
    // popc(heads) in sorted order; lane L's atom is the one whose segment
    // head is the highest head bit at or below L.  The next pack's map and
    // list entry are formed while this pack computes, its positions requested
    // after the zeta pass (one dependent load chain per pack was the packed
    // kernels' long-scoreboard stall).
    struct PackLane {
      int used, kb_next, h, gl, ai, ni, v;
      bool slot, foreign;
    };
    auto pack_at = [&](int base, int kb, PackLane& P) {
      const bool mine = n > 0 && excl >= base && incl <= base + 32;
      const unsigned heads = __reduce_or_sync(kFull, mine ? 1u << (excl - base) : 0u);
      P.used = int(__reduce_max_sync(kFull, mine ? unsigned(incl - base) : 0u));
      const unsigned le = heads & (0xffffffffu >> (31 - lane));   // bit 0 is set
      P.h = 31 - __clz(le);
      const int k = (kb + __popc(le) - 1) & 31;
      P.kb_next = kb + __popc(heads);
      P.slot = lane < P.used;
      P.ai = __shfl_sync(kFull, i, k);
      const int nk = __shfl_sync(kFull, n, k);
      P.foreign = FOREIGN && __shfl_sync(kFull, fgn, k);
      P.ni = P.slot ? nk : 0;
      P.gl = lane - P.h;
      TSF_DCHECK(!heads || (P.h >= 0 && P.h <= lane && P.ai >= 0 && P.ai <= last),
                 "k_force_packed segment head");
      TSF_DCHECK(!P.slot || (P.gl < P.ni && P.ni <= 32), "k_force_packed segment slot");
      P.v = P.slot ? a.nbr[ell_at(P.gl, P.ai, a.npad)] : P.ai;
    };
    if (total == 0) return;                       // warp-uniform: no slot in the chunk
    PackLane cur;
    pack_at(0, __popc(__ballot_sync(kFull, n == 0)), cur);
    double4 pi_c, pj_c;
    {
      const int j0 = unsigned(cur.v) <= unsigned(last) ? cur.v : cur.ai;
      pi_c = a.pos[cur.ai];
      pj_c = a.pos[j0];
    }
    for (int base = 0; base < total;) {           // warp-uniform: one pack per pass
      const bool slot = cur.slot;
      const int ai = cur.ai, ni = cur.ni, h = cur.h, gl = cur.gl, used = cur.used;
      const bool foreign = cur.foreign;
      const int v = cur.v;
      TSF_DCHECK(!slot || (v >= 0 && v <= last && v != ai), "k_force_packed list entry");
      const int j = unsigned(v) <= unsigned(last) ? v : ai;
      const double4 pi = pi_c;
      const double4 pj = pj_c;
      // the next pack: lane map and list entry now, positions after the zeta pass
      const bool more = base + used < total;   // warp-uniform
      PackLane nxt = cur;
      if (kAhead && more) pack_at(base + used, cur.kb_next, nxt);

      double dx = 0, dy = 0, dz = 0, r2 = 1.0;
      if (slot) {
        displacement(pi, pj, a.box, dx, dy, dz);
        r2 = norm_sq_exact(dx, dy, dz);
      }
      const int si = SPEC == kSingle ? 0 : species_of(pi);
      const int sj = SPEC == kSingle ? 0 : species_of(pj);
      const int row_jj = (si * ns + sj) * ns + sj;
      const bool pair_ok = slot && r2 <= (SPEC == kSingle ? cut0 : scut[row_jj]);
      const Row<R>& pjj = SPEC == kSingle ? row0 : srow[row_jj];
      Nbr<R> me;
      me.ir = Fn<R>::rsqrt_(R(r2));
      me.r = R(r2) * me.ir;
      me.ux = R(dx) * me.ir;
      me.uy = R(dy) * me.ir;
      me.uz = R(dz) * me.ir;
      R fc, dfc;
      cutoff_ramp<R, true>(me.r, pjj, fc, dfc);
      const R fr = pjj.a * Fn<R>::exp_row(pjj.e1 * me.r);
      const R fa = -(pjj.b * Fn<R>::exp_row(pjj.e2 * me.r));
      const int meta = SPEC == kGeneric ? (slot ? sj : -1) : (pair_ok ? sj : -1);
      st.put(tid, me, fc, dfc, meta);
      if (SPEC == kGeneric) s_r2[tid] = r2;
      __syncwarp();
      const int rowbase = (si * ns + sj) * ns;
      const int tmax = int(__reduce_max_sync(kFull, unsigned(ni)));

      // partner of rotation t inside this lane's segment (itself once t >= n:
      // its triplet is masked and its k-gradient is zero)
      auto triplet_at = [&](int t, Nbr<R>& k) {
        int m = gl;
        if (t < ni) {
          m = gl + t;
          if (m >= ni) m -= ni;
        }
        const int src = wbase + h + m;
        R fck, dfck;
        int kmeta;
        st.get(src, k, fck, dfck, kmeta);
        bool ok = pair_ok && t < ni && kmeta >= 0;
        const Row<R>* prow = &pjj;
        if (SPEC != kSingle) {
          const int sk = max(kmeta, 0);
          prow = &srow[rowbase + sk];
          if (SPEC == kGeneric) {
            ok = ok && s_r2[src] <= scut[rowbase + sk];
            cutoff_ramp<R, true>(k.r, *prow, fck, dfck);
          }
        }
        fck = ok ? fck : R(0);
        dfck = ok ? dfck : R(0);
        return triplet<R, (SPEC == kSingle ? 1 : -1)>(me, k, fck, dfck, ok, *prow);
      };

      // ---- zeta pass ----
      // (k_force's scalar form: j-gradient u_j sum(B) + sum(u_k A), k-cache (C, D))
      R zeta = 0, sb = 0, gjx = 0, gjy = 0, gjz = 0;
      R ckc[kC + 1], ckd[kC + 1];
      auto accumulate = [&](const Grad<R>& tr, const Nbr<R>& k) {
        zeta += tr.z;
        sb += tr.B;
        gjx += k.ux * tr.A;
        gjy += k.uy * tr.A;
        gjz += k.uz * tr.A;
      };
#pragma unroll
      for (int t = 1; t <= kC; ++t) {
        ckc[t] = ckd[t] = R(0);
        if (t < tmax) {
          Nbr<R> k;
          const Grad<R> tr = triplet_at(t, k);
          accumulate(tr, k);
          ckc[t] = tr.C;
          ckd[t] = tr.D;
        }
      }
      for (int t = kC + 1; t < tmax; ++t) {
        Nbr<R> k;
        accumulate(triplet_at(t, k), k);
      }

      if (kAhead && more) {
        const int jn = unsigned(nxt.v) <= unsigned(last) ? nxt.v : nxt.ai;
        pi_c = a.pos[nxt.ai];
        pj_c = a.pos[jn];
      }

      // ---- pair block ----
      R dvdr = 0, dvdz = 0, vv = 0;
      if (pair_ok) {
        const R dfr = -pjj.lam1 * fr;
        const R dfa = -pjj.lam2 * fa;
        R b, db;
        bond_order(zeta, pjj, b, db);
        const R rep = fr + b * fa;
        vv = R(0.5) * fc * rep;
        dvdr = R(0.5) * (dfc * rep + fc * (dfr + b * dfa));
        dvdz = R(0.5) * fc * fa * db;
        // one test, as in k_force: a non-finite term makes the sum non-finite
        if (!isfinite(vv + dvdr + dvdz)) atomicOr(a.flags, kErrNonFinite);
      }
      R alpha = dvdr + dvdz * sb;
      R px = -(gjx * dvdz);
      R py = -(gjy * dvdz);
      R pz = -(gjz * dvdz);

      // ---- scatter: lane h + (gl - t) mod n sends its rotation-t (C, D) dV/dzeta ----
      auto receive = [&](int t, R sc, R sd) {
        int s = gl;
        if (t < ni) {
          s = gl - t;
          if (s < 0) s += ni;
        }
        const int from = h + s;
        const R rc = __shfl_sync(kFull, sc, from);
        alpha += __shfl_sync(kFull, sd, from);
        R sux, suy, suz;
        st.unit(wbase + from, sux, suy, suz);
        px -= sux * rc;
        py -= suy * rc;
        pz -= suz * rc;
      };
#pragma unroll
      for (int t = 1; t <= kC; ++t)
        if (t < tmax) receive(t, ckc[t] * dvdz, ckd[t] * dvdz);
      for (int t = kC + 1; t < tmax; ++t) {
        Nbr<R> k;
        const Grad<R> tr = triplet_at(t, k);
        receive(t, tr.C * dvdz, tr.D * dvdz);
      }
      px -= me.ux * alpha;
      py -= me.uy * alpha;
      pz -= me.uz * alpha;
      if (!slot) px = py = pz = 0;

      // ---- F_i = -sum of the segment's P (and, queued + deterministic, the
      // atom's energy and virial), summed by the head lane in slot order ----
      const R rx = R(dx), ry = R(dy), rz = R(dz);
      // FP64 atomic mode: each slot lane adds -P to F_i itself (three more
      // reductions per slot instead of the head lane's serial segment sum,
      // which ran max(n_i) iterations with one lane in 32 active: -5% on the
      // f64 SiC and liquid kernels; the float kernels measured +1%, so they
      // keep the sum); deterministic mode sums in slot order
      constexpr bool kLaneAtomics = !DET && std::is_same<R, double>::value;
      if (!kLaneAtomics) {
        s_seg[0][tid] = Acc(px);
        s_seg[1][tid] = Acc(py);
        s_seg[2][tid] = Acc(pz);
      }
      if constexpr (OVF && DET) {
        const bool cnt_ev = slot && !(FOREIGN && foreign);
        const bool cnt_w = cnt_ev && VIR;   // (virial-free callers: zeros)
        s_seg[3][tid] = cnt_ev ? Acc(vv) : Acc(0);
        s_seg[4][tid] = cnt_w ? Acc(rx * px) : Acc(0);
        s_seg[5][tid] = cnt_w ? Acc(ry * py) : Acc(0);
        s_seg[6][tid] = cnt_w ? Acc(rz * pz) : Acc(0);
        // the three off-diagonal components follow in a second round below
      }
      __syncwarp();
      Acc fsum[3] = {0, 0, 0};
      Acc evsum[7] = {0, 0, 0, 0, 0, 0, 0};
      const bool head = slot && gl == 0;
      TSF_DCHECK(!head || lane + ni <= 32, "k_force_packed segment sum");
      if (!kLaneAtomics && head) {
        for (int u = 0; u < ni; ++u) {
          fsum[0] += s_seg[0][tid + u];
          fsum[1] += s_seg[1][tid + u];
          fsum[2] += s_seg[2][tid + u];
          if constexpr (OVF && DET) {
            evsum[0] += s_seg[3][tid + u];
            evsum[1] += s_seg[4][tid + u];
            evsum[2] += s_seg[5][tid + u];
            evsum[3] += s_seg[6][tid + u];
          }
        }
      }
      if constexpr (OVF && DET) {
        __syncwarp();
        const bool cnt_w = slot && !(FOREIGN && foreign) && VIR;
        s_seg[3][tid] = cnt_w ? Acc(rx * py) : Acc(0);
        s_seg[4][tid] = cnt_w ? Acc(rx * pz) : Acc(0);
        s_seg[5][tid] = cnt_w ? Acc(ry * pz) : Acc(0);
        __syncwarp();
        if (head)
          for (int u = 0; u < ni; ++u) {
            evsum[4] += s_seg[3][tid + u];
            evsum[5] += s_seg[4][tid + u];
            evsum[6] += s_seg[5][tid + u];
          }
        if (head)
#pragma unroll
          for (int w = 0; w < 7; ++w) a.atom_ev[8 * std::size_t(ai) + w] = double(evsum[w]);
      }
      if (slot) {
        if constexpr (!(OVF && DET)) if (!FOREIGN || !foreign) {
          e_acc += Acc(vv);
          if constexpr (VIR) {
            w_acc[0] += Acc(rx * px);
            w_acc[1] += Acc(ry * py);
            w_acc[2] += Acc(rz * pz);
            w_acc[3] += Acc(rx * py);
            w_acc[4] += Acc(rx * pz);
            w_acc[5] += Acc(ry * pz);
          }
        }
        if (DET) {
          const std::size_t qs = std::size_t(gl) * a.npad + ai;
          static_cast<Acc*>(a.slot_x)[qs] = Acc(px);
          static_cast<Acc*>(a.slot_y)[qs] = Acc(py);
          static_cast<Acc*>(a.slot_z)[qs] = Acc(pz);
        } else {
          Acc* f = static_cast<Acc*>(a.forces) + 3 * std::size_t(j);
          atomicAdd(f + 0, Acc(px));
          atomicAdd(f + 1, Acc(py));
          atomicAdd(f + 2, Acc(pz));
          if constexpr (kLaneAtomics) {
            Acc* fi = static_cast<Acc*>(a.forces) + 3 * std::size_t(ai);
            atomicAdd(fi + 0, -Acc(px));
            atomicAdd(fi + 1, -Acc(py));
            atomicAdd(fi + 2, -Acc(pz));
          }
        }
      }
      if (!kLaneAtomics && head) {
        if (DET) {
          Acc* f = static_cast<Acc*>(a.fself) + 3 * std::size_t(ai);
          f[0] = -fsum[0];
          f[1] = -fsum[1];
          f[2] = -fsum[2];
        } else {
          Acc* f = static_cast<Acc*>(a.forces) + 3 * std::size_t(ai);
          atomicAdd(f + 0, -fsum[0]);
          atomicAdd(f + 1, -fsum[1]);
          atomicAdd(f + 2, -fsum[2]);
        }
      }
      if (!kAhead && more) {
        pack_at(base + used, cur.kb_next, nxt);
        const int jn = unsigned(nxt.v) <= unsigned(last) ? nxt.v : nxt.ai;
        pi_c = a.pos[nxt.ai];
        pj_c = a.pos[jn];
      }
      base += used;
      cur = nxt;
      __syncwarp();                      // staging is rewritten by the next pack
    }
  };

  if constexpr (OVF) {
    if (a.over4 && *a.over4 == 0) return;  // the filter saw no count over 4
    // ---- tier launch behind a width-G main launch: the atoms it left are
    // exactly the owned centres with more than scan_g short entries.  Each
    // warp scans its own contiguous slot range (counts coalesced, 32 per
    // step), compacts those atoms in slot order into a per-warp buffer and
    // runs a chunk whenever 32 are waiting — no queue, no atomics (a queue
    // fed by one counter serialised 180k same-address atomics in the main
    // launch at 1600 K), and neighbouring atoms share their gathers ----
    int* bi = s_buf[tid / 32];
    int* bn = s_buf[tid / 32] + 64;
    const int lo = a.slot_base, hi = a.n_owned;
    const int per = ((hi - lo + nwarps - 1) / nwarps + 31) & ~31;
    const int w0 = lo + warp * per, w1 = min(hi, w0 + per);
    int nb = 0, s0 = w0;                         // warp-uniform
    while (true) {
      while (nb < 32 && s0 < w1) {               // fill the buffer to a chunk
        const int sl = s0 + lane;
        int c = sl < w1 ? a.cnt[sl] : 0;
        if (c > a.scan_g && has_ghosts && (a.perm ? a.perm[sl] : sl) >= a.center_limit) c = 0;
        const bool over = c > a.scan_g;
        const unsigned m = __ballot_sync(kFull, over);
        if (over) {
          const int q = nb + __popc(m & ((1u << lane) - 1u));
          bi[q] = sl;
          bn[q] = c;
          // into L2 while the chunk fills: the atom's position and list
          // blocks (the tier's atoms are sparse: its loads missed L1 81%
          // and L2 57% of the time, long-scoreboard stalls 3.5 per issue)
          prefetch_l2(&a.pos[sl]);
          prefetch_l2(a.nbr + ell_at(0, sl, a.npad));
          if (c > 4) prefetch_l2(a.nbr + ell_at(4, sl, a.npad));
        }
        nb += __popc(m);
        s0 += 32;
      }
      if (nb == 0) break;
      __syncwarp();
      const int take = min(nb, 32);
      const bool in = lane < take;
      const int i = in ? bi[lane] : 0;
      int n = in ? bn[lane] : 0;
      __syncwarp();
      if (lane < nb - 32) {                      // keep the rest (at most 31)
        bi[lane] = bi[32 + lane];
        bn[lane] = bn[32 + lane];
      }
      nb -= take;
      if (n > 32) {                              // no wider launch behind this one
        atomicOr(a.flags, kErrShortOverflow);
        n = 0;
      }
      const int fgn = has_foreign && in && (a.perm ? a.perm[i] : i) >= a.energy_limit;
      chunk_body(i, n, fgn);
    }
  } else {
    // the main launch: chunks of 32 consecutive slots
    const int items = a.n_owned - a.slot_base;
    constexpr int cw = 32;
    const int chunks = (items + cw - 1) / cw;
    for (int chunk = warp; chunk < chunks; chunk += nwarps) {
      // ---- this lane's atom of the chunk and its count ----
      const int q = chunk * cw + lane;
      const bool in = lane < cw && q < items;
      const int i = in ? a.slot_base + q : 0;
      int n = in ? a.cnt[i] : 0;
      if (!OVF && has_ghosts && in && (a.perm ? a.perm[i] : i) >= a.center_limit) {
        // a decomposition ghost copy: receives forces, is not a centre
        if (DET) {   // zero its self term and the slots k_gather reads
          Acc* f = static_cast<Acc*>(a.fself) + 3 * std::size_t(i);
          f[0] = f[1] = f[2] = Acc(0);
          for (int sl = 0; sl < n; ++sl) {
            const std::size_t qs = std::size_t(sl) * a.npad + i;
            static_cast<Acc*>(a.slot_x)[qs] = Acc(0);
            static_cast<Acc*>(a.slot_y)[qs] = Acc(0);
            static_cast<Acc*>(a.slot_z)[qs] = Acc(0);
          }
        }
        n = 0;
      }
      if (n > 32) {                        // no wider launch behind this one
        atomicOr(a.flags, kErrShortOverflow);
        n = 0;
      }
      if (DET && in && n == 0) {           // no segment, no head: F_self = 0 here
        Acc* f = static_cast<Acc*>(a.fself) + 3 * std::size_t(i);
        f[0] = f[1] = f[2] = Acc(0);
      }
      const int fgn = has_foreign && in && (a.perm ? a.perm[i] : i) >= a.energy_limit;
      chunk_body(i, n, fgn);
    }
  }
}

template <typename R, typename Acc, int SPEC, bool DET, bool OVF, bool FOREIGN = false,
          bool VIR = true>
__global__ void __launch_bounds__(kBlock, kPackedMinBlocks<R>)
    k_force_packed(const __grid_constant__ ForceArgs<R> a) {
  __shared__ PackedShared<R, Acc, SPEC, DET, OVF> sh;
  __shared__ double s_red[kBlock / 32][kRedWidth];

  griddep_wait();
  griddep_launch();
  if (a.skip && (a.skip[0] | a.skip[kFlagMovedAny - kFlagMoved])) return;   // stale list
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (OVF && a.over4 && *a.over4 == 0) {   // the filter saw no count over 4
    if (tid < kRedWidth)
      a.partials[std::size_t(a.partial_base + blockIdx.x) * kRedWidth + tid] = 0.0;
    return;
  }
  Acc e_acc = 0;
  Acc w_acc[6] = {0, 0, 0, 0, 0, 0};
  packed_work<R, Acc, SPEC, DET, OVF, FOREIGN, VIR>(a, sh, e_acc, w_acc);

  // ---- block reduction of energy + virial, fixed order ----
  double red[7] = {double(e_acc), double(w_acc[0]), double(w_acc[1]), double(w_acc[2]),
                   double(w_acc[3]), double(w_acc[4]), double(w_acc[5])};
#pragma unroll
  for (int qq = 0; qq < 7; ++qq)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) red[qq] += __shfl_down_sync(kFull, red[qq], o);
  if (lane == 0)
#pragma unroll
    for (int qq = 0; qq < 7; ++qq) s_red[tid / 32][qq] = red[qq];
  __syncthreads();
  if (tid < kRedWidth) {
    double s = 0;
    if (tid < 7)
      for (int w = 0; w < kBlock / 32; ++w) s += s_red[w][tid];
    a.partials[std::size_t(a.partial_base + blockIdx.x) * kRedWidth + tid] = s;
  }
}

}  // namespace
}  // namespace tsf
