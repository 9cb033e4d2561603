/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the Tersoff force path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this file (via oracle/oracle.py).  The product never links it and
 * never falls back to it.
 *
 * A plain-C restatement of the reference algorithm (arXiv 1607.02904 Alg. 2
 * as implemented in /root/reference/proj), expression for expression, so that
 * built with -ffp-contract=off against the same glibc it reproduces the
 * reference's bits.  Pinned against:
 *   - the reference library itself (oracle/_ref, built by oracle/Makefile),
 *   - the SURVEY.md Appendix D hexfloat goldens (tests/test_oracle.py).
 *
 * Citations are to /root/reference/proj.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ParamField column layout, include/tmd/params.hpp:78-83 */
enum { F_A = 0, F_B, F_LAM1, F_LAM2, F_LAM3, F_BETA, F_ETA, F_C, F_D, F_H,
       F_GAMMA, F_M, F_BIGR, F_BIGD, F_CUT, F_CUTSQ, F_COUNT };

#define ORC_OK 0
#define ORC_CONFIG 2
#define ORC_NUMERIC 3
#define ORC_NOMEM 4

static const double kPi = 3.14159265358979323846;

/* include/tmd/box.hpp:28-30 */
static double min_image_1d(double d, double len) { return d - len * floor(d / len + 0.5); }

static void min_image(double d[3], const double box[3], const uint8_t per[3]) {
  if (per[0]) d[0] = min_image_1d(d[0], box[0]);
  if (per[1]) d[1] = min_image_1d(d[1], box[1]);
  if (per[2]) d[2] = min_image_1d(d[2], box[2]);
}

/* include/tmd/vec3.hpp:25-30 */
static double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

static void delta(const double* xyz, int64_t a, int64_t b, const double box[3],
                  const uint8_t per[3], double d[3]) {
  d[0] = xyz[3 * b + 0] - xyz[3 * a + 0];
  d[1] = xyz[3 * b + 1] - xyz[3 * a + 1];
  d[2] = xyz[3 * b + 2] - xyz[3 * a + 2];
  min_image(d, box, per);
}

/* ---------------------------------------------------------------------
   bond-order math, include/tmd/potential.hpp:58-222 (scalar double)
   --------------------------------------------------------------------- */

/* potential.hpp:58-69 */
void orc_cutoff_fc(double r, double big_r, double big_d, double* value, double* deriv) {
  const double arg = (kPi / 2) * ((r - big_r) / big_d);
  const double ramp = 0.5 - 0.5 * sin(arg);
  const double dramp = ((-kPi / 4) / big_d) * cos(arg);
  const int below = r <= big_r - big_d;
  const int above = r >= big_r + big_d;
  *value = below ? 1.0 : (above ? 0.0 : ramp);
  *deriv = (below | above) ? 0.0 : dramp;
}

/* potential.hpp:75-82 */
static void pair_terms(double r, const double* p, double* fr, double* dfr, double* fa,
                       double* dfa) {
  *fr = p[F_A] * exp(-p[F_LAM1] * r);
  *dfr = -p[F_LAM1] * *fr;
  *fa = -(p[F_B] * exp(-p[F_LAM2] * r));
  *dfa = -p[F_LAM2] * *fa;
}

/* potential.hpp:88-96 */
static void angle_g(double cos_theta, const double* p, double* g, double* dg) {
  const double c2 = p[F_C] * p[F_C];
  const double d2 = p[F_D] * p[F_D];
  const double t = p[F_H] - cos_theta;
  const double denom = d2 + t * t;
  *g = p[F_GAMMA] * (1.0 + c2 / d2 - c2 / denom);
  *dg = p[F_GAMMA] * (-2.0 * c2 * t) / (denom * denom);
}

/* potential.hpp:107-120 */
void orc_bond_order(double zeta, const double* p, double* value, double* deriv) {
  const int at_zero = zeta <= 0.0;
  const double zs = at_zero ? 1.0 : zeta;
  const double u = pow(p[F_BETA] * zs, p[F_ETA]);
  const double base = 1.0 + u;
  const double half_inv_eta = -0.5 / p[F_ETA];
  const double b = pow(base, half_inv_eta);
  const double db = -0.5 * pow(base, half_inv_eta - 1.0) * u / zs;
  *value = at_zero ? 1.0 : b;
  *deriv = at_zero ? 0.0 : db;
}

typedef struct {
  double fc, dfc, g, dg, ex, dex, cos_theta;
  double u_ij[3], u_ik[3];
  double inv_rij, inv_rik;
} ZetaParts;

/* std::min / std::max argument order, potential.hpp:155 */
static double smax(double a, double b) { return (a < b) ? b : a; }
static double smin(double a, double b) { return (b < a) ? b : a; }

/* potential.hpp:132-162 */
static void zeta_parts(const double dij[3], double rij, const double dik[3], double rik,
                       const double* p, ZetaParts* zp) {
  zp->inv_rij = 1.0 / rij;
  zp->inv_rik = 1.0 / rik;
  for (int c = 0; c < 3; ++c) {
    zp->u_ij[c] = dij[c] * zp->inv_rij;
    zp->u_ik[c] = dik[c] * zp->inv_rik;
  }
  zp->cos_theta = smin(1.0, smax(-1.0, dot3(zp->u_ij, zp->u_ik)));
  orc_cutoff_fc(rik, p[F_BIGR], p[F_BIGD], &zp->fc, &zp->dfc);
  angle_g(zp->cos_theta, p, &zp->g, &zp->dg);
  const double t = p[F_LAM3] * (rij - rik);
  const int cubic = p[F_M] > 2.0;
  zp->ex = exp(cubic ? t * t * t : t);
  zp->dex = zp->ex * p[F_LAM3] * (cubic ? 3.0 * t * t : 1.0);
}

/* potential.hpp:165-170 */
static double zeta_value(const double dij[3], double rij, const double dik[3], double rik,
                         const double* p) {
  ZetaParts zp;
  zeta_parts(dij, rij, dik, rik, p, &zp);
  return zp.fc * zp.g * zp.ex;
}

/* potential.hpp:178-198 */
void orc_zeta_term(const double dij[3], double rij, const double dik[3], double rik,
                   const double* p, double* zeta, double gi[3], double gj[3], double gk[3]) {
  ZetaParts zp;
  zeta_parts(dij, rij, dik, rik, p, &zp);
  *zeta = zp.fc * zp.g * zp.ex;
  double gc_j[3], gc_k[3], gc_i[3];
  for (int c = 0; c < 3; ++c) {
    gc_j[c] = (zp.u_ik[c] - zp.u_ij[c] * zp.cos_theta) * zp.inv_rij;
    gc_k[c] = (zp.u_ij[c] - zp.u_ik[c] * zp.cos_theta) * zp.inv_rik;
  }
  for (int c = 0; c < 3; ++c) gc_i[c] = 0.0 - (gc_j[c] + gc_k[c]);
  const double fgd = zp.fc * zp.dg * zp.ex;
  const double fge = zp.fc * zp.g * zp.dex;
  const double cge = zp.dfc * zp.g * zp.ex;
  for (int c = 0; c < 3; ++c) {
    gj[c] = gc_j[c] * fgd + zp.u_ij[c] * fge;
    gk[c] = zp.u_ik[c] * cge + gc_k[c] * fgd - zp.u_ik[c] * fge;
    gi[c] = (0.0 - zp.u_ik[c] * cge) + gc_i[c] * fgd + (zp.u_ik[c] - zp.u_ij[c]) * fge;
  }
}

/* potential.hpp:211-222 */
static void pair_v_terms(double r, double zeta, const double* p, double* energy,
                         double* dv_dr, double* dv_dzeta) {
  double fc, dfc, fr, dfr, fa, dfa, b, db;
  orc_cutoff_fc(r, p[F_BIGR], p[F_BIGD], &fc, &dfc);
  pair_terms(r, p, &fr, &dfr, &fa, &dfa);
  orc_bond_order(zeta, p, &b, &db);
  *energy = 0.5 * fc * (fr + b * fa);
  *dv_dr = 0.5 * (dfc * (fr + b * fa) + fc * (dfr + b * dfa));
  *dv_dzeta = 0.5 * fc * fa * db;
}

/* ---------------------------------------------------------------------
   compute_ref, src/potential_ref.cpp:75-142 (paper Alg. 2)

   `rows` is FlatParams<double> (params.hpp:88-115): ns^3 rows of 16.
   Outputs: energy (naive running sum, bitwise the reference's), energy_ld
   (the same terms summed in long double — the compensated oracle of
   SURVEY.md Appendix E), forces (n*3), virial (6: xx yy zz xy xz yz,
   W_ab = sum over force contributions of d_a f_b with d relative to the
   central atom i; NEW — parity unpinned by the reference, checked against
   finite strain derivatives in the tests).  Returns ORC_NUMERIC with
   bad_i / bad_j set on a non-finite pair term (potential_ref.cpp:109-112).
   --------------------------------------------------------------------- */
int orc_compute_ref(int64_t n, int64_t n_center, const double* xyz, const int32_t* species,
                    const double box[3], const uint8_t per[3], int ns,
                    const double* rows, const int32_t* offsets, const int32_t* nbrs,
                    double* energy, long double* energy_ld, double* forces,
                    double* virial, int64_t* bad_i, int64_t* bad_j) {
  /* n_center < n: only atoms [0, n_center) act as central atoms (the
     decomposition tests' owned atoms; the rest are ghost copies). */
  double e = 0.0;
  long double eld = 0.0L;
  long double w[6] = {0, 0, 0, 0, 0, 0};
  memset(forces, 0, sizeof(double) * 3 * (size_t)n);
  for (int64_t i = 0; i < n_center; ++i) {
    const int si = species[i];
    const int32_t s0 = offsets[i], s1 = offsets[i + 1];
    for (int32_t sj_pos = s0; sj_pos < s1; ++sj_pos) {
      const int32_t j = nbrs[sj_pos];
      const int sj = species[j];
      const double* pij = rows + (size_t)((si * ns + sj) * ns + sj) * F_COUNT;
      double dij[3];
      delta(xyz, i, j, box, per, dij);
      const double r2 = dot3(dij, dij);
      if (r2 > pij[F_CUTSQ]) continue;
      const double rij = sqrt(r2);

      double zeta = 0.0;
      for (int32_t kp = s0; kp < s1; ++kp) {
        const int32_t k = nbrs[kp];
        if (k == j) continue;
        const int sk = species[k];
        const double* pijk = rows + (size_t)((si * ns + sj) * ns + sk) * F_COUNT;
        double dik[3];
        delta(xyz, i, k, box, per, dik);
        const double r2k = dot3(dik, dik);
        if (r2k > pijk[F_CUTSQ]) continue;
        zeta += zeta_value(dij, rij, dik, sqrt(r2k), pijk);
      }

      double pe, dv_dr, dv_dz;
      pair_v_terms(rij, zeta, pij, &pe, &dv_dr, &dv_dz);
      if (!isfinite(pe) || !isfinite(dv_dr) || !isfinite(dv_dz)) {
        if (bad_i) *bad_i = i;
        if (bad_j) *bad_j = j;
        return ORC_NUMERIC;
      }
      e += pe;
      eld += (long double)pe;
      const double inv = 1.0 / rij;
      double fp[3];
      for (int c = 0; c < 3; ++c) {
        fp[c] = (dij[c] * inv) * dv_dr;
        forces[3 * i + c] += fp[c];
        forces[3 * (int64_t)j + c] -= fp[c];
      }
      /* virial of the radial pair: f_j = -fp at d_ij */
      w[0] -= (long double)dij[0] * fp[0];
      w[1] -= (long double)dij[1] * fp[1];
      w[2] -= (long double)dij[2] * fp[2];
      w[3] -= (long double)dij[0] * fp[1];
      w[4] -= (long double)dij[0] * fp[2];
      w[5] -= (long double)dij[1] * fp[2];

      for (int32_t kp = s0; kp < s1; ++kp) {
        const int32_t k = nbrs[kp];
        if (k == j) continue;
        const int sk = species[k];
        const double* pijk = rows + (size_t)((si * ns + sj) * ns + sk) * F_COUNT;
        double dik[3];
        delta(xyz, i, k, box, per, dik);
        const double r2k = dot3(dik, dik);
        if (r2k > pijk[F_CUTSQ]) continue;
        double z, gi[3], gj[3], gk[3];
        orc_zeta_term(dij, rij, dik, sqrt(r2k), pijk, &z, gi, gj, gk);
        double fj[3], fk[3];
        for (int c = 0; c < 3; ++c) {
          forces[3 * i + c] -= gi[c] * dv_dz;
          fj[c] = gj[c] * dv_dz;
          fk[c] = gk[c] * dv_dz;
          forces[3 * (int64_t)j + c] -= fj[c];
          forces[3 * (int64_t)k + c] -= fk[c];
        }
        w[0] -= (long double)dij[0] * fj[0] + (long double)dik[0] * fk[0];
        w[1] -= (long double)dij[1] * fj[1] + (long double)dik[1] * fk[1];
        w[2] -= (long double)dij[2] * fj[2] + (long double)dik[2] * fk[2];
        w[3] -= (long double)dij[0] * fj[1] + (long double)dik[0] * fk[1];
        w[4] -= (long double)dij[0] * fj[2] + (long double)dik[0] * fk[2];
        w[5] -= (long double)dij[1] * fj[2] + (long double)dik[1] * fk[2];
      }
    }
  }
  *energy = e;
  if (energy_ld) *energy_ld = eld;
  if (virial)
    for (int c = 0; c < 6; ++c) virial[c] = (double)w[c];
  return ORC_OK;
}

/* ---------------------------------------------------------------------
   neighbor lists, src/neighbor.cpp:37-180
   --------------------------------------------------------------------- */

typedef struct {
  int32_t* v;
  int64_t n, cap;
} IVec;

static int ivec_push(IVec* a, int32_t x) {
  if (a->n == a->cap) {
    int64_t nc = a->cap ? 2 * a->cap : 16;
    int32_t* nv = (int32_t*)realloc(a->v, sizeof(int32_t) * (size_t)nc);
    if (!nv) return 0;
    a->v = nv;
    a->cap = nc;
  }
  a->v[a->n++] = x;
  return 1;
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static int clamp_cell(double frac, int n) {
  int c = (int)floor(frac * n);
  return c < 0 ? 0 : (c > n - 1 ? n - 1 : c);
}

/* Full, symmetric, ascending skin list (neighbor.cpp:37-132).  Writes
   offsets[n+1]; nbrs is malloc'd and returned through *out_nbrs (free with
   orc_free).  Returns ORC_CONFIG for the reference's ConfigError cases. */
int orc_build_neighbor_list(int64_t n, const double* xyz, const double box[3],
                            const uint8_t per[3], double cutoff, double skin,
                            int32_t* offsets, int32_t** out_nbrs, int64_t* out_total) {
  if (!(cutoff > 0.0)) return ORC_CONFIG;
  if (skin < 0.0) return ORC_CONFIG;
  if (!(box[0] > 0.0) || !(box[1] > 0.0) || !(box[2] > 0.0)) return ORC_CONFIG;
  const double bc = cutoff + skin;
  const double bc_sq = bc * bc;
  for (int ax = 0; ax < 3; ++ax)
    if (per[ax] && box[ax] < 2.0 * bc) return ORC_CONFIG;

  double lo[3] = {0.0, 0.0, 0.0}, hi[3] = {box[0], box[1], box[2]};
  for (int ax = 0; ax < 3; ++ax) {
    if (!per[ax]) {
      double mn = 0.0, mx = box[ax];
      if (n > 0) {
        mn = mx = xyz[ax];
        for (int64_t a = 0; a < n; ++a) {
          const double v = xyz[3 * a + ax];
          mn = (v < mn) ? v : mn; /* std::min(mn, v) */
          mx = (mx < v) ? v : mx; /* std::max(mx, v) */
        }
      }
      lo[ax] = mn;
      hi[ax] = (mx < mn + bc) ? mn + bc : mx;
    }
  }
  const double o[3] = {lo[0], lo[1], lo[2]};
  const double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  int nc[3];
  for (int ax = 0; ax < 3; ++ax) {
    const int c = (int)floor(ext[ax] / bc);
    nc[ax] = c > 1 ? c : 1;
  }
  const int64_t ncells = (int64_t)nc[0] * nc[1] * nc[2];

  /* bins in ascending atom order (neighbor.cpp:79-81) */
  int32_t* cell = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int64_t* start = (int64_t*)calloc((size_t)ncells + 1, sizeof(int64_t));
  int32_t* binned = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  if (!cell || !start || !binned) return ORC_NOMEM;
  for (int64_t a = 0; a < n; ++a) {
    const int cx = clamp_cell((xyz[3 * a] - o[0]) / ext[0], nc[0]);
    const int cy = clamp_cell((xyz[3 * a + 1] - o[1]) / ext[1], nc[1]);
    const int cz = clamp_cell((xyz[3 * a + 2] - o[2]) / ext[2], nc[2]);
    cell[a] = (int32_t)((cz * nc[1] + cy) * nc[0] + cx);
    start[cell[a] + 1]++;
  }
  for (int64_t c = 0; c < ncells; ++c) start[c + 1] += start[c];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncells);
    memcpy(fill, start, sizeof(int64_t) * (size_t)ncells);
    for (int64_t a = 0; a < n; ++a) binned[fill[cell[a]]++] = (int32_t)a;
    free(fill);
  }

  IVec seg = {0, 0, 0};
  IVec all = {0, 0, 0};
  offsets[0] = 0;
  for (int64_t a = 0; a < n; ++a) {
    const int home = cell[a];
    const int cx = home % nc[0], cy = (home / nc[0]) % nc[1], cz = home / (nc[0] * nc[1]);
    /* deduplicated wrapped 27-stencil (neighbor.cpp:84-103) */
    int32_t st[27];
    int ns = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int wx = cx + dx, wy = cy + dy, wz = cz + dz;
          if (per[0]) wx = (wx + nc[0]) % nc[0];
          if (per[1]) wy = (wy + nc[1]) % nc[1];
          if (per[2]) wz = (wz + nc[2]) % nc[2];
          if (wx < 0 || wx >= nc[0] || wy < 0 || wy >= nc[1] || wz < 0 || wz >= nc[2])
            continue;
          st[ns++] = (int32_t)((wz * nc[1] + wy) * nc[0] + wx);
        }
    qsort(st, (size_t)ns, sizeof(int32_t), cmp_i32);
    int m = 0;
    for (int q = 0; q < ns; ++q)
      if (m == 0 || st[q] != st[m - 1]) st[m++] = st[q];
    seg.n = 0;
    for (int q = 0; q < m; ++q)
      for (int64_t t = start[st[q]]; t < start[st[q] + 1]; ++t) {
        const int32_t b = binned[t];
        if (b == a) continue;
        double d[3];
        delta(xyz, a, b, box, per, d);
        if (dot3(d, d) <= bc_sq)
          if (!ivec_push(&seg, b)) return ORC_NOMEM;
      }
    qsort(seg.v, (size_t)seg.n, sizeof(int32_t), cmp_i32);
    for (int64_t q = 0; q < seg.n; ++q)
      if (!ivec_push(&all, seg.v[q])) return ORC_NOMEM;
    offsets[a + 1] = (int32_t)all.n;
  }
  free(seg.v);
  free(cell);
  free(start);
  free(binned);
  *out_nbrs = all.v;
  *out_total = all.n;
  return ORC_OK;
}

/* O(N^2) scan, the reference test's brute-force oracle
   (tests/test_neighbor.cpp:34-53). */
int orc_brute_neighbor_list(int64_t n, const double* xyz, const double box[3],
                            const uint8_t per[3], double bc, int32_t* offsets,
                            int32_t** out_nbrs, int64_t* out_total) {
  const double bc2 = bc * bc;
  IVec all = {0, 0, 0};
  offsets[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double d[3];
      delta(xyz, i, j, box, per, d);
      if (dot3(d, d) <= bc2)
        if (!ivec_push(&all, (int32_t)j)) return ORC_NOMEM;
    }
    offsets[i + 1] = (int32_t)all.n;
  }
  *out_nbrs = all.v;
  *out_total = all.n;
  return ORC_OK;
}

/* Short list: filter_all_segments (neighbor.cpp:143-180).  Caller sizes
   out_nbrs to the skin list's entry count. */
int64_t orc_filter(int64_t n, const double* xyz, const double box[3], const uint8_t per[3],
                   const int32_t* offsets, const int32_t* nbrs, double r_cut_max,
                   int32_t* out_offsets, int32_t* out_nbrs) {
  const double cut_sq = r_cut_max * r_cut_max;
  int64_t w = 0;
  out_offsets[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int32_t p = offsets[i]; p < offsets[i + 1]; ++p) {
      double d[3];
      delta(xyz, i, nbrs[p], box, per, d);
      if (dot3(d, d) <= cut_sq) out_nbrs[w++] = nbrs[p];
    }
    out_offsets[i + 1] = (int32_t)w;
  }
  return w;
}

/* needs_rebuild, neighbor.cpp:134-141 */
int orc_needs_rebuild(int64_t n, const double* xyz, const double* ref_xyz,
                      const double box[3], const uint8_t per[3], double skin) {
  const double limit_sq = 0.25 * skin * skin;
  for (int64_t a = 0; a < n; ++a) {
    double d[3] = {xyz[3 * a] - ref_xyz[3 * a], xyz[3 * a + 1] - ref_xyz[3 * a + 1],
                   xyz[3 * a + 2] - ref_xyz[3 * a + 2]};
    min_image(d, box, per);
    if (dot3(d, d) > limit_sq) return 1;
  }
  return 0;
}

void orc_free(void* p) { free(p); }
