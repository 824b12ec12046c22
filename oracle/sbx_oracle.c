/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Nothing in the product
 * (paper_2109_03592_b200/) links, imports or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, and only as
 * the checker / the reported CPU baseline.
 *
 * Plain-C, single-threaded restatement of the reference's ("sembox",
 * /root/reference/proj) hot-path algorithms: GLL basis, box mesh, geometric
 * factors, gather-scatter map, Dirichlet mask, axhelm, its diagonal, gs_sum,
 * the deterministic weighted dot and Jacobi-PCG, RCB partitioning.  Every
 * floating-point expression keeps the reference's evaluation order (C
 * left-to-right, no contraction: build with -ffp-contract=off) so results are
 * bitwise identical to the reference built for x86-64 (which has no FMA in
 * its baseline ISA).  That claim is pinned by tests/test_oracle.py against
 * oracle/_ref (the reference compiled unmodified) and tests/golden/.
 *
 * Each function cites the reference file:line it restates.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ RNG --
 * std::mt19937_64 + std::uniform_real_distribution<double>(a,b) as
 * implemented by libstdc++ (generate_canonical<double,53> takes one 64-bit
 * draw: u = double(x) / 2^64, clamped below 1; value = u*(b-a)+a).  Used by
 * the reference's tests for random fields (test_schwarz.cpp:30-38,
 * bench.cpp:86-90). */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_mt64;

void or_mt64_seed(or_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

uint64_t or_mt64_next(or_mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = s->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = v;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

void or_fill_uniform(uint64_t seed, int64_t n, double a, double b, double* out) {
  or_mt64 s;
  or_mt64_seed(&s, seed);
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)or_mt64_next(&s) * 1.0;
    u = u / 18446744073709551616.0;
    if (u >= 1.0) u = nextafter(1.0, 0.0);
    out[i] = u * (b - a) + a;
  }
}

/* ---------------------------------------------------------------- basis --
 * basis.cpp:17-35 legendre, :38-47 symmetrize, :49-56 barycentric weights,
 * :60-95 build_gll_basis, :97-112 build_deriv_matrix. */
static void legendre(int n, double x, double* p, double* dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) {
    *p = 1.0;
    *dp = 0.0;
    return;
  }
  for (int k = 1; k < n; ++k) {
    const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1;
    p1 = p2;
  }
  *p = p1;
  if (x == 1.0 || x == -1.0)
    *dp = 0.5 * n * (n + 1) * (x == 1.0 ? 1.0 : (n % 2 == 0 ? -1.0 : 1.0));
  else
    *dp = n * (x * p1 - p0) / (x * x - 1.0);
}

/* returns 0, or 2 (ConfigError) for a degree outside [1,32] */
int or_gll_basis(int degree, double* nodes, double* weights, double* deriv) {
  if (degree < 1 || degree > 32) return 2;
  const int n = degree + 1;
  for (int i = 0; i < n; ++i) nodes[i] = 0.0;
  nodes[0] = -1.0;
  nodes[n - 1] = 1.0;
  for (int i = 1; i < degree; ++i) {
    double x = -cos(M_PI * i / degree);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre(degree, x, &p, &dp);
      const double d2p = (2.0 * x * dp - degree * (degree + 1) * p) / (1.0 - x * x);
      const double dx = dp / d2p;
      x -= dx;
      if (fabs(dx) <= 1e-15) break;
    }
    nodes[i] = x;
  }
  for (int i = 0; i < n / 2; ++i) { /* symmetrize */
    const double m = 0.5 * (nodes[n - 1 - i] - nodes[i]);
    nodes[i] = -m;
    nodes[n - 1 - i] = m;
  }
  if (n % 2 == 1) nodes[n / 2] = 0.0;
  for (int i = 0; i < n; ++i) {
    double p, dp;
    legendre(degree, nodes[i], &p, &dp);
    weights[i] = 2.0 / (degree * (degree + 1) * p * p);
  }
  double bw[64];
  for (int j = 0; j < n; ++j) {
    bw[j] = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j) bw[j] /= (nodes[j] - nodes[k]);
  }
  for (int i = 0; i < n; ++i) {
    double rowsum = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const double v = (bw[j] / bw[i]) / (nodes[i] - nodes[j]);
      deriv[i * n + j] = v;
      rowsum += v;
    }
    deriv[i * n + i] = -rowsum;
  }
  return 0;
}

/* ----------------------------------------------------------------- mesh --
 * mesh.cpp:21-52: element e = ix + ex*(jy + ey*kz); corner c = i+2j+4k,
 * coordinate origin[d] + h[d]*(cell[d]+bit), h[d] = lengths[d]/counts[d]. */
int or_box_corners(int ex, int ey, int ez, const double* origin, const double* lengths,
                   double* corners) {
  if (ex < 1 || ey < 1 || ez < 1) return 2;
  for (int d = 0; d < 3; ++d)
    if (!(lengths[d] > 0.0)) return 2;
  const double h[3] = {lengths[0] / ex, lengths[1] / ey, lengths[2] / ez};
  for (int kz = 0; kz < ez; ++kz)
    for (int jy = 0; jy < ey; ++jy)
      for (int ix = 0; ix < ex; ++ix) {
        const int64_t e = ix + (int64_t)ex * (jy + (int64_t)ey * kz);
        const int cell[3] = {ix, jy, kz};
        for (int c = 0; c < 8; ++c)
          for (int d = 0; d < 3; ++d) {
            const int bit = (c >> d) & 1;
            corners[(e * 8 + c) * 3 + d] = origin[d] + h[d] * (cell[d] + bit);
          }
      }
  return 0;
}

/* Conforming "deformed box" perturbation used by the benchmark configs
 * (SURVEY.md section 8(c) probe recipe): p += a*s*(1, 0.5, 0.25) with
 * s = sin(pi x) sin(pi y) sin(pi z) of the undeformed corner.  Not a
 * reference function -- a test-input generator shared by both sides. */
void or_deform_corners(int64_t elem_count, double a, double* corners) {
  for (int64_t q = 0; q < elem_count * 8; ++q) {
    double* p = corners + q * 3;
    const double s = sin(M_PI * p[0]) * sin(M_PI * p[1]) * sin(M_PI * p[2]);
    const double dx = a * s * 1.0, dy = a * s * 0.5, dz = a * s * 0.25;
    p[0] += dx;
    p[1] += dy;
    p[2] += dz;
  }
}

/* oracle.cpp:67-76 trilinear_point */
void or_trilinear_point(const double* corners, int64_t elem, double r, double s, double t,
                        double* x) {
  x[0] = x[1] = x[2] = 0.0;
  for (int c = 0; c < 8; ++c) {
    const int b[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
    const double sr = b[0] ? 0.5 * (1.0 + r) : 0.5 * (1.0 - r);
    const double ss = b[1] ? 0.5 * (1.0 + s) : 0.5 * (1.0 - s);
    const double st = b[2] ? 0.5 * (1.0 + t) : 0.5 * (1.0 - t);
    const double w = sr * ss * st;
    for (int p = 0; p < 3; ++p) x[p] += w * corners[(elem * 8 + c) * 3 + p];
  }
}

/* ------------------------------------------------------ geometric factors --
 * operators.cpp:19-37 TrilinearMap::jacobian, :39-42 det3, :45-56 inv3,
 * :123-178 build_geometric_factors.  Returns -1, or the first bad element
 * (MeshError: nonpositive Jacobian). */
static void tri_jacobian(const double* cr, double r, double s, double t, double* jac) {
  const double phi[3][2] = {{0.5 * (1 - r), 0.5 * (1 + r)},
                            {0.5 * (1 - s), 0.5 * (1 + s)},
                            {0.5 * (1 - t), 0.5 * (1 + t)}};
  for (int q = 0; q < 9; ++q) jac[q] = 0.0;
  for (int c = 0; c < 8; ++c) {
    const int b[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
    const double dphi[3] = {b[0] ? 0.5 : -0.5, b[1] ? 0.5 : -0.5, b[2] ? 0.5 : -0.5};
    for (int p = 0; p < 3; ++p) {
      const double* x = cr + c * 3;
      double grad[3];
      grad[0] = dphi[0] * phi[1][b[1]] * phi[2][b[2]];
      grad[1] = phi[0][b[0]] * dphi[1] * phi[2][b[2]];
      grad[2] = phi[0][b[0]] * phi[1][b[1]] * dphi[2];
      for (int q = 0; q < 3; ++q) jac[p * 3 + q] += x[p] * grad[q];
    }
  }
}

int64_t or_geometric_factors(int64_t elem_count, int n, const double* nodes,
                             const double* weights, const double* corners, double* g1,
                             double* g2, double* g3, double* g4, double* g5, double* g6,
                             double* bm, double* jacd) {
  for (int64_t e = 0; e < elem_count; ++e) {
    int64_t a = e * n * n * n;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i, ++a) {
          double jm[9], inv[9];
          tri_jacobian(corners + e * 24, nodes[i], nodes[j], nodes[k], jm);
          const double det = jm[0] * (jm[4] * jm[8] - jm[5] * jm[7]) -
                             jm[1] * (jm[3] * jm[8] - jm[5] * jm[6]) +
                             jm[2] * (jm[3] * jm[7] - jm[4] * jm[6]);
          if (!(det > 0.0)) return e;
          const double id = 1.0 / det;
          inv[0] = (jm[4] * jm[8] - jm[5] * jm[7]) * id;
          inv[1] = (jm[2] * jm[7] - jm[1] * jm[8]) * id;
          inv[2] = (jm[1] * jm[5] - jm[2] * jm[4]) * id;
          inv[3] = (jm[5] * jm[6] - jm[3] * jm[8]) * id;
          inv[4] = (jm[0] * jm[8] - jm[2] * jm[6]) * id;
          inv[5] = (jm[2] * jm[3] - jm[0] * jm[5]) * id;
          inv[6] = (jm[3] * jm[7] - jm[4] * jm[6]) * id;
          inv[7] = (jm[1] * jm[6] - jm[0] * jm[7]) * id;
          inv[8] = (jm[0] * jm[4] - jm[1] * jm[3]) * id;
          const double w = weights[i] * weights[j] * weights[k];
          const double wd = w * det;
#define GDOT(P, Q)                                                               \
  (wd * (inv[(P)*3 + 0] * inv[(Q)*3 + 0] + inv[(P)*3 + 1] * inv[(Q)*3 + 1] + \
         inv[(P)*3 + 2] * inv[(Q)*3 + 2]))
          g1[a] = GDOT(0, 0);
          g2[a] = GDOT(1, 1);
          g3[a] = GDOT(2, 2);
          g4[a] = GDOT(0, 1);
          g5[a] = GDOT(0, 2);
          g6[a] = GDOT(1, 2);
#undef GDOT
          bm[a] = wd;
          if (jacd) jacd[a] = det;
        }
  }
  return -1;
}

/* --------------------------------------------------------- gather-scatter --
 * gather.cpp:10-83.  gid = g0 + gdim0*(g1 + gdim1*g2) with g_d = cell_d*N +
 * loc_d (mod gdim_d if periodic); compressed ids/groups in ascending raw gid,
 * copies ascending by local index (a stable counting sort by raw gid is the
 * same permutation as the reference's std::sort on (gid, index)).
 * Outputs: gid[nodes] (compressed), offsets[G+1], group_nodes[nodes],
 * mult[nodes], inv_mult[nodes]; returns G, or -2 for a bad degree. */
int64_t or_gather_scatter(int ex, int ey, int ez, const int* periodic, int degree,
                          int64_t* gid, int64_t* offsets, int64_t* group_nodes,
                          int32_t* mult, double* inv_mult) {
  if (degree < 1) return -2;
  const int n = degree + 1;
  const int counts[3] = {ex, ey, ez};
  int64_t gdim[3];
  for (int d = 0; d < 3; ++d) {
    const int64_t span = (int64_t)counts[d] * degree;
    gdim[d] = periodic[d] ? span : span + 1;
  }
  const int64_t E = (int64_t)ex * ey * ez;
  const int64_t nodes = E * n * n * n;
  const int64_t raw_count = gdim[0] * gdim[1] * gdim[2];
  for (int64_t e = 0; e < E; ++e) {
    const int cell[3] = {(int)(e % ex), (int)((e / ex) % ey), (int)(e / ((int64_t)ex * ey))};
    int64_t a = e * n * n * n;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i, ++a) {
          const int loc[3] = {i, j, k};
          int64_t g[3];
          for (int d = 0; d < 3; ++d) {
            g[d] = (int64_t)cell[d] * degree + loc[d];
            if (periodic[d]) g[d] %= gdim[d];
          }
          gid[a] = g[0] + gdim[0] * (g[1] + gdim[1] * g[2]);
        }
  }
  int64_t* cnt = (int64_t*)calloc((size_t)raw_count + 1, sizeof(int64_t));
  for (int64_t a = 0; a < nodes; ++a) cnt[gid[a] + 1]++;
  for (int64_t r = 0; r < raw_count; ++r) cnt[r + 1] += cnt[r];
  /* cnt[r] = first slot of raw id r */
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)raw_count);
  memcpy(fill, cnt, sizeof(int64_t) * (size_t)raw_count);
  for (int64_t a = 0; a < nodes; ++a) group_nodes[fill[gid[a]]++] = a;
  free(fill);
  int64_t ng = 0;
  offsets[0] = 0;
  for (int64_t r = 0; r < raw_count; ++r) {
    if (cnt[r + 1] == cnt[r]) continue;
    for (int64_t c = cnt[r]; c < cnt[r + 1]; ++c) gid[group_nodes[c]] = ng;
    offsets[++ng] = cnt[r + 1];
  }
  free(cnt);
  for (int64_t g = 0; g < ng; ++g) {
    const int32_t m = (int32_t)(offsets[g + 1] - offsets[g]);
    for (int64_t c = offsets[g]; c < offsets[g + 1]; ++c) {
      mult[group_nodes[c]] = m;
      inv_mult[group_nodes[c]] = 1.0 / m;
    }
  }
  return ng;
}

/* operators.cpp:433-455 build_dirichlet_mask */
void or_dirichlet_mask(int ex, int ey, int ez, const int* periodic, int degree, double* mask) {
  const int n = degree + 1;
  const int counts[3] = {ex, ey, ez};
  const int64_t E = (int64_t)ex * ey * ez;
  for (int64_t e = 0; e < E; ++e) {
    const int cell[3] = {(int)(e % ex), (int)((e / ex) % ey), (int)(e / ((int64_t)ex * ey))};
    int64_t a = e * n * n * n;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i, ++a) {
          const int loc[3] = {i, j, k};
          double v = 1.0;
          for (int d = 0; d < 3; ++d) {
            if (periodic[d]) continue;
            const int64_t g = (int64_t)cell[d] * degree + loc[d];
            if (g == 0 || g == (int64_t)counts[d] * degree) v = 0.0;
          }
          mask[a] = v;
        }
  }
}

/* -------------------------------------------------------------- operators --
 * operators.cpp:215-263 axhelm (scalar h1/h2; flip = debug::axhelm_sign_flip). */
void or_axhelm(int64_t elem_count, int n, const double* d, const double* g1,
               const double* g2, const double* g3, const double* g4, const double* g5,
               const double* g6, const double* bm, double h1, double h2, int flip,
               const double* u, double* out) {
  const double tsign = flip ? -1.0 : 1.0;
  const int nn = n * n * n;
  double* wr = (double*)malloc(sizeof(double) * nn * 3);
  double* ws = wr + nn;
  double* wt = ws + nn;
  for (int64_t e = 0; e < elem_count; ++e) {
    const int64_t base = e * nn;
    const double* ue = u + base;
    double* oe = out + base;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          double rtmp = 0.0, stmp = 0.0, ttmp = 0.0;
          for (int l = 0; l < n; ++l) {
            rtmp += d[i * n + l] * ue[(k * n + j) * n + l];
            stmp += d[j * n + l] * ue[(k * n + l) * n + i];
            ttmp += d[k * n + l] * ue[(l * n + j) * n + i];
          }
          const int64_t a = base + (k * n + j) * n + i;
          const int la = (k * n + j) * n + i;
          wr[la] = (g1[a] * rtmp + g4[a] * stmp + g5[a] * ttmp) * h1;
          ws[la] = (g2[a] * stmp + g4[a] * rtmp + g6[a] * ttmp) * h1;
          wt[la] = (g3[a] * ttmp + g5[a] * rtmp + g6[a] * stmp) * h1;
        }
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          double acc = 0.0;
          for (int l = 0; l < n; ++l)
            acc += d[l * n + i] * wr[(k * n + j) * n + l] + d[l * n + j] * ws[(k * n + l) * n + i] +
                   tsign * d[l * n + k] * wt[(l * n + j) * n + i];
          const int64_t a = base + (k * n + j) * n + i;
          oe[(k * n + j) * n + i] = acc + h2 * bm[a] * ue[(k * n + j) * n + i];
        }
  }
  free(wr);
}

/* operators.cpp:272-298 axhelm_diagonal */
void or_axhelm_diagonal(int64_t elem_count, int n, const double* d, const double* g1,
                        const double* g2, const double* g3, const double* g4,
                        const double* g5, const double* g6, const double* bm, double h1,
                        double h2, double* diag) {
  for (int64_t e = 0; e < elem_count; ++e) {
    const int64_t base = e * n * n * n;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const int64_t a = base + (k * n + j) * n + i;
          double s = 0.0;
          for (int l = 0; l < n; ++l) {
            s += d[l * n + i] * d[l * n + i] * g1[base + (k * n + j) * n + l];
            s += d[l * n + j] * d[l * n + j] * g2[base + (k * n + l) * n + i];
            s += d[l * n + k] * d[l * n + k] * g3[base + (l * n + j) * n + i];
          }
          s += 2.0 * d[i * n + i] * d[j * n + j] * g4[a];
          s += 2.0 * d[i * n + i] * d[k * n + k] * g5[a];
          s += 2.0 * d[j * n + j] * d[k * n + k] * g6[a];
          diag[a] = h1 * s + h2 * bm[a];
        }
  }
}

/* gather.cpp:85-98 gs_sum_inplace (singleton groups skipped) */
void or_gs_sum(int64_t ngroups, const int64_t* offsets, const int64_t* group_nodes,
               double* field) {
  for (int64_t g = 0; g < ngroups; ++g) {
    const int64_t lo = offsets[g], hi = offsets[g + 1];
    if (hi - lo == 1) continue;
    double s = 0.0;
    for (int64_t c = lo; c < hi; ++c) s += field[group_nodes[c]];
    for (int64_t c = lo; c < hi; ++c) field[group_nodes[c]] = s;
  }
}

/* field.cpp:13-22 deterministic_reduce + :69-81 field_dot_weighted
 * (w == NULL gives field_dot, :59-67) */
double or_dot_weighted(int64_t elem_count, int nper, const double* a, const double* b,
                       const double* w) {
  double s = 0.0;
  for (int64_t e = 0; e < elem_count; ++e) {
    const int64_t base = e * nper;
    double p = 0.0;
    if (w)
      for (int i = 0; i < nper; ++i) p += a[base + i] * b[base + i] * w[base + i];
    else
      for (int i = 0; i < nper; ++i) p += a[base + i] * b[base + i];
    s += p;
  }
  return s;
}

/* ------------------------------------------------------------------- PCG --
 * krylov.cpp:7-91 pcg, driving HelmholtzOperator::apply (operators.cpp:
 * 530-534 = axhelm -> gs_sum -> mask), field_dot_weighted and the Jacobi
 * lambda z = r/diag (stepper.cpp:175-186).  diag = assembled diagonal
 * (operators.cpp:536-540), precond 0 = none (z = r copy), 1 = Jacobi.
 * info: [iterations, converged, error_iteration]; res: [rel, rel_precond];
 * history[hist_cap].  Returns 0, 5 breakdown, 6 NaN/Inf. */
typedef struct {
  int64_t E;
  int n;
  const double *d, *g1, *g2, *g3, *g4, *g5, *g6, *bm, *mask, *inv_mult, *diag;
  int64_t ngroups;
  const int64_t *offsets, *group_nodes;
  double h1, h2;
} or_problem;

static void apply_a(const or_problem* P, const double* x, double* out) {
  or_axhelm(P->E, P->n, P->d, P->g1, P->g2, P->g3, P->g4, P->g5, P->g6, P->bm, P->h1, P->h2,
            0, x, out);
  or_gs_sum(P->ngroups, P->offsets, P->group_nodes, out);
  const int64_t N = P->E * P->n * P->n * P->n;
  if (P->mask)
    for (int64_t a = 0; a < N; ++a) out[a] *= P->mask[a];
}

static void precond(const or_problem* P, int kind, const double* r, double* z, int64_t N) {
  if (kind == 1)
    for (int64_t a = 0; a < N; ++a) z[a] = r[a] / P->diag[a];
  else
    memcpy(z, r, sizeof(double) * (size_t)N);
}

int or_pcg(int64_t E, int n, const double* d, const double* g1, const double* g2,
           const double* g3, const double* g4, const double* g5, const double* g6,
           const double* bm, const double* mask, const double* inv_mult,
           const double* diag, int64_t ngroups, const int64_t* offsets,
           const int64_t* group_nodes, double h1, double h2, int pc_kind, const double* b,
           double* x, double tol, int max_iterations, int64_t* info, double* res,
           double* history, int64_t hist_cap, int64_t* hist_len) {
  or_problem P = {E, n, d, g1, g2, g3, g4, g5, g6, bm, mask, inv_mult, diag,
                  ngroups, offsets, group_nodes, h1, h2};
  const int nper = n * n * n;
  const int64_t N = E * nper;
  info[0] = 0;
  info[1] = 0;
  info[2] = -1;
  res[0] = res[1] = 0.0;
  *hist_len = 0;
#define PUSH(v)                                 \
  do {                                          \
    if (*hist_len < hist_cap) history[*hist_len] = (v); \
    ++*hist_len;                                \
  } while (0)
  const double bb = or_dot_weighted(E, nper, b, b, inv_mult);
  if (bb == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)N);
    info[1] = 1;
    return 0;
  }
  const double bnorm = sqrt(bb);
  double* r = (double*)malloc(sizeof(double) * (size_t)N * 4);
  double *z = r + N, *q = z + N, *p = q + N;
  memcpy(r, b, sizeof(double) * (size_t)N);
  int zero_guess = 1;
  for (int64_t a = 0; a < N; ++a)
    if (x[a] != 0.0) {
      zero_guess = 0;
      break;
    }
  if (!zero_guess) {
    apply_a(&P, x, q);
    for (int64_t a = 0; a < N; ++a) r[a] += -1.0 * q[a];
  }
  precond(&P, pc_kind, b, z, N);
  const double bmb = or_dot_weighted(E, nper, b, z, inv_mult);
  precond(&P, pc_kind, r, z, N);
  double rz = or_dot_weighted(E, nper, r, z, inv_mult);
  double rnorm = sqrt(or_dot_weighted(E, nper, r, r, inv_mult));
  PUSH(rnorm / bnorm);
  memcpy(p, z, sizeof(double) * (size_t)N);
  int status = 0;
  int it;
  for (it = 0; it < max_iterations; ++it) {
    res[0] = rnorm / bnorm;
    res[1] = bmb > 0.0 ? sqrt((rz > 0.0 ? rz : 0.0) / bmb) : 0.0;
    if (res[0] <= tol && res[1] <= tol) {
      info[1] = 1;
      goto done;
    }
    apply_a(&P, p, q);
    const double pq = or_dot_weighted(E, nper, p, q, inv_mult);
    if (!isfinite(pq) || pq <= 0.0) {
      info[2] = it;
      status = 5;
      goto done;
    }
    const double alpha = rz / pq;
    for (int64_t a = 0; a < N; ++a) x[a] += alpha * p[a];
    const double malpha = -alpha;
    for (int64_t a = 0; a < N; ++a) r[a] += malpha * q[a];
    precond(&P, pc_kind, r, z, N);
    const double rz_new = or_dot_weighted(E, nper, r, z, inv_mult);
    rnorm = sqrt(or_dot_weighted(E, nper, r, r, inv_mult));
    if (!isfinite(rnorm) || !isfinite(rz_new)) {
      info[2] = it;
      status = 6;
      goto done;
    }
    PUSH(rnorm / bnorm);
    ++info[0];
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int64_t a = 0; a < N; ++a) p[a] *= beta;
    for (int64_t a = 0; a < N; ++a) p[a] += 1.0 * z[a];
  }
  res[0] = rnorm / bnorm;
  res[1] = bmb > 0.0 ? sqrt((rz > 0.0 ? rz : 0.0) / bmb) : 0.0;
  info[1] = (res[0] <= tol && res[1] <= tol) ? 1 : 0;
done:
  free(r);
  return status;
#undef PUSH
}

/* ------------------------------------------------------------------ RCB --
 * mesh.cpp:14-19 centroid, :168-208 rcb_recurse, :212-226 partition_rcb.
 * Returns 0 or 2 (ConfigError). */
typedef struct {
  double key;
  int elem;
} rcb_item;

static int rcb_cmp(const void* pa, const void* pb) {
  const rcb_item* a = (const rcb_item*)pa;
  const rcb_item* b = (const rcb_item*)pb;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return (a->elem > b->elem) - (a->elem < b->elem);
}

static void centroid(const double* corners, int e, double* c) {
  c[0] = c[1] = c[2] = 0.0;
  for (int q = 0; q < 8; ++q)
    for (int d = 0; d < 3; ++d) c[d] += corners[((int64_t)e * 8 + q) * 3 + d] / 8.0;
}

static void rcb_recurse(const double* corners, int* elems, int64_t count, int ranks,
                        int first_rank, int32_t* rank_of) {
  if (ranks == 1) {
    for (int64_t i = 0; i < count; ++i) rank_of[elems[i]] = first_rank;
    return;
  }
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  double* cents = (double*)malloc(sizeof(double) * 3 * (size_t)count);
  for (int64_t i = 0; i < count; ++i) {
    centroid(corners, elems[i], cents + 3 * i);
    for (int d = 0; d < 3; ++d) {
      if (cents[3 * i + d] < lo[d]) lo[d] = cents[3 * i + d];
      if (cents[3 * i + d] > hi[d]) hi[d] = cents[3 * i + d];
    }
  }
  int axis = 0;
  for (int d = 1; d < 3; ++d)
    if (hi[d] - lo[d] > hi[axis] - lo[axis] + 1e-12 * (hi[axis] - lo[axis] + 1.0)) axis = d;
  rcb_item* items = (rcb_item*)malloc(sizeof(rcb_item) * (size_t)count);
  for (int64_t i = 0; i < count; ++i) {
    items[i].key = cents[3 * i + axis];
    items[i].elem = elems[i];
  }
  free(cents);
  qsort(items, (size_t)count, sizeof(rcb_item), rcb_cmp);
  const int r1 = (ranks + 1) / 2, r2 = ranks - r1;
  int64_t n1 = (count * r1 + ranks / 2) / ranks;
  if (n1 < r1) n1 = r1;
  if (n1 > count - r2) n1 = count - r2;
  int* sorted = (int*)malloc(sizeof(int) * (size_t)count);
  for (int64_t i = 0; i < count; ++i) sorted[i] = items[i].elem;
  free(items);
  rcb_recurse(corners, sorted, n1, r1, first_rank, rank_of);
  rcb_recurse(corners, sorted + n1, count - n1, r2, first_rank + r1, rank_of);
  free(sorted);
}

int or_partition_rcb(int64_t elem_count, const double* corners, int ranks, int32_t* rank_of) {
  if (ranks < 1 || ranks > elem_count) return 2;
  int* all = (int*)malloc(sizeof(int) * (size_t)elem_count);
  for (int64_t e = 0; e < elem_count; ++e) all[e] = (int)e;
  rcb_recurse(corners, all, elem_count, ranks, 0, rank_of);
  free(all);
  return 0;
}

/* ---------------------------------------------------- dense element oracle --
 * oracle.cpp:78-125 dense_helmholtz_element (O(n^6) quadrature loop, shares
 * no code with axhelm).  out: nn*nn row-major. */
int or_dense_helmholtz_element(const double* corners, int64_t elem, int n,
                               const double* nodes, const double* weights,
                               const double* deriv, double h1, double h2, double* a) {
  const int nn = n * n * n;
  memset(a, 0, sizeof(double) * (size_t)nn * nn);
  double* gphys = (double*)malloc(sizeof(double) * 3 * (size_t)nn);
  for (int kq = 0; kq < n; ++kq)
    for (int jq = 0; jq < n; ++jq)
      for (int iq = 0; iq < n; ++iq) {
        double jm[9], inv[9];
        /* oracle.cpp:53-65 trilinear_jacobian */
        for (int q = 0; q < 9; ++q) jm[q] = 0.0;
        const double r = nodes[iq], s = nodes[jq], t = nodes[kq];
        for (int c = 0; c < 8; ++c) {
          const int b[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
          const double sh[3] = {b[0] ? 0.5 * (1.0 + r) : 0.5 * (1.0 - r),
                                b[1] ? 0.5 * (1.0 + s) : 0.5 * (1.0 - s),
                                b[2] ? 0.5 * (1.0 + t) : 0.5 * (1.0 - t)};
          const double ds[3] = {b[0] ? 0.5 : -0.5, b[1] ? 0.5 : -0.5, b[2] ? 0.5 : -0.5};
          const double grad[3] = {ds[0] * sh[1] * sh[2], sh[0] * ds[1] * sh[2],
                                  sh[0] * sh[1] * ds[2]};
          for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) jm[p * 3 + q] += corners[(elem * 8 + c) * 3 + p] * grad[q];
        }
        const double det = jm[0] * (jm[4] * jm[8] - jm[5] * jm[7]) -
                           jm[1] * (jm[3] * jm[8] - jm[5] * jm[6]) +
                           jm[2] * (jm[3] * jm[7] - jm[4] * jm[6]);
        if (!(det > 0.0)) {
          free(gphys);
          return 4;
        }
        const double id = 1.0 / det;
        inv[0] = (jm[4] * jm[8] - jm[5] * jm[7]) * id;
        inv[1] = (jm[2] * jm[7] - jm[1] * jm[8]) * id;
        inv[2] = (jm[1] * jm[5] - jm[2] * jm[4]) * id;
        inv[3] = (jm[5] * jm[6] - jm[3] * jm[8]) * id;
        inv[4] = (jm[0] * jm[8] - jm[2] * jm[6]) * id;
        inv[5] = (jm[2] * jm[3] - jm[0] * jm[5]) * id;
        inv[6] = (jm[3] * jm[7] - jm[4] * jm[6]) * id;
        inv[7] = (jm[1] * jm[6] - jm[0] * jm[7]) * id;
        inv[8] = (jm[0] * jm[4] - jm[1] * jm[3]) * id;
        const double w = weights[iq] * weights[jq] * weights[kq] * det;
        for (int ka = 0; ka < n; ++ka)
          for (int ja = 0; ja < n; ++ja)
            for (int ia = 0; ia < n; ++ia) {
              const int aa = (ka * n + ja) * n + ia;
              const double gr = (ja == jq && ka == kq) ? deriv[iq * n + ia] : 0.0;
              const double gs = (ia == iq && ka == kq) ? deriv[jq * n + ja] : 0.0;
              const double gt = (ia == iq && ja == jq) ? deriv[kq * n + ka] : 0.0;
              for (int dd = 0; dd < 3; ++dd)
                gphys[3 * aa + dd] = inv[0 * 3 + dd] * gr + inv[1 * 3 + dd] * gs + inv[2 * 3 + dd] * gt;
            }
        for (int ra = 0; ra < nn; ++ra) {
          const double* ga = gphys + 3 * ra;
          if (ga[0] == 0.0 && ga[1] == 0.0 && ga[2] == 0.0) continue;
          for (int rb = 0; rb < nn; ++rb) {
            const double* gb = gphys + 3 * rb;
            const double dot = ga[0] * gb[0] + ga[1] * gb[1] + ga[2] * gb[2];
            if (dot != 0.0) a[(size_t)ra * nn + rb] += h1 * w * dot;
          }
        }
        const int q = (kq * n + jq) * n + iq;
        a[(size_t)q * nn + q] += h2 * w;
      }
  free(gphys);
  return 0;
}
