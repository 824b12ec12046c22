// Host-side builders of the PCG operator inputs for structured box meshes.
//
// These are the product's own C++ (the reference is never linked): the GLL
// basis, box-mesh corners, trilinear geometric factors, the gather-scatter map
// (built in closed form from the node lattice -- no global sort), the
// Dirichlet mask and recursive coordinate bisection.  Arithmetic follows the
// reference expression by expression so every floating-point output is
// bitwise equal to sembox's (checked in tests/test_setup.py against oracle/);
// the integer outputs (gs map, partition) are bit-exact by construction.
// Compiled with -ffp-contract=off.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "lattice.h"
#include "metric.h"
#include "sbx_internal.h"

namespace sbx {

// ---------------------------------------------------------------- threads --
void host_parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
  if (n <= 0) return;
  int nt = static_cast<int>(std::thread::hardware_concurrency());
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  if (n < 4096 || nt == 1) {
    fn(0, n);
    return;
  }
  const int64_t chunks = std::min<int64_t>(n, 8LL * nt);
  std::atomic<int64_t> next{0};
  auto worker = [&] {
    for (;;) {
      const int64_t c = next.fetch_add(1);
      if (c >= chunks) return;
      fn(c * n / chunks, (c + 1) * n / chunks);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
}

// ------------------------------------------------------------------ basis --
// Legendre P_N and P_N' by the three-term recurrence; the endpoint derivative
// from the closed form (basis.cpp:17-35).
static void legendre_pair(int deg, double x, double& p, double& dp) {
  if (deg == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  double pm = 1.0, pc = x;
  for (int k = 1; k < deg; ++k) {
    const double pn = ((2 * k + 1) * x * pc - k * pm) / (k + 1);
    pm = pc;
    pc = pn;
  }
  p = pc;
  if (x == 1.0 || x == -1.0)
    dp = 0.5 * deg * (deg + 1) * (x == 1.0 ? 1.0 : (deg % 2 == 0 ? -1.0 : 1.0));
  else
    dp = deg * (x * pc - pm) / (x * x - 1.0);
}

int gll_basis(int degree, double* nodes, double* weights, double* deriv) {
  if (degree < 1 || degree > kMaxDegree) return SBX_E_CONFIG;
  const int n = degree + 1;
  std::vector<double> x(n, 0.0);
  x.front() = -1.0;
  x.back() = 1.0;
  // interior nodes: roots of P_N' by Newton from Chebyshev-Lobatto guesses
  for (int i = 1; i < degree; ++i) {
    double xi = -std::cos(M_PI * i / degree);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre_pair(degree, xi, p, dp);
      const double step = dp / ((2.0 * xi * dp - degree * (degree + 1) * p) / (1.0 - xi * xi));
      xi -= step;
      if (std::abs(step) <= 1e-15) break;
    }
    x[i] = xi;
  }
  // exact symmetry about the origin
  for (int i = 0; i < n / 2; ++i) {
    const double half = 0.5 * (x[n - 1 - i] - x[i]);
    x[i] = -half;
    x[n - 1 - i] = half;
  }
  if (n % 2) x[n / 2] = 0.0;
  std::vector<double> bary(n, 1.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) bary[j] /= (x[j] - x[k]);
  for (int i = 0; i < n; ++i) {
    if (nodes) nodes[i] = x[i];
    if (weights) {
      double p, dp;
      legendre_pair(degree, x[i], p, dp);
      weights[i] = 2.0 / (degree * (degree + 1) * p * p);
    }
    if (deriv) {
      double off = 0.0;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const double v = (bary[j] / bary[i]) / (x[i] - x[j]);
        deriv[i * n + j] = v;
        off += v;
      }
      deriv[i * n + i] = -off;  // rows sum to zero
    }
  }
  return SBX_OK;
}

// GL pressure basis of the P_N / P_N-2 pair (basis.cpp:114-145): the m = N-1
// roots of L_m by Newton from the Chebyshev-like guesses, symmetrised, their
// weights, and the velocity-to-pressure interpolation l_j(gl_i) in the
// barycentric form of lagrange_eval (basis.cpp:147-162).
int pressure_basis(int degree, double* nodes, double* weights, double* interp) {
  if (degree < 3 || degree > kMaxDegree) return SBX_E_CONFIG;
  const int m = degree - 1, n = degree + 1;
  std::vector<double> x(m, 0.0), w(m, 0.0);
  for (int i = 0; i < m; ++i) {
    double xi = -std::cos(M_PI * (i + 0.75) / (m + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre_pair(m, xi, p, dp);
      const double dx = p / dp;
      xi -= dx;
      if (std::abs(dx) <= 1e-15) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i < m / 2; ++i) {
    const double half = 0.5 * (x[m - 1 - i] - x[i]);
    x[i] = -half;
    x[m - 1 - i] = half;
  }
  if (m % 2) x[m / 2] = 0.0;
  for (int i = 0; i < m; ++i) {
    double p, dp;
    legendre_pair(m, x[i], p, dp);
    w[i] = 2.0 / ((1.0 - x[i] * x[i]) * dp * dp);
  }
  std::vector<double> v(n);
  gll_basis(degree, v.data(), nullptr, nullptr);
  std::vector<double> bary(n, 1.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) bary[j] /= (v[j] - v[k]);
  for (int i = 0; i < m; ++i) {
    double* row = interp ? interp + (size_t)i * n : nullptr;
    if (!row) continue;
    int hit = -1;
    for (int j = 0; j < n; ++j)
      if (x[i] == v[j]) {
        hit = j;
        break;
      }
    if (hit >= 0) {
      for (int j = 0; j < n; ++j) row[j] = j == hit ? 1.0 : 0.0;
      continue;
    }
    double denom = 0.0;
    for (int j = 0; j < n; ++j) denom += bary[j] / (x[i] - v[j]);
    for (int j = 0; j < n; ++j) row[j] = (bary[j] / (x[i] - v[j])) / denom;
  }
  for (int i = 0; i < m; ++i) {
    if (nodes) nodes[i] = x[i];
    if (weights) weights[i] = w[i];
  }
  return SBX_OK;
}

// ------------------------------------------------------------------- mesh --
int box_corners(int ex, int ey, int ez, const double* origin, const double* lengths,
                double* corners) {
  if (ex < 1 || ey < 1 || ez < 1) return SBX_E_CONFIG;
  for (int d = 0; d < 3; ++d)
    if (!(lengths[d] > 0.0)) return SBX_E_CONFIG;
  const double h[3] = {lengths[0] / ex, lengths[1] / ey, lengths[2] / ez};
  const int64_t E = static_cast<int64_t>(ex) * ey * ez;
  host_parallel_for(E, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      const int64_t cell[3] = {e % ex, (e / ex) % ey, e / (static_cast<int64_t>(ex) * ey)};
      double* c = corners + e * 24;
      for (int v = 0; v < 8; ++v)
        for (int d = 0; d < 3; ++d)
          c[v * 3 + d] = origin[d] + h[d] * static_cast<int>(cell[d] + ((v >> d) & 1));
    }
  });
  return SBX_OK;
}

void deform_corners(int64_t elem_count, double a, double* corners) {
  host_parallel_for(elem_count * 8, [&](int64_t lo, int64_t hi) {
    for (int64_t q = lo; q < hi; ++q) {
      double* p = corners + q * 3;
      const double s = std::sin(M_PI * p[0]) * std::sin(M_PI * p[1]) * std::sin(M_PI * p[2]);
      const double d0 = a * s * 1.0, d1 = a * s * 0.5, d2 = a * s * 0.25;
      p[0] += d0;
      p[1] += d1;
      p[2] += d2;
    }
  });
}

// ------------------------------------------------------ geometric factors --
// Trilinear map Jacobian J[p][q] = dx_p/dxi_q accumulated corner by corner,
// its determinant, inverse, and the symmetric metric w*detJ*J^-1 J^-T
// (reference: operators.cpp:19-57, 123-178).

// node_metric's Jacobian is sum_v X_v grad N_v with N_v = prod_q (1 + sg_q xi_q) / 2
// (sg_q = +-1 from corner bit q); expanding the products gives the bilinear
// forms of trilinear_coeffs, S_A = (1/8) sum_v (prod_{q in A} sg_q) X_v.
void trilinear_coeffs(int64_t E, const double* corners, double* tl) {
  host_parallel_for(E, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      const double* cr = corners + e * 24;
      double* o = tl + e * 24;
      for (int q = 0; q < 24; ++q) o[q] = 0.0;
      for (int v = 0; v < 8; ++v) {
        const double s0 = (v & 1) ? 1.0 : -1.0, s1 = (v & 2) ? 1.0 : -1.0,
                     s2 = (v & 4) ? 1.0 : -1.0;
        const double sg[7] = {s0, s1, s2, s0 * s1, s0 * s2, s1 * s2, s0 * s1 * s2};
        for (int a = 0; a < 7; ++a)
          for (int p = 0; p < 3; ++p) o[a * 3 + p] += 0.125 * sg[a] * cr[v * 3 + p];
      }
    }
  });
}

int geometric_factors(int64_t E, int degree, const double* corners, double* const g[6],
                      double* bm, double* jac, int64_t* bad_elem) {
  const int n = degree + 1;
  std::vector<double> x(n), w(n);
  if (gll_basis(degree, x.data(), w.data(), nullptr) != SBX_OK) return SBX_E_CONFIG;
  const int64_t nper = static_cast<int64_t>(n) * n * n;
  std::atomic<int64_t> bad{INT64_MAX};
  host_parallel_for(E, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      int64_t a = e * nper;
      for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i, ++a) {
            Metric m;
            const double wq = w[i] * w[j] * w[k];
            if (!node_metric(corners + e * 24, x[i], x[j], x[k], wq, m)) {
              int64_t cur = bad.load();
              while (e < cur && !bad.compare_exchange_weak(cur, e)) {
              }
              goto next_elem;
            }
            for (int c = 0; c < 6; ++c)
              if (g[c]) g[c][a] = m.g[c];
            if (bm) bm[a] = m.wdet;
            if (jac) jac[a] = m.det;
          }
    next_elem:;
    }
  });
  *bad_elem = bad.load() == INT64_MAX ? -1 : bad.load();
  return *bad_elem >= 0 ? SBX_E_MESH : SBX_OK;
}

// ---------------------------------------------------------- gather-scatter --
// Closed-form construction on the continuous node lattice.  Per direction d,
// lattice coordinate g is owned by one (cell, loc) pair, or by two when it
// sits on an element boundary (plus the periodic wrap).  A node's copies are
// the Cartesian product of those options; groups are enumerated in lattice
// (= gid) order and copies sorted by local index, which reproduces the
// reference's sort on (gid, local index) (gather.cpp:48-70) exactly.
int gather_scatter(int ex, int ey, int ez, const int* periodic, int degree, int64_t* gid,
                   int64_t* offsets, int64_t* group_nodes, int32_t* mult, double* inv_mult,
                   int64_t* global_count) {
  if (degree < 1) return SBX_E_SHAPE;
  if (ex < 1 || ey < 1 || ez < 1) return SBX_E_CONFIG;
  Lattice L;
  L.counts[0] = ex;
  L.counts[1] = ey;
  L.counts[2] = ez;
  L.N = degree;
  const int n = degree + 1;
  for (int d = 0; d < 3; ++d) {
    L.per[d] = periodic[d] != 0;
    const int64_t span = static_cast<int64_t>(L.counts[d]) * degree;
    L.gdim[d] = L.per[d] ? span : span + 1;
  }
  const int64_t G = L.gdim[0] * L.gdim[1] * L.gdim[2];
  *global_count = G;
  // prefix sums of per-axis option counts -> closed-form group offsets
  std::vector<int64_t> pre[3];
  for (int d = 0; d < 3; ++d) {
    pre[d].assign(L.gdim[d] + 1, 0);
    for (int64_t g = 0; g < L.gdim[d]; ++g) pre[d][g + 1] = pre[d][g] + L.opts(d, g).count;
  }
  const int64_t S0 = pre[0][L.gdim[0]], S1 = pre[1][L.gdim[1]];
  const int64_t nn = static_cast<int64_t>(n) * n * n;
  const int64_t ex_ey = static_cast<int64_t>(ex) * ey;
  offsets[G] = S0 * S1 * pre[2][L.gdim[2]];
  host_parallel_for(L.gdim[1] * L.gdim[2], [&](int64_t lo, int64_t hi) {
    for (int64_t row = lo; row < hi; ++row) {
      const int64_t g1 = row % L.gdim[1], g2 = row / L.gdim[1];
      const AxisOpts o1 = L.opts(1, g1), o2 = L.opts(2, g2);
      int64_t off = S0 * S1 * pre[2][g2] + S0 * pre[1][g1] * o2.count;
      for (int64_t g0 = 0; g0 < L.gdim[0]; ++g0) {
        const int64_t id = g0 + L.gdim[0] * (g1 + L.gdim[1] * g2);
        const AxisOpts o0 = L.opts(0, g0);
        int64_t cp[8];
        int m = 0;
        for (int c2 = 0; c2 < o2.count; ++c2)
          for (int c1 = 0; c1 < o1.count; ++c1)
            for (int c0 = 0; c0 < o0.count; ++c0) {
              const int64_t e = o0.cell[c0] + ex * o1.cell[c1] + ex_ey * o2.cell[c2];
              cp[m++] = e * nn + (static_cast<int64_t>(o2.loc[c2]) * n + o1.loc[c1]) * n +
                        o0.loc[c0];
            }
        for (int x = 1; x < m; ++x)  // insertion sort of <= 8 copies
          for (int y = x; y > 0 && cp[y - 1] > cp[y]; --y) std::swap(cp[y - 1], cp[y]);
        offsets[id] = off;
        for (int c = 0; c < m; ++c) {
          group_nodes[off + c] = cp[c];
          if (gid) gid[cp[c]] = id;
          if (mult) mult[cp[c]] = m;
          if (inv_mult) inv_mult[cp[c]] = 1.0 / m;
        }
        off += m;
      }
    }
  });
  return SBX_OK;
}

int dirichlet_mask(int ex, int ey, int ez, const int* periodic, int degree, double* mask) {
  const int n = degree + 1;
  const int counts[3] = {ex, ey, ez};
  const int64_t E = static_cast<int64_t>(ex) * ey * ez;
  const int64_t nn = static_cast<int64_t>(n) * n * n;
  host_parallel_for(E, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      const int64_t cell[3] = {e % ex, (e / ex) % ey, e / (static_cast<int64_t>(ex) * ey)};
      for (int64_t l = 0; l < nn; ++l) {
        const int loc[3] = {static_cast<int>(l % n), static_cast<int>((l / n) % n),
                            static_cast<int>(l / (n * n))};
        double v = 1.0;
        for (int d = 0; d < 3; ++d) {
          if (periodic[d]) continue;
          const int64_t g = cell[d] * degree + loc[d];
          if (g == 0 || g == static_cast<int64_t>(counts[d]) * degree) v = 0.0;
        }
        mask[e * nn + l] = v;
      }
    }
  });
  return SBX_OK;
}

// -------------------------------------------------------------------- RCB --
// Recursive coordinate bisection over element centroids (mesh.cpp:168-226):
// cut the longest centroid-bbox axis (ties x < y < z), order by (centroid,
// element id), split proportionally to the rank counts of the two halves.
namespace {
void rcb_split(const std::vector<std::array<double, 3>>& cen, std::vector<int64_t>& ids,
               int ranks, int first, int32_t* rank_of) {
  if (ranks == 1) {
    for (int64_t e : ids) rank_of[e] = first;
    return;
  }
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t e : ids)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], cen[e][d]);
      hi[d] = std::max(hi[d], cen[e][d]);
    }
  int ax = 0;
  for (int d = 1; d < 3; ++d)
    if (hi[d] - lo[d] > hi[ax] - lo[ax] + 1e-12 * (hi[ax] - lo[ax] + 1.0)) ax = d;
  std::sort(ids.begin(), ids.end(), [&](int64_t a, int64_t b) {
    if (cen[a][ax] != cen[b][ax]) return cen[a][ax] < cen[b][ax];
    return a < b;
  });
  const int r1 = (ranks + 1) / 2, r2 = ranks - r1;
  const int64_t cnt = static_cast<int64_t>(ids.size());
  const int64_t n1 = std::clamp<int64_t>((cnt * r1 + ranks / 2) / ranks, r1, cnt - r2);
  std::vector<int64_t> left(ids.begin(), ids.begin() + n1), right(ids.begin() + n1, ids.end());
  ids.clear();
  ids.shrink_to_fit();
  rcb_split(cen, left, r1, first, rank_of);
  rcb_split(cen, right, r2, first + r1, rank_of);
}
}  // namespace

int partition_rcb(int64_t E, const double* corners, int ranks, int32_t* rank_of) {
  if (ranks < 1 || ranks > E) return SBX_E_CONFIG;
  std::vector<std::array<double, 3>> cen(E);
  host_parallel_for(E, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      std::array<double, 3> c{0, 0, 0};
      for (int v = 0; v < 8; ++v)
        for (int d = 0; d < 3; ++d) c[d] += corners[e * 24 + v * 3 + d] / 8.0;
      cen[e] = c;
    }
  });
  std::vector<int64_t> ids(E);
  std::iota(ids.begin(), ids.end(), 0);
  rcb_split(cen, ids, ranks, 0, rank_of);
  return SBX_OK;
}

}  // namespace sbx
