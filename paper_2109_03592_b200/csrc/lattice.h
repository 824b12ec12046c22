// Continuous node lattice of a structured box (shared by the gather-scatter
// builders).  Per direction d, lattice coordinate g is owned by one (cell,
// loc) pair, or by two when it sits on an element boundary (plus the periodic
// wrap): the reference's gid = g0 + gdim0*(g1 + gdim1*g2) with
// g_d = cell_d*N + loc_d (mod gdim_d when periodic) (gather.cpp:15-46), read
// backwards.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define SBX_HD __host__ __device__
#else
#define SBX_HD
#endif

namespace sbx {

struct AxisOpts {
  int count = 1;
  int64_t cell[2];
  int loc[2];
};

struct Lattice {
  int counts[3];
  int N;
  bool per[3];
  int64_t gdim[3];

  SBX_HD void init(int ex, int ey, int ez, const int* periodic, int degree) {
    counts[0] = ex;
    counts[1] = ey;
    counts[2] = ez;
    N = degree;
    for (int d = 0; d < 3; ++d) {
      per[d] = periodic[d] != 0;
      const int64_t span = static_cast<int64_t>(counts[d]) * degree;
      gdim[d] = per[d] ? span : span + 1;
    }
  }

  SBX_HD AxisOpts opts(int d, int64_t g) const {
    AxisOpts o;
    const int64_t span = static_cast<int64_t>(counts[d]) * N;
    if (g % N != 0) {
      o.count = 1;
      o.cell[0] = g / N;
      o.loc[0] = static_cast<int>(g % N);
      return o;
    }
    o.count = 0;
    if (per[d]) {
      // g == c*N: loc 0 of cell c and loc N of cell c-1 (wrapping)
      o.cell[o.count] = g / N;
      o.loc[o.count++] = 0;
      o.cell[o.count] = (g / N - 1 + counts[d]) % counts[d];
      o.loc[o.count++] = N;
    } else {
      if (g > 0) {
        o.cell[o.count] = g / N - 1;
        o.loc[o.count++] = N;
      }
      if (g < span) {
        o.cell[o.count] = g / N;
        o.loc[o.count++] = 0;
      }
    }
    return o;
  }

  // lattice coordinate of local index loc in cell c along d
  SBX_HD int64_t coord(int d, int64_t c, int loc) const {
    int64_t g = c * N + loc;
    if (per[d]) g %= gdim[d];
    return g;
  }

  // All copies (global element, local node index within the element) of the
  // lattice point (g0, g1, g2), sorted in the reference's canonical order
  // (ascending global local-node index).  Returns the count (<= 8).
  SBX_HD int copies(int64_t g0, int64_t g1, int64_t g2, int64_t* elem, int* lidx) const {
    const int n = N + 1;
    const AxisOpts o0 = opts(0, g0), o1 = opts(1, g1), o2 = opts(2, g2);
    int64_t key[8];
    int m = 0;
    for (int c2 = 0; c2 < o2.count; ++c2)
      for (int c1 = 0; c1 < o1.count; ++c1)
        for (int c0 = 0; c0 < o0.count; ++c0) {
          const int64_t e = o0.cell[c0] + counts[0] * (o1.cell[c1] + (int64_t)counts[1] * o2.cell[c2]);
          const int l = (o2.loc[c2] * n + o1.loc[c1]) * n + o0.loc[c0];
          elem[m] = e;
          lidx[m] = l;
          key[m] = e * (int64_t)n * n * n + l;
          ++m;
        }
    for (int x = 1; x < m; ++x)
      for (int y = x; y > 0 && key[y - 1] > key[y]; --y) {
        const int64_t tk = key[y - 1];
        key[y - 1] = key[y];
        key[y] = tk;
        const int64_t te = elem[y - 1];
        elem[y - 1] = elem[y];
        elem[y] = te;
        const int tl = lidx[y - 1];
        lidx[y - 1] = lidx[y];
        lidx[y] = tl;
      }
    return m;
  }
};

}  // namespace sbx
