// Geometric factors at one node of a trilinear hexahedron: Jacobian J[p][q] =
// dx_p/dxi_q accumulated corner by corner, its determinant, inverse, and the
// symmetric metric w*detJ*J^-1 J^-T (reference: operators.cpp:19-57,
// 123-178, expression by expression).  Shared by the host builder
// (setup.cpp, -ffp-contract=off) and the device builder (setup_dev.cu,
// -fmad=false), so both round every operation the way the reference does and
// produce identical bits.
#pragma once

#include "lattice.h"  // SBX_HD

namespace sbx {

struct Metric {
  double g[6];
  double wdet;
  double det;
};

SBX_HD inline bool node_metric(const double* cr, double r, double s, double t, double w,
                               Metric& m) {
  const double sh[3][2] = {{0.5 * (1 - r), 0.5 * (1 + r)},
                           {0.5 * (1 - s), 0.5 * (1 + s)},
                           {0.5 * (1 - t), 0.5 * (1 + t)}};
  double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int v = 0; v < 8; ++v) {
    const int b0 = v & 1, b1 = (v >> 1) & 1, b2 = (v >> 2) & 1;
    const double d0 = b0 ? 0.5 : -0.5, d1 = b1 ? 0.5 : -0.5, d2 = b2 ? 0.5 : -0.5;
    const double gr[3] = {d0 * sh[1][b1] * sh[2][b2], sh[0][b0] * d1 * sh[2][b2],
                          sh[0][b0] * sh[1][b1] * d2};
    for (int p = 0; p < 3; ++p) {
      const double xp = cr[v * 3 + p];
      J[p * 3 + 0] += xp * gr[0];
      J[p * 3 + 1] += xp * gr[1];
      J[p * 3 + 2] += xp * gr[2];
    }
  }
  const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                     J[2] * (J[3] * J[7] - J[4] * J[6]);
  if (!(det > 0.0)) return false;
  const double id = 1.0 / det;
  const double R[9] = {(J[4] * J[8] - J[5] * J[7]) * id, (J[2] * J[7] - J[1] * J[8]) * id,
                       (J[1] * J[5] - J[2] * J[4]) * id, (J[5] * J[6] - J[3] * J[8]) * id,
                       (J[0] * J[8] - J[2] * J[6]) * id, (J[2] * J[3] - J[0] * J[5]) * id,
                       (J[3] * J[7] - J[4] * J[6]) * id, (J[1] * J[6] - J[0] * J[7]) * id,
                       (J[0] * J[4] - J[1] * J[3]) * id};
  const double wd = w * det;
  auto gd = [&](int p, int q) {
    return wd * (R[p * 3] * R[q * 3] + R[p * 3 + 1] * R[q * 3 + 1] + R[p * 3 + 2] * R[q * 3 + 2]);
  };
  m.g[0] = gd(0, 0);
  m.g[1] = gd(1, 1);
  m.g[2] = gd(2, 2);
  m.g[3] = gd(0, 1);
  m.g[4] = gd(0, 2);
  m.g[5] = gd(1, 2);
  m.wdet = wd;
  m.det = det;
  return true;
}

}  // namespace sbx
