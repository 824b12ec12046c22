// Internal declarations shared by the host setup, the CUDA kernels and the
// C ABI (include/sbx.h).  Not a public header.
#pragma once

#include <cstdint>
#include <functional>
#include <string>

#include "../../include/sbx.h"

namespace sbx {

constexpr int kMaxDegree = 32;     // build_gll_basis limit (basis.cpp:11, 61-63)
constexpr int kMaxTemplN = 15;     // tensor kernels are specialised for N <= 15 (n <= 16)

void set_error(const std::string& msg);

// host setup (setup.cpp)
void host_parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn);
int gll_basis(int degree, double* nodes, double* weights, double* deriv);
int pressure_basis(int degree, double* nodes, double* weights, double* interp);
int box_corners(int ex, int ey, int ez, const double* origin, const double* lengths,
                double* corners);
void deform_corners(int64_t elem_count, double a, double* corners);
int geometric_factors(int64_t E, int degree, const double* corners, double* const g[6],
                      double* bm, double* jac, int64_t* bad_elem);
int gather_scatter(int ex, int ey, int ez, const int* periodic, int degree, int64_t* gid,
                   int64_t* offsets, int64_t* group_nodes, int32_t* mult, double* inv_mult,
                   int64_t* global_count);
int dirichlet_mask(int ex, int ey, int ez, const int* periodic, int degree, double* mask);
int partition_rcb(int64_t E, const double* corners, int ranks, int32_t* rank_of);
// Coefficients of each element's trilinear map derivatives (on-the-fly
// metrics of the fused CG kernel): tl[e][24] = S0, S1, S2, S01, S02, S12,
// S012 (xyz each) and 3 pads, with
//   dX/dr = S0 + S01 s + S02 t + S012 s t,  dX/ds = S1 + S01 r + S12 t + S012 r t,
//   dX/dt = S2 + S02 r + S12 s + S012 r s.
void trilinear_coeffs(int64_t E, const double* corners, double* tl);

}  // namespace sbx
