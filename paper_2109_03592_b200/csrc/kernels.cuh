// Device-side data views and kernel launchers (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sbx {

// Operator data resident in HBM.
struct OpDev {
  int64_t E = 0;
  int n = 0;                    // N+1
  int64_t nodes = 0;            // E*n^3
  const double* G = nullptr;    // packed geometry [E][6][n^3]  (g1,g2,g3,g4,g5,g6)
  const double* bm = nullptr;   // [E*n^3] or null
  const double* mask = nullptr; // [E*n^3] or null
  const double* inv_mult = nullptr;
  const uint8_t* mult8 = nullptr;  // multiplicity per node (clamped to 255)
  const double* Dd = nullptr;   // device copy of D (n*n)
  double Dh[33 * 33];           // host copy of D (kernel parameter source), n <= 33
  // boundary CSR: every gs group that is not an element-interior singleton
  // (shared groups + masked or element-boundary singletons), groups ascending
  // by gid, copies ascending by local index; copy index ~a marks mask == 0.
  int64_t nB = 0;
  int64_t nBcopies = 0;
  const int32_t* b_off = nullptr;  // nB+1
  const int32_t* b_idx = nullptr;  // nBcopies
  // Structured box (set when the map/mask are known to be build_gather_scatter /
  // build_dirichlet_mask of an ex*ey*ez box): enables the element-centric
  // gather-scatter that derives every copy from the cell lattice instead of
  // reading the CSR.  Requires count_d >= 2 in every periodic direction.
  bool box = false;
  int ex = 0, ey = 0, ez = 0;
  int per[3] = {0, 0, 0};
};

// Device-resident CG scalars for the fused (FAST) solver.
struct CgScalars {
  double rz;        // r'z (weighted) of the current residual
  double rr;        // r'r (weighted)
  double pq;        // p'Aq of the current iteration
  double alpha;     // rz/pq of the current iteration
  double alpha_prev;
  double beta;      // rz_new/rz
  double bnorm;     // ||b||
  double bmb;       // b'Mb
  double tol;
  double rel, relp;
  int32_t it;       // iterations completed
  int32_t max_it;
  int32_t first;    // 1 before the first p-update
  int32_t done;     // 1: converged / max iterations / error
  int32_t converged;
  int32_t status;   // 0 ok, 5 breakdown, 6 NaN
  int32_t err_it;
  int32_t pad;
  uint32_t counter[4];  // last-block-done tickets
};

// ---- standalone operators (ops.cu) ----------------------------------------
cudaError_t launch_axhelm(const OpDev& op, const double* u, double* w, double h1, double h2,
                          bool exact, bool flip, cudaStream_t s);
cudaError_t launch_axhelm_diag(const OpDev& op, double h1, double h2, double* diag,
                               cudaStream_t s);
// gs over the boundary CSR; apply_mask multiplies every copy by its mask
// (HelmholtzOperator::apply), otherwise masked singletons are untouched and
// only groups with >1 copy are summed (gs_sum_inplace).
cudaError_t launch_gs(const OpDev& op, double* f, bool apply_mask, cudaStream_t s);
// reference-order dot: per-element sequential partials, then a serial sum
cudaError_t launch_dot_exact(const OpDev& op, const double* a, const double* b,
                             const double* w, double* partials, double* out, cudaStream_t s);
// deterministic tree dot (block partials + last-block fixed-order sum)
cudaError_t launch_dot_fast(int64_t N, const double* a, const double* b, const double* w,
                            double* partials, uint32_t* counter, double* out, cudaStream_t s);
cudaError_t launch_axpy(int64_t N, double alpha, const double* x, double* y, cudaStream_t s);
cudaError_t launch_scale(int64_t N, double alpha, double* y, cudaStream_t s);
cudaError_t launch_div(int64_t N, const double* r, const double* d, double* z, cudaStream_t s);
cudaError_t launch_mul(int64_t N, const double* a, double* b, cudaStream_t s);
cudaError_t launch_pack_geometry(const OpDev& op, const double* const* g_soa, double* G,
                                 cudaStream_t s);
cudaError_t launch_recip(int64_t N, const double* d, double* dinv, cudaStream_t s);

// ---- fused FAST CG (cg.cu) -------------------------------------------------
struct CgVecs {
  double* x;
  double* r;
  double* p;
  double* w;
  const double* dinv;  // 1/diag (Jacobi) or ones
  double* partials;    // >= 2 * max blocks
  CgScalars* sc;
};

}  // namespace sbx
