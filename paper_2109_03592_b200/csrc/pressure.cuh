// Pressure-operator engine (pressure.cu): setup of the P_N / P_N-2 data, the
// standalone operators, and the FAST pressure PCG with the deflated Jacobi
// preconditioner of FlowSolver::pressure_precond (stepper.cpp:277-308).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sbx.h"
#include "kernels.cuh"

namespace sbx {

class PressureEngine {
 public:
  PressureEngine() = default;
  ~PressureEngine();
  // mats, inv_bdiag (mask / gs_sum(bm)); needs the trilinear map (op.tl)
  int setup(const OpDev& op, cudaStream_t s);
  int ensure_diag(cudaStream_t s);  // pressure_operator_diagonal and its reciprocal
  int grad(const double* p, double* const g[3], cudaStream_t s);
  int div(const double* const v[3], double* q, cudaStream_t s);
  int apply(const double* p, double* q, cudaStream_t s);
  int solve(cudaStream_t s, const double* b, double* x, const sbx_pcg_config& cfg,
            sbx_pcg_result* res);
  // EXACT (reference evaluation order, bitwise): pressure_exact.cu kernels
  int grad_exact(const double* p, double* const g[3], cudaStream_t s);
  int div_exact(const double* const v[3], double* q, cudaStream_t s);
  int apply_exact(const double* p, double* q, cudaStream_t s);
  int ensure_diag_exact(cudaStream_t s);
  const double* diag_exact() const { return pdiag_x_; }
  int solve_exact(cudaStream_t s, const double* b, double* x, const sbx_pcg_config& cfg,
                  sbx_pcg_result* res);
  // ProjectionHistory (krylov.cpp:93-124) on the pressure grid: the
  // A-orthonormal (x, E x) pairs live on the device
  int proj_reset(int depth);
  int proj_guess(cudaStream_t s, const double* b, double* guess, double* deflated, bool exact);
  int proj_append(cudaStream_t s, const double* x, bool exact);
  int proj_size() const { return (int)basis_.size(); }
  const double* diag() const { return pdiag_; }
  int64_t pnodes() const { return P_.Np; }
  int m1d() const { return P_.m; }
  bool ready() const { return ready_; }
  const std::string& error() const { return err_; }

 private:
  int ensure_work(int max_it);
  int build_graph(cudaStream_t s, double* x, const double* dinv);

  const OpDev* op_ = nullptr;
  PresDev P_;
  bool ready_ = false;
  double* mats_ = nullptr;
  std::vector<double> hmats_;
  PresExact X_;
  double* xmats_ = nullptr;   // d | iv | ivt | glx | glw (EXACT kernels)
  double* pdiag_x_ = nullptr;
  double* zx_ = nullptr;      // EXACT loop: z
  double* scal_ = nullptr;    // device scalars [4]
  double* inv_bdiag_ = nullptr;
  double* pdiag_ = nullptr;
  double* pdinv_ = nullptr;
  double* g_[3] = {};
  double* v_[3] = {};
  double *r_ = nullptr, *p_ = nullptr, *q_ = nullptr, *partials_ = nullptr, *hist_ = nullptr;
  int64_t hist_len_ = 0;
  double* sums_ = nullptr;  // device [8]
  uint32_t* counter_ = nullptr;
  int* flag_ = nullptr;
  CgScalars* sc_ = nullptr;
  CgScalars* hsc_ = nullptr;
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
  const void* gkey_[4] = {};
  int pdot(cudaStream_t s, const double* a, const double* b, bool exact, double* out);
  std::deque<std::pair<double*, double*>> basis_;
  std::vector<double*> pool_;
  int depth_ = 0;
  double *pv_ = nullptr, *pw_ = nullptr;  // append scratch
  std::string err_;
};

}  // namespace sbx
