// Fused FAST PCG engine: two kernels per iteration, device-resident scalars,
// the whole iteration loop in one CUDA graph with a conditional WHILE node.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/sbx.h"
#include "kernels.cuh"

namespace sbx {

struct CgRun {
  const OpDev* op = nullptr;
  cudaStream_t stream = nullptr;
  const double* b = nullptr;  // device
  double* x = nullptr;        // device, initial guess in / solution out
  const double* dinv = nullptr;  // 1/assembled diagonal, or null (no preconditioner)
  double h1 = 1.0, h2 = 0.0, tol = 1e-8;
  int max_it = 500;
  double* history = nullptr;  // host
  int64_t history_capacity = 0;
  bool interior_clean = false;
  bool timing = false;
  const DistDev* dist = nullptr;  // multi-GPU exchange state, or null
};

// Returned by solve() when the FAST schedule's preconditions do not hold
// (non-continuous / unmasked right-hand side, exotic maps): run EXACT instead.
constexpr int kCgFallback = -1;

class CgEngine {
 public:
  CgEngine() = default;
  ~CgEngine();
  int solve(const CgRun& run, sbx_pcg_result* res);
  const std::string& error() const { return err_; }
  int kernel_time(const char* name, double* total_ms, int64_t* launches) const;
  // Batched solve of count <= kMaxComp right-hand sides with one operator
  // (the velocity components of FlowSolver::solve_velocity_star): one graph,
  // K1 / K2 with grid.y = component, each component's initial guess applied
  // in the graph; per component the same arithmetic as solve().
  int solve_multi(const CgRun* runs, int count, sbx_pcg_result* res);
  // Test hook: one launch of the solver's K1 in its first-iteration form
  // (p = r, no preconditioner, x untouched) on u, so w = A_local u comes out
  // of exactly the kernel (and metric variant) the solve runs.
  int debug_k1(const OpDev& op, cudaStream_t s, const double* u, double* w, double h1,
               double h2);

 private:
  int ensure(const CgRun& run);
  int build_graph(const CgRun& run);
  int build_solve_graph(const CgRun& run);
  int solve_graph(const CgRun& run, sbx_pcg_result* res, bool* general);
  int collect(const CgRun& run, sbx_pcg_result* res);
  int collect_from(const CgScalars& o, const double* dhist, const CgRun& run,
                   sbx_pcg_result* res);
  int ensure_multi(const CgRun& run, int count);
  int build_multi_graph(const CgRun* runs, int count);
  int run_timed_loop(const CgRun& run);

  const OpDev* op_ = nullptr;
  int64_t nodes_ = 0;
  double* r_ = nullptr;
  double* p_ = nullptr;
  double* w_ = nullptr;
  double* partials_ = nullptr;
  int64_t partials_len_ = 0;
  CgScalars* sc_ = nullptr;
  CgScalars* hsc_ = nullptr;  // pinned
  double* hist_ = nullptr;    // device history
  int64_t hist_len_ = 0;
  double* init_ = nullptr;    // device init sums [4]
  int* flag_ = nullptr;       // device continuity flag
  CgParams* prm_ = nullptr;   // device solve parameters
  CgParams* hprm_ = nullptr;  // pinned
  // the single-graph solve (prologue + loop + finish), cached like graph_
  cudaGraph_t sgraph_ = nullptr;
  cudaGraphExec_t sexec_ = nullptr;
  bool have_sgraph_ = false;
  // batched solves
  const OpDev* mop_ = nullptr;
  int mcount_ = 0;
  double *mr_[kMaxComp] = {}, *mp_[kMaxComp] = {}, *mw_[kMaxComp] = {};
  double* mhist_[kMaxComp] = {};
  int64_t mhist_len_ = 0;
  CgScalars* msc_ = nullptr;   // device [kMaxComp]
  CgScalars* mhsc_ = nullptr;  // pinned
  double* mpart_ = nullptr;
  int64_t mstride_ = 0;
  int* mflag_ = nullptr;       // rhs check per component
  CgParams* mprm_ = nullptr;
  CgParams* mhprm_ = nullptr;  // pinned
  CgMulti* dmulti_ = nullptr;
  cudaGraph_t mgraph_ = nullptr;
  cudaGraphExec_t mexec_ = nullptr;
  const void* mkey_[2 * kMaxComp + 4] = {};
  double mkey_h_[2] = {0.0, 0.0};
  // graph cache
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
  struct Key {
    const void* op;
    const void* x;
    const void* dinv;
    double h1, h2;
    const void* hist;
    cudaStream_t stream;
    const void* b;
    bool operator==(const Key& o) const {
      return op == o.op && x == o.x && dinv == o.dinv && h1 == o.h1 && h2 == o.h2 &&
             hist == o.hist && stream == o.stream && b == o.b;
    }
  } key_{}, skey_{};
  bool have_graph_ = false;
  // per-kernel timing (timing mode)
  double t_ax_ms_ = 0, t_upd_ms_ = 0;
  int64_t n_ax_ = 0, n_upd_ = 0;
  std::string err_;
};

}  // namespace sbx
