// Device-side data views and kernel launchers (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sbx {

struct DistDev;

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
  int ex = 0, ey = 0, ez = 0;  // GLOBAL box dims
  int per[3] = {0, 0, 0};
  // multi-GPU: this rank's elements are a subset; partners via the
  // 27-neighbourhood table (local id / -1 outside / -2 on another rank)
  bool table = false;
  const int32_t* nbr27 = nullptr;
  const int64_t* gelem = nullptr;
  const DistDev* dd = nullptr;  // device copy of the exchange state (multi-GPU)
  // trilinear elements (box contexts): per-element map coefficients [E][24]
  // (see trilinear_coeffs) and the GLL nodes / weights, so the fused CG
  // kernel can form the metric at each node instead of streaming G
  const double* tl = nullptr;
  // per-node Helmholtz coefficients (HelmholtzCoeffs::h1_field / h2_field,
  // operators.hpp:42-43; sbx_ctx_set_coeff_fields), or null: the scalars
  const double* h1f = nullptr;
  const double* h2f = nullptr;
  const double* corners = nullptr;  // [E][8][3] (box / verified-hint contexts)
  double Xh[33], Wh[33];
  // lattice gather-scatter: mask / multiplicities / gs / rhs check derived
  // from the box lattice on the device (setup_dev.cu); no boundary CSR
  bool lat = false;
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
  int32_t nranks;   // > 1: distributed (rank-local partials, exchange kernels)
  uint32_t counter[4];  // last-block-done tickets
  double pq_loc, rz_loc, rr_loc;  // this rank's partials (distributed)
  // single-graph solve: what the device prologue found (kPre* bits)
  int32_t pre;
  // distributed: the update kernel left this rank's r'z / r'r partials in
  // rz_loc / rr_loc; the next K1 exchanges them and takes the scalar step
  int32_t xpend;
  double mu;  // pressure CG: mean of r/diag (the deflated preconditioner)
  // distributed: the residual history (the scalar step runs in K1) and a
  // marker for a K1 that only found the solve finished (timing mode)
  double* hist;
  int64_t hist_cap;
  int32_t k1_idle;
  int32_t pad_;
};
// A batched solve of up to kMaxComp right-hand sides with one operator (the
// three velocity components of FlowSolver::solve_velocity_star,
// stepper.cpp:188-238): the fused kernels run with grid.y = component, every
// component with its own vectors and scalars (device copy of this struct).
constexpr int kMaxComp = 3;
struct CgMulti {
  int ncomp;
  double* r[kMaxComp];
  double* p[kMaxComp];
  double* x[kMaxComp];
  double* w[kMaxComp];
  CgScalars* sc[kMaxComp];
  double* hist[kMaxComp];
  int64_t part_stride;  // partials per component
};
// any component still iterating (the batched loop's WHILE condition)
__device__ __forceinline__ bool multi_active(const CgMulti* m) {
  bool a = false;
  for (int c = 0; c < m->ncomp; ++c) a |= (*(const volatile int32_t*)&m->sc[c]->done) == 0;
  return a;
}
// CgScalars::pre
constexpr int kPreNonzeroX = 1;  // x0 != 0: r = b - A x0 needs the general path
constexpr int kPreRhsBad = 2;    // b not continuous / not masked: EXACT fallback
constexpr int kPreZeroRhs = 4;   // b'Wb == 0: x = 0, converged (krylov.cpp:11-16)
// solve parameters read by the device prologue (H2D before each graph launch)
struct CgParams {
  double tol;
  int32_t max_it;
  int32_t pad_;
};

// ---- multi-GPU peer windows ------------------------------------------------
constexpr int kMaxRanks = 8;
// Window layout (bytes): flags [4 phases][kMaxRanks] u64 at 0, mailboxes
// [4 phases][2 parities][kMaxRanks][4] f64 at 256, RECEIVE buffers
// [2 slots][2 parities][recv_total] f64 at 2304.  Phases: 0 halo+p'Ap in the
// CG loop, 1 r'z/r'r, 2 standalone gather-scatter halo, 3 setup reductions.
// The halo is PUSHED: a sender stores its interface copy values into each
// neighbour's receive buffer over NVLink as soon as they are computed (the
// K1 epilogue); the next kernel (K2), once K1 has completed, releases the
// phase with one system fence and relaxed flag stores; the receiver then
// reads only local memory.  The r'z / r'r partials of K2 are released by the
// next K1's head.  Parity = sequence number & 1: a peer can run at most one
// use of a phase ahead (it needs this rank's flag of the previous use, and a
// kernel starts only after its predecessor -- the last reader of the other
// parity -- has completed), so double buffering makes every access race-free.
constexpr size_t kWinFlags = 0, kWinMbox = 256, kWinRecv = 2304;

__host__ __device__ constexpr int mbox_index(int phase, int par, int src, int c) {
  return ((phase * 2 + par) * kMaxRanks + src) * 4 + c;
}

struct DistDev {
  int nranks = 1, rank = 0;
  int64_t nodes_local = 0;
  unsigned long long* flags = nullptr;  // my window
  double* mbox = nullptr;
  double* recvb = nullptr;              // my receive buffer [2 slots][2 par][recv_total]
  int64_t recv_total = 0;
  int64_t send_total = 0;
  unsigned long long* pflags[kMaxRanks] = {};  // peer windows (own rank: mine)
  double* pmbox[kMaxRanks] = {};
  double* precv[kMaxRanks] = {};       // peer q's receive buffer
  int64_t precv_total[kMaxRanks] = {};
  int64_t pbase_for_me[kMaxRanks] = {};  // offset of my block in q's receive buffer
  int nnbr = 0;
  int nbr[kMaxRanks] = {};
  int64_t send_off[kMaxRanks + 1] = {};
  int64_t recv_base[kMaxRanks + 1] = {};  // per neighbour index, + total
  const int32_t* send_idx = nullptr;
  int64_t n_if = 0;
  const int32_t* if_off = nullptr;
  const int32_t* if_code = nullptr;
  const int32_t* nbr27 = nullptr;  // local elements' 27-neighbourhood
  const int64_t* gelem = nullptr;  // global element id of each local element
  // sends regrouped by local element (K1 epilogue puts them on the wire)
  const int32_t* esend_off = nullptr;
  const int32_t* esend_node = nullptr;
  const int32_t* esend_q = nullptr;
  const int32_t* esend_pos = nullptr;
  unsigned long long* seq = nullptr;  // device [4]
  unsigned int* counter = nullptr;    // device [4]
  unsigned int* gbar = nullptr;       // device [2]: grid barrier of the update kernel
  int* status = nullptr;              // device: 1 on exchange timeout
  // SBX_TRACE: per-iteration %globaltimer stamps [kTraceIters][8] (diagnostics)
  unsigned long long* trace = nullptr;
};
constexpr int kTraceIters = 4096;

// distributed gather-scatter of a local field (halo exchange over the peer
// windows, interface groups summed in canonical order, then the local
// boundary CSR); apply_mask as in launch_gs
cudaError_t launch_dist_gs(const OpDev& op, const DistDev& D, double* f, bool apply_mask,
                           cudaStream_t s);
// sum of up to 4 doubles over all ranks, in rank order (device in/out)
cudaError_t launch_dist_allreduce(const DistDev& D, int phase, const double* in, double* out,
                                  int count, cudaStream_t s);

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

// ---- device-side setup of box contexts (setup_dev.cu) ----------------------
// packed geometry G [E][6][n^3] and bm from the element corners [E][8][3];
// *bad = smallest element with detJ <= 0 (initialise to ~0ull)
cudaError_t launch_geom_box(const double* corners, int64_t E, int n, const double* x,
                            const double* w, double* G, double* bm, unsigned long long* bad,
                            cudaStream_t s);
cudaError_t launch_lattice_fields(const OpDev& op, double* mask, double* inv_mult,
                                  uint8_t* mult8, cudaStream_t s);
cudaError_t launch_gs_box(const OpDev& op, double* f, bool apply_mask, cudaStream_t s);
cudaError_t launch_check_rhs_box(const OpDev& op, const double* f, int* flag, cudaStream_t s);
// *flag := 1 unless the caller's map (device int64 copies; may be null) and
// mask (may be null) are the box lattice's of op (ex/ey/ez/per/n set)
cudaError_t launch_validate_box(const OpDev& op, int64_t G, const int64_t* offsets,
                                const int64_t* group_nodes, const double* mask, int* flag,
                                cudaStream_t s);
// *flag := 1 unless packed G (and bm, if given) equal the corners' metric bitwise
cudaError_t launch_validate_geom(const double* corners, int64_t E, int n, const double* x,
                                 const double* w, const double* G, const double* bm, int* flag,
                                 cudaStream_t s);

// ---- consistent-Poisson pressure operator (pressure.cu) --------------------
// Element data of the P_N / P_N-2 pair: n = N+1 GLL, m = N-1 GL points; the
// 1-D operators [I^T | (I D)^T | I | I D | GL w | GL x] (device) and the
// trilinear map coefficients of every element (the GL metric is formed on
// the fly).
struct PresDev {
  int n = 0, m = 0;
  int64_t E = 0, Np = 0;  // elements, pressure nodes E*m^3
  const double* tl = nullptr;
  const double* mats = nullptr;
  const double* hmats = nullptr;  // host copy (kernel-parameter operators)
};
cudaError_t launch_p_grad(const PresDev& P, const double* p, double* const g[3], cudaStream_t s);
cudaError_t launch_p_div(const PresDev& P, const double* const v[3], double* q, cudaStream_t s);
cudaError_t launch_p_diag(const PresDev& P, const double* inv_bdiag, double* diag,
                          cudaStream_t s);
// g_c := scale * gs_sum(g_c) for c = 0..2 (gather-scatter of the velocity-grid
// gradient, then the masked inverse assembled mass; stepper.cpp:242-245)
cudaError_t launch_gs3_scale(const OpDev& op, double* const g[3], const double* scale,
                             cudaStream_t s, double* const* out = nullptr);
struct PIterArgs {
  const OpDev* op;
  const double* inv_bdiag;
  double* r;
  const double* dinv;  // null: no preconditioner (deflation only)
  double* p;
  double* x;
  double* q;
  double* g[3];
  double* v[3];  // scale * gs(g) (out of place)
  double* partials;
  CgScalars* sc;
  double* hist;
  int64_t hist_cap;
};
// EXACT (reference-order) pressure operators (pressure_exact.cu)
struct PresExact {
  int n = 0, m = 0;
  int64_t E = 0;
  const double* corners = nullptr;  // [E][8][3]
  const double* d = nullptr;        // GLL derivative n x n
  const double* iv = nullptr;       // interp_v2p m x n
  const double* ivt = nullptr;      // n x m
  const double* glx = nullptr;      // GL nodes
  const double* glw = nullptr;      // GL weights
};
cudaError_t launch_p_grad_exact(const PresExact& X, const double* p, double* const g[3],
                                cudaStream_t s);
cudaError_t launch_p_div_exact(const PresExact& X, const double* const u[3], double* out,
                               cudaStream_t s);
cudaError_t launch_p_diag_exact(const PresExact& X, const double* inv_bdiag, double* diag,
                                cudaStream_t s);
// advect (operators.cpp:412-431): out_c = bm (c . grad u_c), reference order
// (bitwise); D, gllx device arrays of the GLL basis
cudaError_t launch_advect(int64_t E, int n, const double* corners, const double* D,
                          const double* gllx, const double* bm, const double* const u[3],
                          const double* const c[3], double* const out[3], cudaStream_t s);
// z -= mean(z) with the mean summed sequentially (stepper.cpp:278-283)
cudaError_t launch_deflate_exact(int64_t N, double* z, double* mean_scratch, cudaStream_t s);
// field_dot (field.cpp:59-67): per-element sequential partials, serial sum
cudaError_t launch_dot_exact_n(int64_t E, int nper, const double* a, const double* b,
                               double* partials, double* out, cudaStream_t s);
cudaError_t launch_p_iteration(const PresDev& P, const PIterArgs& A,
                               cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s);
// out[8] = [b'b, b'(b/d), sum b/d, sum b, r'(r/d), sum r/d, sum r, r'r]
cudaError_t launch_p_init(const PresDev& P, const double* b, const double* r, const double* dinv,
                          double* partials, uint32_t* counter, double* out, cudaStream_t s);
cudaError_t launch_p_finish(const PresDev& P, const double* p, double* x, const CgScalars* sc,
                            cudaStream_t s);

// ---- fused FAST CG (cg.cu) -------------------------------------------------
// Whether the multi-GPU solver has a pipelined K1 (the halo leaves from its
// epilogue) for n = N+1 points per direction: Poisson with and without
// Jacobi (the trilinear or the stored-geometry layout must fit shared memory).
bool dist_k1_supported(int n);
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
