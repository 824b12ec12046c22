/*
 * sbx.h -- C ABI of the B200-native spectral-element PCG hot path.
 *
 * Drop-in boundary for the reference's ("sembox", /root/reference/proj)
 * operator API on the preconditioned-CG path.
 * Plain pointers and sizes only: no C++ or torch types cross this boundary.
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj).
 *
 * Data layout (identical to the reference, so host<->device copies are flat):
 *   field  : E * n^3 doubles, index ((e*n + k)*n + j)*n + i, x fastest,
 *            elements outermost                     (include/sembox/field.hpp:15-36)
 *   deriv  : n*n row-major, D[i*n+j] = l_j'(x_i)     (include/sembox/basis.hpp:15)
 *   g1..g6, bm : E*n^3 each (GeometricFactors SoA)   (include/sembox/operators.hpp:18-26)
 *   gather-scatter map: group_offsets[G+1], group_nodes[E*n^3] (int64), groups
 *            ascending by gid, copies ascending by local index (include/sembox/gather.hpp:14-29)
 *
 * Vector arguments of the operator/solver calls may be DEVICE pointers (the
 * fast path) or HOST pointers (pageable or pinned; staged through the
 * context's buffers) -- detected per call with cudaPointerGetAttributes.
 *
 * Errors: every call returns an sbx_status; sbx_last_error() gives the
 * message (thread-local).  The codes map one-to-one onto the reference's
 * exception taxonomy (include/sembox/errors.hpp:10-41).
 *
 * Threading: calls on one context are synchronous (stream-ordered inside,
 * synchronised at return).  Distinct contexts may be used from distinct
 * threads.  Results are deterministic for a fixed device count.
 */
#ifndef SBX_H
#define SBX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SBX_OK = 0,
  SBX_E_INVALID = 1,   /* null pointer / bad flag / bad handle                     */
  SBX_E_CONFIG = 2,    /* sembox::ConfigError  (bad degree, bad rank count, ...)   */
  SBX_E_SHAPE = 3,     /* sembox::ContractViolation (grid/shape/map mismatch)      */
  SBX_E_MESH = 4,      /* sembox::MeshError (nonpositive Jacobian)                 */
  SBX_E_BREAKDOWN = 5, /* sembox::SolverError: p'Ap <= 0 or non-finite (krylov.cpp:61-64) */
  SBX_E_NAN = 6,       /* sembox::SolverError: residual NaN/Inf (krylov.cpp:72-75)  */
  SBX_E_CUDA = 7,      /* CUDA runtime failure                                      */
  SBX_E_COMM = 8,      /* NCCL / communicator failure                               */
  SBX_E_NOMEM = 9      /* device allocation failed                                  */
} sbx_status;

/* operator flags */
#define SBX_FLAG_EXACT 0x1u  /* reference evaluation order, no FMA: bitwise equal to sembox */
#define SBX_FLAG_FLIP_T 0x2u /* debug::axhelm_sign_flip (operators.hpp:114-118, operators.cpp:221) */
#define SBX_FLAG_NO_MASK 0x4u /* HelmholtzOperator with mask == nullptr (operators.hpp:107) */

const char* sbx_last_error(void);
const char* sbx_version(void);

/* ------------------------------------------------------------ host setup --
 * Host-side builders of the operator inputs.  The product's own C++ (not the
 * reference); bitwise equal to the reference builders (tests/test_setup.py). */

/* build_gll_basis (basis.cpp:60-112): nodes[n], weights[n], deriv[n*n]. */
sbx_status sbx_gll_basis(int degree, double* nodes, double* weights, double* deriv);

/* build_box_mesh corners (mesh.cpp:21-52): corners[E][8][3]. */
sbx_status sbx_box_corners(int ex, int ey, int ez, const double origin[3],
                           const double lengths[3], double* corners);

/* conforming sin-bump deformation of the benchmark meshes. */
sbx_status sbx_deform_corners(int64_t elem_count, double amplitude, double* corners);

/* build_geometric_factors (operators.cpp:123-178).  Any of the outputs may be
 * NULL.  *bad_elem = -1, or the first element with detJ <= 0 (SBX_E_MESH). */
sbx_status sbx_geometric_factors(int64_t elem_count, int degree, const double* corners,
                                 double* g1, double* g2, double* g3, double* g4,
                                 double* g5, double* g6, double* bm, double* jac,
                                 int64_t* bad_elem);

/* build_gather_scatter (gather.cpp:10-83) for a structured box.  gid, mult,
 * inv_mult may be NULL; group_offsets needs room for nodes+1 entries.
 * *global_count receives G. */
sbx_status sbx_gather_scatter(int ex, int ey, int ez, const int periodic[3], int degree,
                              int64_t* gid, int64_t* group_offsets, int64_t* group_nodes,
                              int32_t* mult, double* inv_mult, int64_t* global_count);

/* build_dirichlet_mask (operators.cpp:433-455). */
sbx_status sbx_dirichlet_mask(int ex, int ey, int ez, const int periodic[3], int degree,
                              double* mask);

/* partition_rcb (mesh.cpp:168-226): rank_of[E]. */
sbx_status sbx_partition_rcb(int64_t elem_count, const double* corners, int ranks,
                             int32_t* rank_of);

/* ------------------------------------------------------------ context ----- */
typedef struct sbx_ctx sbx_ctx;

/* Everything HelmholtzOperator holds (operators.hpp:103-108), as host arrays
 * in the reference layout.  Uploaded and re-laid-out for the device once. */
typedef struct {
  int64_t elem_count;           /* E (this rank's elements)                       */
  int32_t degree;               /* N (n = N+1 points per direction)               */
  const double* deriv;          /* n*n                                            */
  const double* g[6];           /* g1..g6                                         */
  const double* bm;             /* may be NULL when only h2 == 0 is used          */
  const double* mask;           /* may be NULL: no Dirichlet mask                 */
  int64_t global_count;         /* G                                              */
  const int64_t* group_offsets; /* G+1                                            */
  const int64_t* group_nodes;   /* E*n^3                                          */
  /* Optional structured-box hint (HexMesh::ex/ey/ez, periodic, corners;
   * mesh.hpp:14-33).  The reference's build_gather_scatter only accepts a
   * structured box (gather.cpp:11-12), so a sembox caller always has these.
   * When box[0] > 0 the context checks, on the device, that the map and mask
   * ARE the box lattice's (and, with corners, that g1..g6 are the corners'
   * trilinear metric, bitwise); if so it uses the lattice gather-scatter (no
   * CSR is built) and the fused solver's trilinear K1 / lattice K2, else it
   * falls back to the general path silently.  Zero-initialise to omit. */
  int32_t box[3];               /* ex, ey, ez (0: no hint)                        */
  int32_t periodic[3];
  const double* corners;        /* [E][8][3] or NULL                              */
} sbx_problem_desc;

sbx_status sbx_ctx_create(const sbx_problem_desc* desc, int device, sbx_ctx** out);

/* Product-native setup of a structured (optionally deformed) box: builds
 * corners, G, gs map, mask with the builders above (multi-threaded host) and
 * uploads them.  periodic[3]; amplitude 0 = undeformed. */
typedef struct {
  int ex, ey, ez;
  int degree;
  int periodic[3];
  double origin[3];
  double lengths[3];
  double deform_amplitude;
} sbx_box_desc;

sbx_status sbx_ctx_create_box(const sbx_box_desc* desc, int device, sbx_ctx** out);

void sbx_ctx_destroy(sbx_ctx* ctx);

/* E, n, local nodes, G, device bytes */
sbx_status sbx_ctx_info(const sbx_ctx* ctx, int64_t* elem_count, int32_t* n1d,
                        int64_t* nodes, int64_t* global_count, int64_t* device_bytes);

/* Which fused paths a context runs (a problem built without the box hint,
 * or whose hint did not verify, runs the general CSR / stored-geometry path). */
#define SBX_FEAT_LATTICE_GS 0x1u /* gather-scatter on the box lattice, no CSR      */
#define SBX_FEAT_BOX_K2 0x2u     /* lattice K2 (partner copies from the lattice)   */
#define SBX_FEAT_TRILINEAR 0x4u  /* K1 forms the metric from the trilinear map     */
sbx_status sbx_ctx_features(const sbx_ctx* ctx, uint32_t* features);

/* copy context-owned arrays (reference layout) to host or device memory:
 * which = 0 mask, 1 inv_mult, 2 bm, 3..8 g1..g6, 9 deriv */
sbx_status sbx_ctx_copy_array(const sbx_ctx* ctx, int which, double* out);

/* Launch stream (cudaStream_t as void*); NULL = the context's own stream. */
sbx_status sbx_ctx_set_stream(sbx_ctx* ctx, void* stream);

/* ------------------------------------------------------------ operators --- */

/* Per-node Helmholtz coefficients (HelmholtzCoeffs::h1_field / h2_field,
 * operators.hpp:42-43): E*n^3 fields (host or device pointers, copied into the
 * context) that replace the scalar h1 / h2 in every later axhelm,
 * axhelm_diagonal, apply and pcg on this context, read at each node where
 * operators.cpp:242, 258, 292-293 read them; NULL restores the scalar.  With
 * fields the operators and the solve run in the reference evaluation order in
 * either mode (the fused FAST kernels take scalars).  Single-process contexts;
 * h2 fields need bm. */
sbx_status sbx_ctx_set_coeff_fields(sbx_ctx* ctx, const double* h1_field,
                                    const double* h2_field);

/* axhelm (operators.hpp:59-60, operators.cpp:215-263): w = D^T G D u h1 + h2 bm u */
sbx_status sbx_axhelm(sbx_ctx* ctx, const double* u, double* w, double h1, double h2,
                      uint32_t flags);

/* axhelm_diagonal (operators.cpp:272-298); assembled != 0 adds gs_sum
 * (HelmholtzOperator::assembled_diagonal, operators.cpp:536-540). */
sbx_status sbx_axhelm_diagonal(sbx_ctx* ctx, double h1, double h2, int assembled,
                               double* diag);

/* gs_sum_inplace (gather.hpp:39, gather.cpp:85-98), bitwise equal. */
sbx_status sbx_gs_sum(sbx_ctx* ctx, double* field);

/* HelmholtzOperator::apply (operators.hpp:110, operators.cpp:530-534):
 * q = mask * gs_sum(axhelm(x)). */
sbx_status sbx_apply(sbx_ctx* ctx, const double* x, double* q, double h1, double h2,
                     uint32_t flags);

/* field_dot_weighted (field.hpp:60-62, field.cpp:69-81); weighted = 0 gives
 * field_dot.  SBX_FLAG_EXACT reproduces the reference's summation order. */
sbx_status sbx_dot(sbx_ctx* ctx, const double* a, const double* b, int weighted,
                   uint32_t flags, double* result);

/* --------------------------------------------------------------- solver --- */
typedef enum { SBX_PRECOND_NONE = 0, SBX_PRECOND_JACOBI = 1 } sbx_precond;

typedef enum {
  SBX_MODE_EXACT = 0, /* reference operation order; bitwise equal residual history   */
  SBX_MODE_FAST = 1   /* fused kernels, device-resident scalars, CUDA graph          */
} sbx_mode;

/* KrylovConfig (krylov.hpp:18-22) + the operator/preconditioner choice. */
typedef struct {
  double tolerance;       /* relative residual (default 1e-8)                      */
  int32_t max_iterations; /* default 500                                           */
  int32_t precond;        /* sbx_precond                                           */
  int32_t mode;           /* sbx_mode                                              */
  double h1, h2;          /* HelmholtzCoeffs (operators.hpp:39-44), scalars          */
  double* history;        /* host, optional: relative residual per iteration         */
  int64_t history_capacity;
} sbx_pcg_config;

/* PcgResult (krylov.hpp:24-30) + error iteration (SolverError::iteration). */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double rel_residual;
  double rel_residual_precond;
  int32_t error_iteration; /* -1 unless SBX_E_BREAKDOWN / SBX_E_NAN               */
  int64_t history_length;  /* entries produced (may exceed capacity)              */
} sbx_pcg_result;

void sbx_pcg_config_default(sbx_pcg_config* cfg);

/* pcg (krylov.hpp:38-40, krylov.cpp:7-91) on the assembled operator with the
 * multiplicity-weighted dot and (optionally) Jacobi on assembled_diagonal().
 * x carries the initial guess in and the solution out.  Reaching
 * max_iterations is reported (converged = 0), not an error. */
sbx_status sbx_pcg(sbx_ctx* ctx, const double* b, double* x, const sbx_pcg_config* cfg,
                   sbx_pcg_result* result);

/* ------------------------------------ consistent-Poisson pressure path ---
 * The P_N / P_N-2 pressure operator E = Div M^-1 QQ^T Grad of the paper's
 * splitting scheme.  Pressure fields: E * m^3 doubles,
 * m = N-1 GL points per direction (GridTag::pressure, field.hpp:13-16), same
 * element-major x-fastest order.  Needs N >= 3 and a context with the element
 * corners (sbx_ctx_create_box, or sbx_ctx_create with a verified box hint);
 * flags: SBX_FLAG_EXACT = the reference's evaluation order (bitwise equal,
 * the geometry from the corners as build_pressure_geometry forms it); default
 * FAST (fused kernels, the GL metric from the trilinear map on the fly, the
 * reference's results to rounding). */

/* build_pressure_basis (basis.cpp:114-145): nodes[m], weights[m],
 * interp_v2p[m*(N+1)] (row-major l_j(gl_i)). */
sbx_status sbx_pressure_basis(int degree, double* nodes, double* weights, double* interp_v2p);
/* pressure nodes E*m^3 and m */
sbx_status sbx_pressure_info(sbx_ctx* ctx, int64_t* pressure_nodes, int32_t* m1d);
/* gradient_from_pressure (operators.hpp:78-80, operators.cpp:365-410) */
sbx_status sbx_gradient_from_pressure(sbx_ctx* ctx, const double* p, double* gx, double* gy,
                                      double* gz, uint32_t flags);
/* divergence_to_pressure (operators.hpp:73-75, operators.cpp:327-363) */
sbx_status sbx_divergence_to_pressure(sbx_ctx* ctx, const double* ux, const double* uy,
                                      const double* uz, double* out, uint32_t flags);
/* FlowSolver::apply_pressure_operator (stepper.cpp:240-248): Div (mask/gs(bm)) gs Grad p */
sbx_status sbx_pressure_apply(sbx_ctx* ctx, const double* p, double* out, uint32_t flags);
/* FlowSolver::pressure_operator_diagonal (stepper.cpp:250-275) */
sbx_status sbx_pressure_diagonal(sbx_ctx* ctx, double* diag, uint32_t flags);
/* the pressure solve of FlowSolver::solve_pressure_update (stepper.cpp:326-347):
 * pcg with apply_pressure_operator, field_dot (plain) and pressure_precond
 * (stepper.cpp:277-308: Jacobi on the diagonal or none, each followed by the
 * mean deflation).  cfg->precond JACOBI or NONE; cfg->mode EXACT (the
 * reference's residual history bit for bit) or FAST; h1/h2 unused.
 * b must already have its mean removed (stepper.cpp:313-324). */
sbx_status sbx_pressure_pcg(sbx_ctx* ctx, const double* b, double* x, const sbx_pcg_config* cfg,
                            sbx_pcg_result* result);

/* ProjectionHistory (krylov.hpp:45-64, krylov.cpp:93-124) of the pressure
 * solve (stepper.cpp:326, 345): A-orthonormal (x, E x) pairs kept on the
 * device, plain field_dot; depth 0 disables.  flags: SBX_FLAG_EXACT for the
 * reference's evaluation order (bitwise), else FAST. */
sbx_status sbx_projection_reset(sbx_ctx* ctx, int depth);
sbx_status sbx_projection_size(sbx_ctx* ctx, int32_t* size);
/* guess = sum_i (x_i . b) x_i; deflated_rhs (may be NULL) = b - E guess */
sbx_status sbx_projection_guess(sbx_ctx* ctx, const double* b, double* guess,
                                double* deflated_rhs, uint32_t flags);
/* append a converged solution (A-orthonormalised; the oldest entry evicted) */
sbx_status sbx_projection_append(sbx_ctx* ctx, const double* x, uint32_t flags);

/* advect (operators.hpp:84-87, operators.cpp:412-431) with grad_velocity
 * (:300-325): out_d = bm (c . grad u_d), d = 0..2, in the reference's
 * evaluation order (bitwise; dr/dx formed at each GLL node from the element
 * corners as build_geometric_factors does).  Velocity-grid fields. */
sbx_status sbx_advect(sbx_ctx* ctx, const double* const u[3], const double* const c[3],
                      double* const out[3]);

/* Batched velocity solve (FlowSolver::solve_velocity_star, stepper.cpp:188-238):
 * count <= 3 right-hand sides b[d] with the SAME operator / preconditioner
 * (cfg: h1, h2, tolerance, max_iterations, precond), each with its own initial
 * guess in x[d] (the previous velocity) and its own convergence; results[d]
 * per component.  FAST: one graph -- every component's initial residual
 * b - A x0 computed in the graph, then K1 / K2 launched once per iteration for
 * all components (grid.y = component); per component the arithmetic of
 * sbx_pcg.  EXACT: the components one after the other.  history, when given,
 * holds count * history_capacity entries (component-major). */
sbx_status sbx_pcg_multi(sbx_ctx* ctx, int count, const double* const* b, double* const* x,
                         const sbx_pcg_config* cfg, sbx_pcg_result* results);

/* -------------------------------------------------------- multi-GPU ------ */
/* One process per GPU; elements of a structured box are partitioned by
 * partition_rcb (mesh.cpp:168-226).  Shared nodes on rank boundaries are
 * assembled from raw copy values exchanged over peer memory (CUDA IPC windows
 * written directly by the kernels over NVLink), summed on every rank in the
 * reference's canonical copy order (bitwise the single-process gs_sum).  CG
 * scalars are exchanged the same way and summed in rank order.
 *
 * Exchange plan (host only, no GPU needed; used by the tests): */
typedef struct sbx_dist_plan sbx_dist_plan;
sbx_status sbx_dist_plan_create(const sbx_box_desc* desc, const int32_t* rank_of, int nranks,
                                int rank, sbx_dist_plan** out);
void sbx_dist_plan_destroy(sbx_dist_plan* plan);
/* [local elements, local nodes, boundary groups, boundary copies, interface
 *  groups, interface copies, neighbours, receive total, send total] */
sbx_status sbx_dist_plan_sizes(const sbx_dist_plan* plan, int64_t sizes[9]);
/* 0 loc_elems (i64) | 1 b_off 2 b_idx 3 if_off 4 if_code 5 nbr (i32) | 6 send
 * counts (i64) | 7 send_idx (i32) | 8 recv_count 9 recv_base (i64) | 10 nbr27
 * (i32) | 11 inv_mult 12 mask (f64) | 13 if_gid (i64) */
sbx_status sbx_dist_plan_array(const sbx_dist_plan* plan, int which, void* out);

/* Distributed context: this rank's part of the box, device data + a peer
 * window.  Connect it with the windows of all ranks (blobs gathered by the
 * application, e.g. torch.distributed.all_gather_object) before any call.
 * Contract of the distributed FAST pcg: the right-hand side must be
 * continuous across ranks and masked (as every reference caller passes it:
 * gs_sum then * inv_mult * mask).  Each rank checks its own shared groups and
 * the pcg returns SBX_E_SHAPE on any rank's violation; copies that differ
 * ACROSS ranks are not detected (the fused p'Ap identity then gives a wrong
 * alpha).  An exchange timeout (SBX_E_COMM) leaves the context unusable. */
sbx_status sbx_ctx_create_box_dist(const sbx_box_desc* desc, const int32_t* rank_of,
                                   int nranks, int rank, int device, sbx_ctx** out);
/* size of one rank's window blob; this rank's blob */
size_t sbx_ctx_dist_blob_size(int nranks);
sbx_status sbx_ctx_dist_blob(sbx_ctx* ctx, uint8_t* blob);
/* blobs: nranks * sbx_ctx_dist_blob_size(nranks) bytes, rank order */
sbx_status sbx_ctx_dist_connect(sbx_ctx* ctx, const uint8_t* blobs);

/* local element ids (global numbering, ascending) of a context */
sbx_status sbx_ctx_local_elements(const sbx_ctx* ctx, int64_t* global_ids);

/* --------------------------------------------------------- instrumentation */
/* Per-kernel device time of the last sbx_pcg call in FAST mode, measured with
 * CUDA events on the launching stream when enabled (adds no sync inside the
 * solve).  names: "ax", "gs", "update"; returns total ms and launch count. */
sbx_status sbx_ctx_enable_timing(sbx_ctx* ctx, int enable);
sbx_status sbx_ctx_kernel_time(const sbx_ctx* ctx, const char* name, double* total_ms,
                               int64_t* launches);

/* Test hook (no reference counterpart): one launch of the fused solver's
 * element kernel K1 in its first-iteration form (p = u, no preconditioner),
 * so w = D^T G D u h1 + h2 bm u comes out of exactly the kernel -- and the
 * metric variant (on-the-fly trilinear on box contexts) -- that sbx_pcg
 * runs.  Single-process contexts only. */
sbx_status sbx_debug_cg_k1(sbx_ctx* ctx, const double* u, double* w, double h1, double h2);

#ifdef __cplusplus
}
#endif

#endif /* SBX_H */
