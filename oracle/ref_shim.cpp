// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
//
// C-ABI shim over the UNMODIFIED reference implementation ("sembox", compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the Python test-suite, the golden-vector generator and bench.py's CPU
// baseline leg call the reference's own hot-path code:
//   build_box_mesh        proj/src/mesh.cpp:21-75
//   build_gll_basis       proj/src/basis.cpp:60-95
//   build_geometric_factors proj/src/operators.cpp:123-178
//   build_gather_scatter  proj/src/gather.cpp:10-83
//   build_dirichlet_mask  proj/src/operators.cpp:433-455
//   axhelm                proj/src/operators.cpp:215-263
//   axhelm_diagonal       proj/src/operators.cpp:272-298
//   gs_sum_inplace        proj/src/gather.cpp:85-98
//   HelmholtzOperator     proj/src/operators.cpp:530-540
//   field_dot_weighted    proj/src/field.cpp:69-81
//   pcg                   proj/src/krylov.cpp:7-91
//   partition_rcb         proj/src/mesh.cpp:168-226
//   oracle::dense_helmholtz_element proj/src/oracle.cpp:78-125
//
// Exceptions are mapped to integer status codes (same numbering as the
// product's include/sbx.h) with the message kept in ref_last_error().
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>

#include <algorithm>
#include <memory>

#include "sembox/basis.hpp"
#include "sembox/errors.hpp"
#include "sembox/field.hpp"
#include "sembox/gather.hpp"
#include "sembox/krylov.hpp"
#include "sembox/mesh.hpp"
#include "sembox/operators.hpp"
#include "sembox/oracle.hpp"
#include "sembox/parallel.hpp"

using namespace sembox;

namespace {

thread_local std::string g_err;

enum {
  OK = 0,
  E_CONFIG = 2,
  E_SHAPE = 3,
  E_MESH = 4,
  E_BREAKDOWN = 5,
  E_NAN = 6,
  E_OTHER = 99,
};

struct Problem {
  HexMesh mesh;
  SpectralBasis basis;
  GeometricFactors gf;
  GatherScatterMap map;
  Field mask;
  // benchmark session (ref_bench_prepare / ref_bench_solve): rhs, solution
  // and Jacobi diagonal kept here so a timed step is the pcg call itself
  Field bench_b, bench_x, bench_diag;
  double bench_h1 = 0.0, bench_h2 = 0.0;
  // consistent-Poisson pressure path (ref_pressure_setup)
  bool has_p = false;
  std::unique_ptr<ProjectionHistory> proj;
  PressureBasis pb;
  PressureGeometry pg;
  Field inv_bdiag, pdiag;
  // per-node Helmholtz coefficients (HelmholtzCoeffs::h1_field / h2_field,
  // operators.hpp:42-43), applied by every operator below when set
  Field h1f, h2f;
  bool has_h1f = false, has_h2f = false;
};

HelmholtzCoeffs coeffs_of(const Problem& p, double h1, double h2) {
  return {h1, h2, p.has_h1f ? &p.h1f : nullptr, p.has_h2f ? &p.h2f : nullptr};
}

// FlowSolver::apply_pressure_operator (stepper.cpp:240-248), restated with the
// reference's own operators (stepper.cpp itself cannot be linked: it needs
// schwarz.cpp / Eigen3).
void pressure_apply(const Problem& p, const Field& x, Field& out) {
  VectorField g = gradient_from_pressure(x, p.pg, p.basis, p.pb);
  for (int d = 0; d < 3; ++d) {
    gs_sum_inplace(p.map, g[d]);
    field_pointwise_mul(p.inv_bdiag, g[d]);
  }
  out = divergence_to_pressure(g[0], g[1], g[2], p.pg, p.basis, p.pb);
}

// FlowSolver::pressure_operator_diagonal (stepper.cpp:250-275), restated.
Field pressure_diagonal(const Problem& p) {
  const int m = p.pb.m(), n = p.basis.n();
  const int mm = m * m * m, nn = n * n * n;
  Field diag(GridTag::pressure, p.mesh.elem_count, m);
  parallel_for(p.mesh.elem_count, [&](std::int64_t e) {
    PressureGeometry pge;
    pge.elem_count = 1;
    pge.m1d = m;
    pge.wdetj.assign(p.pg.wdetj.begin() + e * mm, p.pg.wdetj.begin() + (e + 1) * mm);
    pge.drdx.assign(p.pg.drdx.begin() + e * mm * 9, p.pg.drdx.begin() + (e + 1) * mm * 9);
    Field unit(GridTag::pressure, 1, m);
    for (int q = 0; q < mm; ++q) {
      std::fill(unit.v.begin(), unit.v.end(), 0.0);
      unit.v[q] = 1.0;
      const VectorField g = gradient_from_pressure(unit, pge, p.basis, p.pb);
      double s = 0.0;
      for (int d = 0; d < 3; ++d)
        for (int a = 0; a < nn; ++a) {
          const double v = g[d].v[a];
          s += v * v * p.inv_bdiag.v[e * nn + a];
        }
      diag.v[e * mm + q] = s;
    }
  });
  return diag;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return E_CONFIG;
  } catch (const ContractViolation& e) {
    g_err = e.what();
    return E_SHAPE;
  } catch (const MeshError& e) {
    g_err = e.what();
    return E_MESH;
  } catch (const SolverError& e) {
    g_err = e.what();
    return std::string(e.what()).find("breakdown") != std::string::npos ? E_BREAKDOWN
                                                                         : E_NAN;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_OTHER;
  }
}

Field wrap(const Problem& p, const double* v) {
  Field f(GridTag::velocity, p.mesh.elem_count, p.basis.n());
  std::memcpy(f.v.data(), v, f.v.size() * sizeof(double));
  return f;
}

void unwrap(const Field& f, double* out) {
  std::memcpy(out, f.v.data(), f.v.size() * sizeof(double));
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_workers(int n) { set_worker_count(n); }
int ref_workers() { return worker_count(); }

// corners: optional [E][8][3] override (deformed meshes); null keeps the box.
int ref_problem_create(int ex, int ey, int ez, const double* origin, const double* lengths,
                       const int* periodic, int degree, const double* corners,
                       int with_gradients, void** out) {
  *out = nullptr;
  return guarded([&] {
    auto* p = new Problem;
    try {
      p->mesh = build_box_mesh(ex, ey, ez, {origin[0], origin[1], origin[2]},
                               {lengths[0], lengths[1], lengths[2]},
                               {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0});
      if (corners)
        for (int e = 0; e < p->mesh.elem_count; ++e)
          for (int c = 0; c < 8; ++c)
            for (int d = 0; d < 3; ++d)
              p->mesh.corners[e][c][d] = corners[(static_cast<std::int64_t>(e) * 8 + c) * 3 + d];
      p->basis = build_gll_basis(degree);
      p->gf = build_geometric_factors(p->mesh, p->basis, with_gradients != 0);
      p->map = build_gather_scatter(p->mesh, degree);
      p->mask = build_dirichlet_mask(p->mesh, degree);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

void ref_problem_destroy(void* h) { delete static_cast<Problem*>(h); }

void ref_problem_sizes(void* h, std::int64_t* sizes) {
  auto* p = static_cast<Problem*>(h);
  sizes[0] = p->mesh.elem_count;
  sizes[1] = p->basis.n();
  sizes[2] = p->map.node_count();
  sizes[3] = p->map.global_count;
}

// which: 0 nodes, 1 weights, 2 deriv, 3..8 g1..g6, 9 bm, 10 jac, 11 mask,
// 12 inv_mult, 13 corners
void ref_copy_double(void* h, int which, double* out) {
  auto* p = static_cast<Problem*>(h);
  const std::vector<double>* src = nullptr;
  switch (which) {
    case 0: src = &p->basis.nodes; break;
    case 1: src = &p->basis.weights; break;
    case 2: src = &p->basis.deriv; break;
    case 3: src = &p->gf.g1; break;
    case 4: src = &p->gf.g2; break;
    case 5: src = &p->gf.g3; break;
    case 6: src = &p->gf.g4; break;
    case 7: src = &p->gf.g5; break;
    case 8: src = &p->gf.g6; break;
    case 9: src = &p->gf.bm; break;
    case 10: src = &p->gf.jac; break;
    case 11: src = &p->mask.v; break;
    case 12: src = &p->map.inv_mult; break;
    case 13: {
      for (int e = 0; e < p->mesh.elem_count; ++e)
        for (int c = 0; c < 8; ++c)
          for (int d = 0; d < 3; ++d)
            out[(static_cast<std::int64_t>(e) * 8 + c) * 3 + d] = p->mesh.corners[e][c][d];
      return;
    }
    default: return;
  }
  std::memcpy(out, src->data(), src->size() * sizeof(double));
}

// which: 0 gid (compressed), 1 group_offsets, 2 group_nodes
void ref_copy_int64(void* h, int which, std::int64_t* out) {
  auto* p = static_cast<Problem*>(h);
  const std::vector<std::int64_t>* src =
      which == 0 ? &p->map.gid : which == 1 ? &p->map.group_offsets : &p->map.group_nodes;
  std::memcpy(out, src->data(), src->size() * sizeof(std::int64_t));
}

void ref_copy_mult(void* h, std::int32_t* out) {
  auto* p = static_cast<Problem*>(h);
  std::memcpy(out, p->map.mult.data(), p->map.mult.size() * sizeof(std::int32_t));
}

// h1f / h2f: E*n^3 per-node coefficients, or NULL for the scalar
void ref_set_coeff_fields(void* h, const double* h1f, const double* h2f) {
  auto* p = static_cast<Problem*>(h);
  p->has_h1f = h1f != nullptr;
  p->has_h2f = h2f != nullptr;
  if (h1f) p->h1f = wrap(*p, h1f);
  if (h2f) p->h2f = wrap(*p, h2f);
}

int ref_axhelm(void* h, const double* u, double h1, double h2, int flip, double* out) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    debug::axhelm_sign_flip.store(flip != 0);
    Field uf = wrap(*p, u), of;
    HelmholtzCoeffs hc = coeffs_of(*p, h1, h2);
    try {
      axhelm(uf, hc, p->gf, p->basis, of);
    } catch (...) {
      debug::axhelm_sign_flip.store(false);
      throw;
    }
    debug::axhelm_sign_flip.store(false);
    unwrap(of, out);
  });
}

int ref_axhelm_diagonal(void* h, double h1, double h2, int assembled, double* out) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    HelmholtzOperator op{&p->gf, &p->basis, &p->map, &p->mask, coeffs_of(*p, h1, h2)};
    const Field d = assembled ? op.assembled_diagonal()
                              : axhelm_diagonal(op.coeffs, p->gf, p->basis);
    unwrap(d, out);
  });
}

int ref_gs_sum(void* h, double* field) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    Field f = wrap(*p, field);
    gs_sum_inplace(p->map, f);
    unwrap(f, field);
  });
}

int ref_apply(void* h, double h1, double h2, int use_mask, const double* x, double* out) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    HelmholtzOperator op{&p->gf, &p->basis, &p->map, use_mask ? &p->mask : nullptr,
                         coeffs_of(*p, h1, h2)};
    Field xf = wrap(*p, x), of(GridTag::velocity, p->mesh.elem_count, p->basis.n());
    op.apply(xf, of);
    unwrap(of, out);
  });
}

double ref_dot_weighted(void* h, const double* a, const double* b) {
  auto* p = static_cast<Problem*>(h);
  return field_dot_weighted(wrap(*p, a), wrap(*p, b), p->map.inv_mult);
}

// Jacobi-preconditioned (precond=1) or unpreconditioned (0) PCG on the
// assembled, masked Helmholtz operator with the multiplicity-weighted dot --
// the configuration of acceptance.cpp:89-103, test_schwarz.cpp:159-185 and
// stepper.cpp:175-226.  info: [iterations, converged, error_iteration];
// res: [rel_residual, rel_residual_precond]; history capacity hist_cap.
int ref_pcg(void* h, double h1, double h2, int precond, const double* b, double* x,
            double tol, int max_iterations, std::int64_t* info, double* res,
            double* history, std::int64_t hist_cap, std::int64_t* hist_len) {
  auto* p = static_cast<Problem*>(h);
  info[0] = 0;
  info[1] = 0;
  info[2] = -1;
  *hist_len = 0;
  return guarded([&] {
    HelmholtzOperator op{&p->gf, &p->basis, &p->map, &p->mask, coeffs_of(*p, h1, h2)};
    const Field diag = op.assembled_diagonal();
    const DotFn dot = [&](const Field& a, const Field& bb) {
      return field_dot_weighted(a, bb, p->map.inv_mult);
    };
    PrecondFn pre = nullptr;
    if (precond == 1)
      pre = [&](const Field& r, Field& z) {
        if (!z.same_shape(r)) z = Field(r.tag, r.elem_count, r.n1d);
        parallel_for_ranges(r.size(), [&](std::int64_t lo, std::int64_t hi) {
          for (std::int64_t a = lo; a < hi; ++a) z.v[a] = r.v[a] / diag.v[a];
        });
      };
    KrylovConfig cfg;
    cfg.tolerance = tol;
    cfg.max_iterations = max_iterations;
    Field bf = wrap(*p, b), xf = wrap(*p, x);
    try {
      const PcgResult r = pcg([&](const Field& in, Field& o) { op.apply(in, o); }, bf, pre,
                              dot, cfg, xf);
      info[0] = r.iterations;
      info[1] = r.converged ? 1 : 0;
      res[0] = r.rel_residual;
      res[1] = r.rel_residual_precond;
      const std::int64_t n =
          std::min<std::int64_t>(hist_cap, static_cast<std::int64_t>(r.residual_history.size()));
      for (std::int64_t i = 0; i < n; ++i) history[i] = r.residual_history[i];
      *hist_len = static_cast<std::int64_t>(r.residual_history.size());
    } catch (const SolverError& e) {
      info[2] = e.iteration;
      throw;
    }
    unwrap(xf, x);
  });
}

// Benchmark session, setup part (untimed): the operator's assembled
// diagonal (HelmholtzOperator::assembled_diagonal, operators.cpp:536-540) and
// the right-hand side.
int ref_bench_prepare(void* h, double h1, double h2, const double* b) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    HelmholtzOperator op{&p->gf, &p->basis, &p->map, &p->mask, coeffs_of(*p, h1, h2)};
    p->bench_diag = op.assembled_diagonal();
    p->bench_b = wrap(*p, b);
    p->bench_x = Field(GridTag::velocity, p->mesh.elem_count, p->basis.n());
    p->bench_h1 = h1;
    p->bench_h2 = h2;
  });
}

// Benchmark session, timed part: x = 0 (parallel fill, as the GPU arm zeroes
// its x on the device), then the reference's own pcg (krylov.cpp:7-91) with
// HelmholtzOperator::apply, the parallel Jacobi lambda of stepper.cpp:180-185
// and field_dot_weighted, for exactly `iters` iterations (tolerance 0).
int ref_bench_solve(void* h, int iters, std::int64_t* info, double* res) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    HelmholtzOperator op{&p->gf, &p->basis, &p->map, &p->mask,
                         {p->bench_h1, p->bench_h2, nullptr, nullptr}};
    const Field& diag = p->bench_diag;
    const DotFn dot = [&](const Field& a, const Field& bb) {
      return field_dot_weighted(a, bb, p->map.inv_mult);
    };
    const PrecondFn pre = [&](const Field& r, Field& z) {
      if (!z.same_shape(r)) z = Field(r.tag, r.elem_count, r.n1d);
      parallel_for_ranges(r.size(), [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t a = lo; a < hi; ++a) z.v[a] = r.v[a] / diag.v[a];
      });
    };
    Field& x = p->bench_x;
    parallel_for_ranges(x.size(), [&](std::int64_t lo, std::int64_t hi) {
      for (std::int64_t a = lo; a < hi; ++a) x.v[a] = 0.0;
    });
    KrylovConfig cfg;
    cfg.tolerance = 0.0;
    cfg.max_iterations = iters;
    const PcgResult r =
        pcg([&](const Field& in, Field& o) { op.apply(in, o); }, p->bench_b, pre, dot, cfg, x);
    info[0] = r.iterations;
    info[1] = r.converged ? 1 : 0;
    res[0] = r.rel_residual;
    res[1] = r.rel_residual_precond;
  });
}

// ---- consistent-Poisson pressure path ----------------
// Setup as FlowSolver's constructor does it (stepper.cpp:59-84, 110-111):
// the GL pressure basis and geometry, the inverse assembled (masked) mass.
int ref_pressure_setup(void* h) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    p->pb = build_pressure_basis(p->basis.order);
    p->pg = build_pressure_geometry(p->mesh, p->pb);
    Field bdiag(GridTag::velocity, p->mesh.elem_count, p->basis.n());
    std::copy(p->gf.bm.begin(), p->gf.bm.end(), bdiag.v.begin());
    gs_sum_inplace(p->map, bdiag);
    p->inv_bdiag = Field(GridTag::velocity, p->mesh.elem_count, p->basis.n());
    for (std::int64_t a = 0; a < bdiag.size(); ++a)
      p->inv_bdiag.v[a] = p->mask.v[a] / bdiag.v[a];
    p->pdiag = pressure_diagonal(*p);
    p->has_p = true;
  });
}

// which: 0 GL nodes [m], 1 GL weights [m], 2 interp_v2p [m*n], 3 wdetj
// [E m^3], 4 drdx [E m^3 9], 5 inv_bdiag [E n^3], 6 the Jacobi diagonal [E m^3]
void ref_pressure_copy(void* h, int which, double* out) {
  auto* p = static_cast<Problem*>(h);
  const std::vector<double>* src = which == 0   ? &p->pb.nodes
                                   : which == 1 ? &p->pb.weights
                                   : which == 2 ? &p->pb.interp_v2p
                                   : which == 3 ? &p->pg.wdetj
                                   : which == 4 ? &p->pg.drdx
                                   : which == 5 ? &p->inv_bdiag.v
                                                : &p->pdiag.v;
  std::memcpy(out, src->data(), src->size() * sizeof(double));
}

int ref_gradient_from_pressure(void* h, const double* pin, double* gx, double* gy,
                               double* gz) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    Field f(GridTag::pressure, p->mesh.elem_count, p->pb.m());
    std::memcpy(f.v.data(), pin, f.v.size() * sizeof(double));
    const VectorField g = gradient_from_pressure(f, p->pg, p->basis, p->pb);
    unwrap(g[0], gx);
    unwrap(g[1], gy);
    unwrap(g[2], gz);
  });
}

int ref_divergence_to_pressure(void* h, const double* ux, const double* uy, const double* uz,
                               double* out) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    const Field d = divergence_to_pressure(wrap(*p, ux), wrap(*p, uy), wrap(*p, uz), p->pg,
                                           p->basis, p->pb);
    unwrap(d, out);
  });
}

int ref_pressure_apply(void* h, const double* x, double* out) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    Field f(GridTag::pressure, p->mesh.elem_count, p->pb.m()), o;
    std::memcpy(f.v.data(), x, f.v.size() * sizeof(double));
    pressure_apply(*p, f, o);
    unwrap(o, out);
  });
}

// The pressure solve of FlowSolver::solve_pressure_update (stepper.cpp:310-348)
// on a given (already deflated) right-hand side and initial guess: the
// reference pcg with apply_pressure_operator, the preconditioner of
// pressure_precond (stepper.cpp:277-308: Jacobi on pressure_operator_diagonal
// or none, each followed by the mean deflation) and the plain field_dot.
int ref_pressure_pcg(void* h, int precond, const double* b, double* x, double tol,
                     int max_iterations, std::int64_t* info, double* res, double* history,
                     std::int64_t hist_cap, std::int64_t* hist_len) {
  auto* p = static_cast<Problem*>(h);
  info[0] = 0;
  info[1] = 0;
  info[2] = -1;
  *hist_len = 0;
  return guarded([&] {
    const int m = p->pb.m();
    const auto deflate = [](Field& z) {
      double mean = 0.0;
      for (double v : z.v) mean += v;
      mean /= static_cast<double>(z.size());
      for (double& v : z.v) v -= mean;
    };
    PrecondFn pre;
    if (precond == 1) {
      const Field* diag = &p->pdiag;
      pre = [diag, deflate](const Field& r, Field& z) {
        if (!z.same_shape(r)) z = Field(r.tag, r.elem_count, r.n1d);
        for (std::int64_t a = 0; a < r.size(); ++a) z.v[a] = r.v[a] / diag->v[a];
        deflate(z);
      };
    } else {
      pre = [deflate](const Field& r, Field& z) {
        field_copy(r, z);
        deflate(z);
      };
    }
    const ApplyFn apply_e = [p](const Field& in, Field& out) { pressure_apply(*p, in, out); };
    KrylovConfig cfg;
    cfg.tolerance = tol;
    cfg.max_iterations = max_iterations;
    Field bf(GridTag::pressure, p->mesh.elem_count, m), xf(GridTag::pressure,
                                                          p->mesh.elem_count, m);
    std::memcpy(bf.v.data(), b, bf.v.size() * sizeof(double));
    std::memcpy(xf.v.data(), x, xf.v.size() * sizeof(double));
    try {
      const PcgResult r = pcg(apply_e, bf, pre, field_dot, cfg, xf);
      info[0] = r.iterations;
      info[1] = r.converged ? 1 : 0;
      res[0] = r.rel_residual;
      res[1] = r.rel_residual_precond;
      const std::int64_t n =
          std::min<std::int64_t>(hist_cap, static_cast<std::int64_t>(r.residual_history.size()));
      for (std::int64_t i = 0; i < n; ++i) history[i] = r.residual_history[i];
      *hist_len = static_cast<std::int64_t>(r.residual_history.size());
    } catch (const SolverError& e) {
      info[2] = e.iteration;
      throw;
    }
    unwrap(xf, x);
  });
}

// ProjectionHistory of the pressure solve (krylov.cpp:93-124) with the
// pressure operator and field_dot, as solve_pressure_update uses it
// (stepper.cpp:326, 345).
void ref_projection_reset(void* h, int depth) {
  static_cast<Problem*>(h)->proj.reset(new ProjectionHistory(depth));
}
int ref_projection_size(void* h) { return static_cast<Problem*>(h)->proj->size(); }
int ref_projection_guess(void* h, const double* b, double* guess, double* deflated) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    const int m = p->pb.m();
    Field bf(GridTag::pressure, p->mesh.elem_count, m), dfl;
    std::memcpy(bf.v.data(), b, bf.v.size() * sizeof(double));
    const Field g = p->proj->project_guess(bf, field_dot, deflated ? &dfl : nullptr);
    unwrap(g, guess);
    if (deflated) unwrap(dfl, deflated);
  });
}
int ref_projection_append(void* h, const double* x) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    Field xf(GridTag::pressure, p->mesh.elem_count, p->pb.m());
    std::memcpy(xf.v.data(), x, xf.v.size() * sizeof(double));
    p->proj->append(xf, [p](const Field& in, Field& out) { pressure_apply(*p, in, out); },
                    field_dot);
  });
}

// advect (operators.cpp:412-431); the problem must be built with gradients
int ref_advect(void* h, const double* u0, const double* u1, const double* u2, const double* c0,
               const double* c1, const double* c2, double* o0, double* o1, double* o2) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    const VectorField u{wrap(*p, u0), wrap(*p, u1), wrap(*p, u2)};
    const VectorField c{wrap(*p, c0), wrap(*p, c1), wrap(*p, c2)};
    const VectorField o = advect(u, c, p->gf, p->basis);
    unwrap(o[0], o0);
    unwrap(o[1], o1);
    unwrap(o[2], o2);
  });
}

int ref_partition_rcb(void* h, int ranks, std::int32_t* rank_of) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    const Partition part = partition_rcb(p->mesh, ranks);
    for (int e = 0; e < p->mesh.elem_count; ++e) rank_of[e] = part.rank_of[e];
  });
}

int ref_dense_helmholtz_element(void* h, int elem, double h1, double h2, double* out) {
  auto* p = static_cast<Problem*>(h);
  return guarded([&] {
    const auto a = oracle::dense_helmholtz_element(p->mesh, elem, p->basis, h1, h2);
    std::memcpy(out, a.data(), a.size() * sizeof(double));
  });
}

void ref_trilinear_point(void* h, int elem, double r, double s, double t, double* x) {
  auto* p = static_cast<Problem*>(h);
  const auto v = oracle::trilinear_point(p->mesh, elem, r, s, t);
  x[0] = v[0];
  x[1] = v[1];
  x[2] = v[2];
}

} // extern "C"

extern "C" {
// std::mt19937_64 + std::uniform_real_distribution<double>(a, b), the random
// fields of the reference's tests (test_schwarz.cpp:30-38, bench.cpp:86-90).
void ref_fill_uniform(std::uint64_t seed, std::int64_t n, double a, double b, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(a, b);
  for (std::int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}
}
