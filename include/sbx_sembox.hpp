// sbx_sembox.hpp -- header-only C++ adapter that plugs the B200 PCG hot path
// (include/sbx.h, libsbx.so) into the reference's own operator API
// ("sembox", /root/reference/proj/include/sembox).  A sembox maintainer adds
// this header, links libsbx.so, and swaps the CPU operators for device ones:
//
//   sbx_sembox::Device dev(gf, basis, map, &mask);               // upload once
//   sembox::pcg(dev.apply_fn(coeffs), b, dev.jacobi_fn(coeffs),   // krylov.hpp:38-40
//               dev.dot_fn(), cfg, x);                            // the reference loop
//   auto res = dev.pcg(b, x, cfg, coeffs);                        // or the fused solver
//
// Every wrapper names the reference entry point it replaces.  Errors come
// back as the reference's exception types (errors.hpp:10-41).
#pragma once

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sbx.h"
#include "sembox/errors.hpp"
#include "sembox/field.hpp"
#include "sembox/gather.hpp"
#include "sembox/krylov.hpp"
#include "sembox/mesh.hpp"
#include "sembox/operators.hpp"

namespace sbx_sembox {

inline void check(sbx_status st, int iteration = -1) {
  if (st == SBX_OK) return;
  const std::string msg = sbx_last_error();
  switch (st) {
    case SBX_E_CONFIG: throw sembox::ConfigError(msg);
    case SBX_E_SHAPE: throw sembox::ContractViolation(msg);
    case SBX_E_MESH: throw sembox::MeshError(msg);
    case SBX_E_BREAKDOWN:
    case SBX_E_NAN: throw sembox::SolverError(msg, iteration);
    default: throw std::runtime_error("sbx: " + msg);
  }
}

// Device-resident copy of everything HelmholtzOperator points at
// (operators.hpp:103-108).
class Device {
 public:
  Device(const sembox::GeometricFactors& gf, const sembox::SpectralBasis& basis,
         const sembox::GatherScatterMap& map, const sembox::Field* mask, int device = 0)
      : Device(nullptr, gf, basis, map, mask, device) {}

  // With the mesh the map was built on (build_gather_scatter requires a
  // structured box, gather.cpp:11-12): the context verifies on the device
  // that map, mask and geometry are the box lattice's / the corners'
  // trilinear metric and then runs the lattice gather-scatter and the
  // trilinear-metric fused kernels -- the same kernels as a context built by
  // sbx_ctx_create_box.
  Device(const sembox::HexMesh& mesh, const sembox::GeometricFactors& gf,
         const sembox::SpectralBasis& basis, const sembox::GatherScatterMap& map,
         const sembox::Field* mask, int device = 0)
      : Device(&mesh, gf, basis, map, mask, device) {}

 private:
  Device(const sembox::HexMesh* mesh, const sembox::GeometricFactors& gf,
         const sembox::SpectralBasis& basis, const sembox::GatherScatterMap& map,
         const sembox::Field* mask, int device) {
    sbx_problem_desc d{};
    d.elem_count = gf.elem_count;
    d.degree = basis.order;
    d.deriv = basis.deriv.data();
    const std::vector<double>* g[6] = {&gf.g1, &gf.g2, &gf.g3, &gf.g4, &gf.g5, &gf.g6};
    for (int q = 0; q < 6; ++q) d.g[q] = g[q]->data();
    d.bm = gf.bm.data();
    d.mask = mask ? mask->v.data() : nullptr;
    d.global_count = map.global_count;
    d.group_offsets = map.group_offsets.data();
    d.group_nodes = map.group_nodes.data();
    std::vector<double> corners;
    if (mesh && mesh->structured() && mesh->elem_count == gf.elem_count) {
      d.box[0] = mesh->ex;
      d.box[1] = mesh->ey;
      d.box[2] = mesh->ez;
      for (int q = 0; q < 3; ++q) d.periodic[q] = mesh->periodic[q] ? 1 : 0;
      corners.reserve((size_t)mesh->elem_count * 24);
      for (const auto& el : mesh->corners)
        for (const auto& p : el)
          for (double v : p) corners.push_back(v);
      d.corners = corners.data();
    }
    check(sbx_ctx_create(&d, device, &ctx_));
    n1d_ = basis.n();
    elems_ = gf.elem_count;
  }

 public:
  ~Device() { sbx_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  sbx_ctx* handle() const { return ctx_; }

  // axhelm (operators.hpp:59-60); exact = the reference's evaluation order
  void axhelm(const sembox::Field& u, const sembox::HelmholtzCoeffs& c, sembox::Field& out,
              bool exact = false) const {
    shape(u);
    if (!out.same_shape(u)) out = sembox::Field(u.tag, u.elem_count, u.n1d);
    fields(c);
    check(sbx_axhelm(ctx_, u.v.data(), out.v.data(), c.h1, c.h2, exact ? SBX_FLAG_EXACT : 0));
  }

  // gs_sum_inplace (gather.hpp:39), bitwise equal
  void gs_sum_inplace(sembox::Field& f) const {
    shape(f);
    check(sbx_gs_sum(ctx_, f.v.data()));
  }

  // HelmholtzOperator::apply (operators.hpp:110) as a sembox::ApplyFn
  sembox::ApplyFn apply_fn(sembox::HelmholtzCoeffs c, bool exact = true) const {
    return [this, c, exact](const sembox::Field& x, sembox::Field& y) {
      shape(x);
      if (!y.same_shape(x)) y = sembox::Field(x.tag, x.elem_count, x.n1d);
      fields(c);
      check(sbx_apply(ctx_, x.v.data(), y.v.data(), c.h1, c.h2, exact ? SBX_FLAG_EXACT : 0));
    };
  }

  // field_dot_weighted (field.hpp:60-62) as a sembox::DotFn
  sembox::DotFn dot_fn(bool exact = true) const {
    return [this, exact](const sembox::Field& a, const sembox::Field& b) {
      double r = 0.0;
      check(sbx_dot(ctx_, a.v.data(), b.v.data(), 1, exact ? SBX_FLAG_EXACT : 0, &r));
      return r;
    };
  }

  // Jacobi on HelmholtzOperator::assembled_diagonal (stepper.cpp:175-186)
  sembox::PrecondFn jacobi_fn(sembox::HelmholtzCoeffs c) const {
    auto diag = std::make_shared<sembox::Field>(sembox::GridTag::velocity, elems_, n1d_);
    fields(c);
    check(sbx_axhelm_diagonal(ctx_, c.h1, c.h2, 1, diag->v.data()));
    return [diag](const sembox::Field& r, sembox::Field& z) {
      if (!z.same_shape(r)) z = sembox::Field(r.tag, r.elem_count, r.n1d);
      for (std::size_t a = 0; a < r.v.size(); ++a) z.v[a] = r.v[a] / diag->v[a];
    };
  }

  // pcg (krylov.hpp:38-40) with HelmholtzOperator + Jacobi + weighted dot,
  // run entirely on the device (fast: fused kernels in a CUDA graph).
  sembox::PcgResult pcg(const sembox::Field& b, sembox::Field& x,
                        const sembox::KrylovConfig& kc, sembox::HelmholtzCoeffs c,
                        bool jacobi = true, bool fast = true) const {
    shape(b);
    if (!x.same_shape(b)) x = sembox::Field(b.tag, b.elem_count, b.n1d);
    sbx_pcg_config cfg;
    sbx_pcg_config_default(&cfg);
    cfg.tolerance = kc.tolerance;
    cfg.max_iterations = kc.max_iterations;
    cfg.precond = jacobi ? SBX_PRECOND_JACOBI : SBX_PRECOND_NONE;
    cfg.mode = fast ? SBX_MODE_FAST : SBX_MODE_EXACT;
    cfg.h1 = c.h1;
    cfg.h2 = c.h2;
    std::vector<double> hist(kc.max_iterations + 1);
    cfg.history = hist.data();
    cfg.history_capacity = (int64_t)hist.size();
    sbx_pcg_result r{};
    fields(c);
    check(sbx_pcg(ctx_, b.v.data(), x.v.data(), &cfg, &r), r.error_iteration);
    sembox::PcgResult out;
    out.iterations = r.iterations;
    out.rel_residual = r.rel_residual;
    out.rel_residual_precond = r.rel_residual_precond;
    out.converged = r.converged != 0;
    out.residual_history.assign(hist.begin(), hist.begin() + std::min<int64_t>(r.history_length,
                                                                               (int64_t)hist.size()));
    return out;
  }

 private:
  // HelmholtzCoeffs::h1_field / h2_field (operators.hpp:42-43) onto the
  // context (sbx_ctx_set_coeff_fields) whenever a call carries them (their values
  // may have changed) or the context still holds earlier ones
  void fields(const sembox::HelmholtzCoeffs& c) const {
    const double* f1 = c.h1_field ? c.h1_field->v.data() : nullptr;
    const double* f2 = c.h2_field ? c.h2_field->v.data() : nullptr;
    if (f1 == f1_ && f2 == f2_ && !f1 && !f2) return;
    check(sbx_ctx_set_coeff_fields(ctx_, f1, f2));
    f1_ = f1;
    f2_ = f2;
  }
  mutable const double* f1_ = nullptr;
  mutable const double* f2_ = nullptr;
  void shape(const sembox::Field& f) const {
    if (f.tag != sembox::GridTag::velocity || f.elem_count != elems_ || f.n1d != n1d_)
      throw sembox::ContractViolation("sbx: field grid/shape mismatch");
  }
  sbx_ctx* ctx_ = nullptr;
  int n1d_ = 0;
  int elems_ = 0;
};

}  // namespace sbx_sembox
