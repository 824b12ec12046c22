// Drop-in demonstration and parity check (needs a GPU at run time):
// the reference's OWN sembox::pcg loop (krylov.cpp:7-91) driving the B200
// operators through include/sbx_sembox.hpp, compared bit for bit with the
// all-CPU reference run, plus the fused device solver.
//
// Built by `make -C oracle hybrid` (links the reference objects in
// oracle/_ref and libsbx.so); run by tests/test_gpu_hybrid.py.
#include <cmath>
#include <cstdio>
#include <random>

#include "sbx_sembox.hpp"
#include "sembox/basis.hpp"
#include "sembox/gather.hpp"
#include "sembox/krylov.hpp"
#include "sembox/mesh.hpp"
#include "sembox/operators.hpp"

using namespace sembox;

int main() {
  // C1: 8^3 deformed box, N = 7, Poisson, Jacobi, seed-77 continuous rhs
  HexMesh mesh = build_box_mesh(8, 8, 8, {0, 0, 0}, {1, 1, 1}, {false, false, false});
  for (auto& cs : mesh.corners)
    for (auto& p : cs) {
      const double s = std::sin(M_PI * p[0]) * std::sin(M_PI * p[1]) * std::sin(M_PI * p[2]);
      const double d0 = 0.05 * s * 1.0, d1 = 0.05 * s * 0.5, d2 = 0.05 * s * 0.25;
      p[0] += d0;
      p[1] += d1;
      p[2] += d2;
    }
  const SpectralBasis basis = build_gll_basis(7);
  const GeometricFactors gf = build_geometric_factors(mesh, basis, false);
  const GatherScatterMap map = build_gather_scatter(mesh, 7);
  const Field mask = build_dirichlet_mask(mesh, 7);
  HelmholtzOperator op{&gf, &basis, &map, &mask, {1.0, 0.0, nullptr, nullptr}};
  Field b(GridTag::velocity, mesh.elem_count, basis.n());
  std::mt19937_64 rng(77);
  std::uniform_real_distribution<double> dist(-1, 1);
  for (double& v : b.v) v = dist(rng);
  gs_sum_inplace(map, b);
  for (std::int64_t a = 0; a < b.size(); ++a) b.v[a] *= map.inv_mult[a] * mask.v[a];
  const Field diag = op.assembled_diagonal();
  KrylovConfig cfg;
  cfg.tolerance = 1e-8;
  cfg.max_iterations = 2000;

  // 1. all-CPU reference
  Field x_cpu(GridTag::velocity, mesh.elem_count, basis.n());
  const PcgResult r_cpu = pcg([&](const Field& x, Field& y) { op.apply(x, y); }, b,
                              [&](const Field& r, Field& z) {
                                z = r;
                                for (std::size_t a = 0; a < r.v.size(); ++a)
                                  z.v[a] = r.v[a] / diag.v[a];
                              },
                              [&](const Field& u, const Field& v) {
                                return field_dot_weighted(u, v, map.inv_mult);
                              },
                              cfg, x_cpu);

  // 2. the reference pcg loop, operators on the B200 (exact evaluation order)
  sbx_sembox::Device dev(gf, basis, map, &mask);
  const HelmholtzCoeffs hc{1.0, 0.0, nullptr, nullptr};
  Field x_hyb(GridTag::velocity, mesh.elem_count, basis.n());
  const PcgResult r_hyb =
      pcg(dev.apply_fn(hc, true), b, dev.jacobi_fn(hc), dev.dot_fn(true), cfg, x_hyb);

  // 3. the fused device solver
  Field x_dev(GridTag::velocity, mesh.elem_count, basis.n());
  const PcgResult r_dev = dev.pcg(b, x_dev, cfg, hc, true, true);

  const bool hyb_bitwise = r_hyb.iterations == r_cpu.iterations &&
                           r_hyb.residual_history == r_cpu.residual_history &&
                           x_hyb.v == x_cpu.v;
  double num = 0, den = 0;
  for (std::size_t a = 0; a < x_cpu.v.size(); ++a) {
    num += (x_dev.v[a] - x_cpu.v[a]) * (x_dev.v[a] - x_cpu.v[a]);
    den += x_cpu.v[a] * x_cpu.v[a];
  }
  const double err = std::sqrt(num / den);
  const bool dev_ok = r_dev.iterations == r_cpu.iterations && err <= 1e-10;
  std::printf("cpu  : %d iterations, rel %.9e\n", r_cpu.iterations, r_cpu.rel_residual);
  std::printf("hybrid (sembox::pcg + B200 operators): %d iterations, rel %.9e, bitwise %s\n",
              r_hyb.iterations, r_hyb.rel_residual, hyb_bitwise ? "yes" : "NO");
  std::printf("device (fused sbx_pcg): %d iterations, rel %.9e, |x-x_cpu|/|x_cpu| %.2e\n",
              r_dev.iterations, r_dev.rel_residual, err);
  std::printf("%s\n", hyb_bitwise && dev_ok ? "HYBRID PASS" : "HYBRID FAIL");
  return hyb_bitwise && dev_ok ? 0 : 1;
}
