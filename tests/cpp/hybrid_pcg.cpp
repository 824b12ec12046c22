// Drop-in demonstration and parity check (needs a GPU at run time):
// the reference's OWN sembox::pcg loop (krylov.cpp:7-91) driving the B200
// operators through include/sbx_sembox.hpp, compared bit for bit with the
// all-CPU reference run, plus the fused device solver.
//
// Built by `make -C oracle hybrid` (links the reference objects in
// oracle/_ref and libsbx.so); run by tests/test_gpu_hybrid.py.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <random>
#include <string>

#include "sbx_sembox.hpp"
#include "sembox/basis.hpp"
#include "sembox/gather.hpp"
#include "sembox/krylov.hpp"
#include "sembox/mesh.hpp"
#include "sembox/operators.hpp"

using namespace sembox;

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// bench mode: Device::pcg (reference-built problem + mesh hint) against a
// context the product builds itself (sbx_ctx_create_box), same host vectors,
// 100 iterations per solve (tol 0), E^3 deformed box, N = 7.
static int bench(int ex) {
  HexMesh mesh = build_box_mesh(ex, ex, ex, {0, 0, 0}, {1, 1, 1}, {false, false, false});
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
  Field b(GridTag::velocity, mesh.elem_count, basis.n());
  std::mt19937_64 rng(77);
  std::uniform_real_distribution<double> dist(-1, 1);
  for (double& v : b.v) v = dist(rng);
  gs_sum_inplace(map, b);
  for (std::int64_t a = 0; a < b.size(); ++a) b.v[a] *= map.inv_mult[a] * mask.v[a];
  const HelmholtzCoeffs hc{1.0, 0.0, nullptr, nullptr};
  KrylovConfig cfg;
  cfg.tolerance = 0.0;
  cfg.max_iterations = 100;
  const double nodes = (double)b.size();
  double t0 = now();
  sbx_sembox::Device dev(mesh, gf, basis, map, &mask);
  const double t_dev = now() - t0;
  Field x(GridTag::velocity, mesh.elem_count, basis.n());
  auto time_dev = [&] {
    for (int w = 0; w < 2; ++w) dev.pcg(b, x, cfg, hc);
    const double t = now();
    for (int r = 0; r < 5; ++r) {
      std::fill(x.v.begin(), x.v.end(), 0.0);
      dev.pcg(b, x, cfg, hc);
    }
    return (now() - t) / 5;
  };
  const double s_dev = time_dev();
  // the product's own box context on the same mesh
  sbx_box_desc bd{};
  bd.ex = bd.ey = bd.ez = ex;
  bd.degree = 7;
  bd.lengths[0] = bd.lengths[1] = bd.lengths[2] = 1.0;
  bd.deform_amplitude = 0.05;
  sbx_ctx* box = nullptr;
  t0 = now();
  sbx_sembox::check(sbx_ctx_create_box(&bd, 0, &box));
  const double t_box = now() - t0;
  sbx_pcg_config pc;
  sbx_pcg_config_default(&pc);
  pc.tolerance = 0.0;
  pc.max_iterations = 100;
  sbx_pcg_result pr{};
  for (int w = 0; w < 2; ++w) sbx_sembox::check(sbx_pcg(box, b.v.data(), x.v.data(), &pc, &pr));
  t0 = now();
  for (int r = 0; r < 5; ++r) {
    std::fill(x.v.begin(), x.v.end(), 0.0);
    sbx_sembox::check(sbx_pcg(box, b.v.data(), x.v.data(), &pc, &pr));
  }
  const double s_box = (now() - t0) / 5;
  sbx_ctx_destroy(box);
  std::printf("{\"mesh\": %d, \"device_create_s\": %.3f, \"box_create_s\": %.3f, "
              "\"device_pcg_ms\": %.3f, \"box_pcg_ms\": %.3f, \"device_gdofs\": %.3f, "
              "\"box_gdofs\": %.3f, \"ratio\": %.4f}\n",
              ex, t_dev, t_box, s_dev * 1e3, s_box * 1e3, nodes * 100 / s_dev / 1e9,
              nodes * 100 / s_box / 1e9, s_box / s_dev);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[1]) == "bench") return bench(std::atoi(argv[2]));
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

  // 2./3. for both adapters: without the mesh (CSR gather-scatter, stored
  // geometry) and with it (verified lattice gather-scatter, trilinear K1)
  bool all_ok = true;
  for (int with_mesh = 0; with_mesh < 2; ++with_mesh) {
    std::unique_ptr<sbx_sembox::Device> devp(
        with_mesh ? new sbx_sembox::Device(mesh, gf, basis, map, &mask)
                  : new sbx_sembox::Device(gf, basis, map, &mask));
    const sbx_sembox::Device& dev = *devp;
    // 2. the reference pcg loop, operators on the B200 (exact evaluation order)
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
    const char* tag = with_mesh ? "Device(mesh, ...)" : "Device(...)";
    uint32_t feat = 0;
    sbx_sembox::check(sbx_ctx_features(dev.handle(), &feat));
    const uint32_t want = with_mesh ? (SBX_FEAT_LATTICE_GS | SBX_FEAT_BOX_K2 | SBX_FEAT_TRILINEAR)
                                    : 0u;
    std::printf("%s features 0x%x (want 0x%x)\n", tag, feat, want);
    all_ok = all_ok && feat == want;
    std::printf("cpu  : %d iterations, rel %.9e\n", r_cpu.iterations, r_cpu.rel_residual);
    std::printf("%s hybrid (sembox::pcg + B200 operators): %d iterations, rel %.9e, "
                "bitwise %s\n",
                tag, r_hyb.iterations, r_hyb.rel_residual, hyb_bitwise ? "yes" : "NO");
    std::printf("%s device (fused sbx_pcg): %d iterations, rel %.9e, |x-x_cpu|/|x_cpu| %.2e\n",
                tag, r_dev.iterations, r_dev.rel_residual, err);
    all_ok = all_ok && hyb_bitwise && dev_ok;
  }
  // 4. per-node coefficients (HelmholtzCoeffs::h1_field / h2_field): the
  // reference pcg, all-CPU vs B200 operators through the adapter, bitwise;
  // and the adapter's own solve (reference order on the device with fields)
  {
    Field h1f(GridTag::velocity, mesh.elem_count, basis.n());
    Field h2f(GridTag::velocity, mesh.elem_count, basis.n());
    std::uniform_real_distribution<double> d1(0.5, 2.0), d2(0.0, 3.0);
    for (double& v : h1f.v) v = d1(rng);
    for (double& v : h2f.v) v = d2(rng);
    const HelmholtzCoeffs hf{1.0, 1.0, &h1f, &h2f};
    HelmholtzOperator opf{&gf, &basis, &map, &mask, hf};
    const Field diagf = opf.assembled_diagonal();
    Field xc(GridTag::velocity, mesh.elem_count, basis.n());
    const PcgResult rc = pcg([&](const Field& x, Field& y) { opf.apply(x, y); }, b,
                             [&](const Field& r, Field& z) {
                               z = r;
                               for (std::size_t a = 0; a < r.v.size(); ++a)
                                 z.v[a] = r.v[a] / diagf.v[a];
                             },
                             [&](const Field& u, const Field& v) {
                               return field_dot_weighted(u, v, map.inv_mult);
                             },
                             cfg, xc);
    sbx_sembox::Device dev(mesh, gf, basis, map, &mask);
    Field xh(GridTag::velocity, mesh.elem_count, basis.n());
    const PcgResult rh =
        pcg(dev.apply_fn(hf, true), b, dev.jacobi_fn(hf), dev.dot_fn(true), cfg, xh);
    Field xd(GridTag::velocity, mesh.elem_count, basis.n());
    const PcgResult rd = dev.pcg(b, xd, cfg, hf, true, true);
    const bool ok_h = rh.iterations == rc.iterations &&
                      rh.residual_history == rc.residual_history && xh.v == xc.v;
    const bool ok_d = rd.iterations == rc.iterations &&
                      rd.residual_history == rc.residual_history && xd.v == xc.v;
    std::printf("fields: cpu %d iterations; hybrid bitwise %s; device solve bitwise %s\n",
                rc.iterations, ok_h ? "yes" : "NO", ok_d ? "yes" : "NO");
    all_ok = all_ok && ok_h && ok_d;
  }
  std::printf("%s\n", all_ok ? "HYBRID PASS" : "HYBRID FAIL");
  return all_ok ? 0 : 1;
}
