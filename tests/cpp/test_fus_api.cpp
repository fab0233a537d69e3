// C++ drop-in check: the reference's own test cases (tests/test_*.cpp, tests/acceptance.cpp),
// written against the `namespace fus` API exactly as a reference user would, linked against
// libfus.so -> libfusg.so.  `test_fus_api host` runs the host-arithmetic cases (no GPU);
// `test_fus_api all` adds the device cases.
#include <Eigen/Dense>
#include <cuda_runtime.h>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

#include "fus/cascade.hpp"
#include "fus/grid.hpp"
#include "fus/medium.hpp"
#include "fus/potential.hpp"
#include "fus/transducer.hpp"
#include "fus/vie.hpp"
#include "fus/io.hpp"
#include "fus/analysis.hpp"
#include <fstream>
#include <map>

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                           \
  do {                                                                        \
    if (cond) {                                                               \
      ++g_pass;                                                               \
    } else {                                                                  \
      ++g_fail;                                                               \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);             \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                              \
  do {                                                                        \
    bool caught_ = false;                                                     \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const T&) {                                                      \
      caught_ = true;                                                         \
    }                                                                         \
    CHECK(caught_);                                                           \
  } while (0)

namespace {

const fus::Medium kWater = fus::medium_preset("water");

Eigen::VectorXcd random_vector(std::size_t n, unsigned seed) {  // tests/test_potential.cpp:14-20
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  Eigen::VectorXcd v(static_cast<Eigen::Index>(n));
  for (auto& x : v) {
    const double re = u(rng);
    const double im = u(rng);
    x = {re, im};
  }
  return v;
}

double max_abs(const Eigen::VectorXcd& v) { return v.cwiseAbs().maxCoeff(); }

// direct quadrature (the reference's direct_potential_oracle, src/potential.cpp:203-238)
Eigen::VectorXcd direct(const fus::Wavenumber& k, const fus::VoxelGrid& g, const Eigen::VectorXcd& f) {
  const double vol = g.dx * g.dx * g.dx;
  const std::complex<double> self = fus::self_weight(k, g.dx);
  Eigen::VectorXcd out(static_cast<Eigen::Index>(g.count()));
  for (int iz = 0; iz < g.dims.z(); ++iz)
    for (int iy = 0; iy < g.dims.y(); ++iy)
      for (int ix = 0; ix < g.dims.x(); ++ix) {
        std::complex<double> acc = 0.0;
        for (int jz = 0; jz < g.dims.z(); ++jz)
          for (int jy = 0; jy < g.dims.y(); ++jy)
            for (int jx = 0; jx < g.dims.x(); ++jx) {
              const std::complex<double> fj = f[g.index(jx, jy, jz)];
              if (ix == jx && iy == jy && iz == jz) {
                acc += self * fj;
              } else {
                acc += vol * fus::green_function(g.center(ix, iy, iz), g.center(jx, jy, jz), k) * fj;
              }
            }
        out[g.index(ix, iy, iz)] = acc;
      }
  return out;
}

void host_cases() {
  // tests/test_grid.cpp:15-36
  fus::DomainBox box{{0, 0, 0}, {10e-3, 7e-3, 5e-3}};
  const fus::VoxelGrid g = fus::make_grid(box, 1e-3, 1);
  CHECK(g.dims == Eigen::Vector3i(10, 7, 5));
  CHECK(g.count() == 350);
  CHECK(g.index(0, 1, 0) == 10 && g.index(0, 0, 1) == 70);
  CHECK(g.box.contains(box, 1e-12));
  CHECK_THROWS_AS(fus::make_grid(box, -1.0, 1), std::invalid_argument);
  // golden: proj/test_output.txt:31
  const fus::BowlTransducer h131 = fus::transducer_preset("H131", 100.0, 16);
  const fus::MeshPlan plan = fus::plan_nested_meshes(h131, kWater, 10.2e-3, 6, 5);
  CHECK(plan.reference.dims == Eigen::Vector3i(914, 737, 737));
  CHECK(plan.for_harmonic(2).grid.dims == Eigen::Vector3i(366, 295, 295));
  CHECK(std::fabs(plan.reduction_factor(2) - 15.586767385165057) < 1e-9);
  CHECK_THROWS_AS(plan.for_harmonic(9), std::out_of_range);
  CHECK(!plan.report().empty());
  // tests/test_transducer.cpp:50-69 (count, on sphere)
  for (int np : {1, 7, 128, 4096}) {
    const auto pts = fus::distribute_points(35e-3, 16.5e-3, np);
    CHECK(int(pts.size()) == np);
    bool on = true;
    for (const auto& p : pts)
      on = on && std::fabs((p - Eigen::Vector3d(35e-3, 0, 0)).norm() - 35e-3) < 1e-13 * 35e-3;
    CHECK(on);
  }
  // tests/test_medium.cpp
  const fus::Medium liver = fus::medium_preset("liver");
  const fus::Wavenumber k1 = fus::complex_wavenumber(liver, 1.1e6, 1);
  const fus::Wavenumber k4 = fus::complex_wavenumber(liver, 1.1e6, 4);
  CHECK(std::fabs(k4.k.real() - 4 * k1.k.real()) <= 1e-14 * k4.k.real());
  CHECK(std::fabs(k4.k.imag() / k1.k.imag() - std::pow(4.0, liver.eta)) < 1e-12);
  CHECK_THROWS_AS(fus::complex_wavenumber(liver, -1.0, 1), std::invalid_argument);
  CHECK_THROWS_AS(fus::medium_preset("granite"), std::invalid_argument);
  // tests/test_potential.cpp:40-46
  CHECK(std::fabs(fus::equivalent_sphere_radius(1.0) - 0.6203504908994001) < 1e-12);
}

// tests/test_io.cpp: parser, CSVs, field dump round trip; medium-map raster round trip
void io_cases() {
  {
    std::ofstream("t_kv.txt") << "# comment\n\n  key1 = 7.5  \nkey2=text value\n";
    const auto kv = fus::parse_key_value_file("t_kv.txt");
    CHECK(kv.size() == 2);
    CHECK(fus::require_double(kv, "key1", "test") == 7.5);
    CHECK(fus::require_string(kv, "key2", "test") == "text value");
    CHECK_THROWS_AS(fus::require_double(kv, "missing", "test"), std::runtime_error);
    CHECK_THROWS_AS(fus::require_double(kv, "key2", "test"), std::runtime_error);
    std::ofstream("t_bad.txt") << "ok = 1\nno equals sign here\n";
    bool line2 = false;
    try {
      fus::parse_key_value_file("t_bad.txt");
    } catch (const std::runtime_error& e) {
      line2 = std::string(e.what()).find(":2") != std::string::npos;
    }
    CHECK(line2);
    CHECK_THROWS_AS(fus::parse_key_value_file("no_such_file_anywhere.txt"), std::runtime_error);
  }
  {
    Eigen::VectorXd x(2);
    x[0] = 0.01;
    x[1] = 0.02;
    Eigen::VectorXcd p(2);
    p[0] = std::complex<double>(3, 4);
    p[1] = std::complex<double>(1, 0);
    fus::write_on_axis_csv("t_axis.csv", x, p);
    std::ifstream in("t_axis.csv");
    std::string header, row1;
    std::getline(in, header);
    std::getline(in, row1);
    CHECK(header == "x_m,re_Pa,im_Pa,abs_Pa");
    CHECK(row1.substr(0, 5) == "0.01," && row1.find(",5") != std::string::npos);
  }
  {
    fus::HarmonicField f;
    f.grid = fus::make_grid({{0, 0, 0}, {3e-4, 2e-4, 2e-4}}, 1e-4, 2);
    f.wavenumber = fus::complex_wavenumber(kWater, 1.1e6, 2);
    f.values = random_vector(f.grid.count(), 3);
    fus::write_field_dump("t_field.bin", f);
    const auto hdr = fus::parse_key_value_file("t_field.bin.hdr");
    CHECK(fus::require_double(hdr, "nx", "hdr") == f.grid.dims.x());
    CHECK(fus::require_double(hdr, "dx", "hdr") == f.grid.dx);
    CHECK(fus::require_double(hdr, "harmonic", "hdr") == 2);
    CHECK(fus::require_double(hdr, "k_re", "hdr") == f.wavenumber.k.real());
    CHECK(fus::require_string(hdr, "layout", "hdr") == "x_fastest_complex_f64_le");
    Eigen::VectorXcd back(f.values.size());
    std::ifstream in("t_field.bin", std::ios::binary);
    in.read(reinterpret_cast<char*>(back.data()), std::streamsize(back.size() * 16));
    CHECK(in.gcount() == std::streamsize(back.size() * 16));
    bool same = true;
    for (Eigen::Index i = 0; i < back.size(); ++i) same = same && back[i] == f.values[i];
    CHECK(same);
  }
  {
    fus::write_csv("t_gen.csv", {"a", "b"}, {{1, 2}, {3, 4.5}});
    std::ifstream in("t_gen.csv");
    std::string l0, l1, l2;
    std::getline(in, l0);
    std::getline(in, l1);
    std::getline(in, l2);
    CHECK(l0 == "a,b" && l1 == "1,2" && l2 == "3,4.5");
  }
  {
    const fus::VoxelGrid g = fus::make_grid({{0, 0, 0}, {5e-3, 4e-3, 3e-3}}, 1e-3, 1);
    const fus::MediumMap m = fus::slab_map(g, kWater, fus::medium_preset("liver"), 2e-3, 2e-3);
    fus::write_medium_map("t_map.hdr", "t_map.bin", m);
    const fus::MediumMap back = fus::load_medium_map("t_map.hdr", kWater);
    CHECK(back.grid.dims == g.dims && back.grid.dx == g.dx);
    bool same = back.c.size() == m.c.size();
    for (Eigen::Index i = 0; same && i < m.c.size(); ++i) same = back.c[i] == m.c[i] && back.beta[i] == m.beta[i];
    CHECK(same);
  }
  for (const char* f : {"t_kv.txt", "t_bad.txt", "t_axis.csv", "t_field.bin", "t_field.bin.hdr", "t_gen.csv",
                        "t_map.hdr", "t_map.bin"})
    std::remove(f);
}

void device_cases() {
  // tests/test_potential.cpp:75-92 and criterion 2
  fus::DomainBox box{{0, 0, 0}, {20e-4, 18e-4, 16e-4}};
  const fus::VoxelGrid grid = fus::make_grid(box, 1e-4, 2);
  CHECK(grid.dims == Eigen::Vector3i(20, 18, 16));
  const fus::Wavenumber k = fus::complex_wavenumber(kWater, 1.1e6, 2);
  for (unsigned seed : {1234u, 2024u}) {
    const Eigen::VectorXcd f = random_vector(grid.count(), seed);
    const fus::GreenKernel kernel(grid, k);
    const Eigen::VectorXcd u = kernel.apply(f);
    const Eigen::VectorXcd ref = direct(k, grid, f);
    CHECK(max_abs(u - ref) < 1e-12 * max_abs(ref));
    const fus::GreenKernel padded(grid, k, true);
    CHECK(max_abs(padded.apply(f) - ref) < 1e-12 * max_abs(ref));
  }
  CHECK_THROWS_AS(fus::GreenKernel(grid, k).apply(Eigen::VectorXcd(7)), std::invalid_argument);
  // delta column, tests/test_potential.cpp:117-139
  {
    const fus::VoxelGrid g = fus::make_grid({{0, 0, 0}, {9e-4, 8e-4, 7e-4}}, 1e-4, 1);
    const fus::Wavenumber k1 = fus::complex_wavenumber(kWater, 1.1e6, 1);
    Eigen::VectorXcd delta = Eigen::VectorXcd::Zero(static_cast<Eigen::Index>(g.count()));
    const std::size_t j = g.index(4, 3, 2);
    delta[static_cast<Eigen::Index>(j)] = 1.0;
    const Eigen::VectorXcd col = fus::GreenKernel(g, k1).apply(delta);
    const double vol = g.dx * g.dx * g.dx;
    bool ok = true;
    for (int iz = 0; iz < g.dims.z(); ++iz)
      for (int iy = 0; iy < g.dims.y(); ++iy)
        for (int ix = 0; ix < g.dims.x(); ++ix) {
          const std::size_t i = g.index(ix, iy, iz);
          const std::complex<double> want =
              i == j ? fus::self_weight(k1, g.dx)
                     : vol * fus::green_function(g.center(ix, iy, iz), g.center(4, 3, 2), k1);
          ok = ok && std::abs(col[static_cast<Eigen::Index>(i)] - want) < 1e-13 * std::abs(want) + 1e-20;
        }
    CHECK(ok);
  }
  // evaluate_potential_at agrees with apply at voxel centres, tests/test_potential.cpp:181-207
  {
    const fus::VoxelGrid g = fus::make_grid({{0, 0, 0}, {12e-4, 10e-4, 8e-4}}, 1e-4, 1);
    const fus::Wavenumber k2 = fus::complex_wavenumber(kWater, 1.1e6, 2);
    const Eigen::VectorXcd f = random_vector(g.count(), 99);
    const Eigen::VectorXcd u = fus::GreenKernel(g, k2).apply(f);
    std::vector<Eigen::Vector3d> pts;
    std::vector<std::size_t> idx;
    for (int iz = 0; iz < g.dims.z(); iz += 2)
      for (int iy = 0; iy < g.dims.y(); iy += 3)
        for (int ix = 0; ix < g.dims.x(); ix += 2) {
          pts.push_back(g.center(ix, iy, iz));
          idx.push_back(g.index(ix, iy, iz));
        }
    const Eigen::VectorXcd v = fus::evaluate_potential_at(k2, g, f, pts);
    bool ok = true;
    for (std::size_t i = 0; i < idx.size(); ++i)
      ok = ok && std::abs(v[Eigen::Index(i)] - u[Eigen::Index(idx[i])]) < 1e-12 * u.cwiseAbs().maxCoeff();
    CHECK(ok);
    const Eigen::VectorXcd w =
        fus::evaluate_potential_at(k2, g, f, {g.center(3, 2, 2) + Eigen::Vector3d(3e-5, 0, 0)});
    CHECK(std::isfinite(std::abs(w[0])));
    CHECK_THROWS_AS(fus::evaluate_potential_at(k2, g, Eigen::VectorXcd(3), pts), std::invalid_argument);
  }
  // VIE mode, tests/test_vie.cpp:105-213 through the drop-in
  {
    const int n = 48;
    std::mt19937 rng(7);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::vector<std::complex<double>> A(std::size_t(n) * n);  // dense, row-major
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) A[std::size_t(i) * n + j] = std::complex<double>(u(rng), u(rng)) * 0.1;
    for (int i = 0; i < n; ++i) A[std::size_t(i) * n + i] += 3.0;
    auto matvec = [](const std::vector<std::complex<double>>& M, int m, const Eigen::VectorXcd& x) {
      Eigen::VectorXcd y = Eigen::VectorXcd::Zero(m);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) y[i] += M[std::size_t(i) * m + j] * x[j];
      return y;
    };
    const Eigen::VectorXcd b = random_vector(n, 9);
    const fus::VieSolution sol =
        fus::gmres([&](const Eigen::VectorXcd& x) { return matvec(A, n, x); }, b, 1e-12, 500, 20);
    CHECK((matvec(A, n, sol.field) - b).norm() < 1e-11 * b.norm());
    CHECK(!sol.residual_history.empty() && sol.residual_history.back() < 1e-12);
    std::vector<std::complex<double>> S(64 * 64, 0.0);
    for (int i = 0; i < 64; ++i) S[std::size_t(i) * 64 + (i + 1) % 64] = 1.0;
    Eigen::VectorXcd e0 = Eigen::VectorXcd::Zero(64);
    e0[0] = 1.0;
    bool threw = false;
    try {
      fus::gmres([&](const Eigen::VectorXcd& x) { return matvec(S, 64, x); }, e0, 1e-14, 3, 3);
    } catch (const fus::ConvergenceError& e) {
      threw = !e.residual_history.empty();
    }
    CHECK(threw);
    const fus::VoxelGrid g = fus::make_grid({{0, 0, 0}, {3e-3, 3e-3, 3e-3}}, 0.3e-3, 1);
    const fus::Wavenumber k1 = fus::complex_wavenumber(kWater, 1.1e6, 1);
    const Eigen::VectorXcd rhs = random_vector(g.count(), 11);
    const fus::VieSolution z =
        fus::solve_vie(rhs, Eigen::VectorXcd::Zero(Eigen::Index(g.count())), fus::GreenKernel(g, k1), 1e-10);
    CHECK(max_abs(z.field - rhs) < 1e-10 * max_abs(rhs) && z.iterations <= 1);
    fus::CascadeConfig cfg;
    cfg.medium = kWater;
    cfg.transducer = fus::transducer_preset("H131", 15.0, 128);
    cfg.transducer.f0 = 0.25e6;
    cfg.plan = fus::plan_nested_meshes(cfg.transducer, cfg.medium, 6e-3, 3, 3, 0.35);
    cfg.n_harmonics = 3;
    const fus::CascadeResult homo = fus::run_cascade(cfg);
    fus::VieConfig vie;
    vie.tol = 1e-8;
    const fus::CascadeResult inhomo =
        fus::run_cascade_inhomogeneous(cfg, fus::homogeneous_map(cfg.plan.for_harmonic(2).grid, kWater), vie);
    for (int h = 1; h <= 3; ++h)
      CHECK((inhomo.p(h).values - homo.p(h).values).norm() / homo.p(h).values.norm() < 1e-6);
    const fus::MediumMap slab = fus::slab_map(cfg.plan.for_harmonic(2).grid, kWater,
                                              fus::medium_preset("liver"), 20e-3, 4e-3);
    CHECK(!slab.is_homogeneous());
    const fus::CascadeResult ws = fus::run_cascade_inhomogeneous(cfg, slab);
    const double rel = (ws.p(1).values - homo.p(1).values).norm() / homo.p(1).values.norm();
    CHECK(rel > 1e-3 && rel < 0.5);
  }
  // analysis through the drop-in: criterion 1's recorded errors and slope (proj/test_output.txt:20)
  // and the domain-shrink full-size level (tests/test_analysis.cpp:116-131)
  {
    const fus::Medium liver = fus::medium_preset("liver");
    const fus::BowlTransducer t = fus::transducer_preset("H131", 30.0, 128);
    const double lam = liver.c0 / t.f0;
    const Eigen::Vector3d focus = t.focus();
    fus::DomainBox box;
    box.lo = Eigen::Vector3d(focus.x() - 7.0 * lam, -1.5 * lam, -1.5 * lam);
    box.hi = Eigen::Vector3d(focus.x() + 7.0 * lam, 1.5 * lam, 1.5 * lam);
    const fus::QuadratureStudy st = fus::quadrature_convergence_study(t, liver, box, {4, 6, 8, 10}, 20);
    auto g4 = [](double v) {
      char b[32];
      std::snprintf(b, sizeof(b), "%.4g", v);
      return std::string(b);
    };
    CHECK(st.records.size() == 4 && g4(st.records[0].error_percent) == "0.6437" &&
          g4(st.records[1].error_percent) == "0.2641" && g4(st.records[2].error_percent) == "0.138" &&
          g4(st.records[3].error_percent) == "0.07983");
    CHECK(g4(st.slope) == "-2.269");
    fus::CascadeConfig cfg;
    cfg.medium = kWater;
    cfg.transducer = fus::transducer_preset("H131", 15.0, 128);
    cfg.transducer.f0 = 0.25e6;
    cfg.plan = fus::plan_full_domain(cfg.transducer, cfg.medium, 6e-3, 3, 2, 0.35);
    cfg.n_harmonics = 2;
    const fus::CascadeResult ref = fus::run_cascade(cfg);
    const auto recs = fus::domain_shrink_study(cfg, ref, {1.0, 0.5}, false);
    CHECK(recs.size() == 2 && recs[0].error_percent < 1e-6 && recs[1].error_percent > recs[0].error_percent &&
          recs[1].control == "fraction");
  }
  // rhs coefficients, tests/test_cascade.cpp:33-63
  {
    const fus::VoxelGrid g = fus::make_grid({{0, 0, 0}, {2e-3, 2e-3, 2e-3}}, 1e-3, 1);
    const double omega = 2 * M_PI * 1.1e6;
    const std::complex<double> a(2.0, 1.0), b(0.5, -3.0);
    std::vector<fus::HarmonicField> lower;
    lower.push_back({g, Eigen::VectorXcd::Constant(static_cast<Eigen::Index>(g.count()), a),
                     fus::complex_wavenumber(kWater, 1.1e6, 1)});
    lower.push_back({g, Eigen::VectorXcd::Constant(static_cast<Eigen::Index>(g.count()), b),
                     fus::complex_wavenumber(kWater, 1.1e6, 2)});
    const double base = kWater.beta * omega * omega / (2 * kWater.rho0 * std::pow(kWater.c0, 4));
    const Eigen::VectorXcd f3 = fus::rhs_source(3, lower, kWater, omega);
    CHECK(std::abs(f3[0] - base * 9.0 * 2.0 * a * b) < 1e-10 * std::abs(f3[0]));
    CHECK_THROWS_AS(fus::rhs_source(1, lower, kWater, omega), std::invalid_argument);
  }
  // interpolation exact on affine fields, tests/test_grid.cpp:90-122
  {
    const fus::VoxelGrid coarse = fus::make_grid({{0, 0, 0}, {8e-3, 8e-3, 8e-3}}, 1e-3, 1);
    const fus::VoxelGrid fine = fus::make_grid({{1e-3, 1e-3, 1e-3}, {7e-3, 7e-3, 7e-3}}, 0.4e-3, 2);
    auto affine = [](const Eigen::Vector3d& p) {
      return std::complex<double>(2.0 + 100.0 * p.x() - 40.0 * p.y(), 7.0 * p.z());
    };
    fus::HarmonicField f{coarse, Eigen::VectorXcd(static_cast<Eigen::Index>(coarse.count())),
                         fus::complex_wavenumber(kWater, 1.1e6, 1)};
    for (int iz = 0; iz < coarse.dims.z(); ++iz)
      for (int iy = 0; iy < coarse.dims.y(); ++iy)
        for (int ix = 0; ix < coarse.dims.x(); ++ix)
          f.values[static_cast<Eigen::Index>(coarse.index(ix, iy, iz))] = affine(coarse.center(ix, iy, iz));
    const fus::HarmonicField gfield = fus::interpolate(f, fine);
    double err = 0;
    for (int iz = 0; iz < fine.dims.z(); ++iz)
      for (int iy = 0; iy < fine.dims.y(); ++iy)
        for (int ix = 0; ix < fine.dims.x(); ++ix)
          err = std::max(err, std::abs(gfield.values[static_cast<Eigen::Index>(fine.index(ix, iy, iz))] -
                                       affine(fine.center(ix, iy, iz))));
    CHECK(err < 1e-12);
  }
  // power normalisation, tests/test_transducer.cpp:95-113
  {
    fus::BowlTransducer t = fus::transducer_preset("H131", 40.0, 512);
    const fus::Wavenumber k1 = fus::complex_wavenumber(kWater, t.f0, 1);
    const double s = fus::power_scale_factor(t, kWater, k1);
    CHECK(std::fabs(fus::radiated_power(t, kWater, k1, s) - 40.0) < 1e-12 * 40.0);
    t.power = 0.0;
    CHECK(fus::power_scale_factor(t, kWater, k1) == 0.0);
    CHECK_THROWS_AS(fus::unnormalized_field(t, {t.source_points[3]}, k1), std::invalid_argument);
  }
  // cascade structure, homogeneity and bitwise determinism, tests/test_cascade.cpp:65-106
  {
    auto tiny = [](double power) {
      fus::CascadeConfig cfg;
      cfg.medium = kWater;
      cfg.transducer = fus::transducer_preset("H131", power, 128);
      cfg.transducer.f0 = 0.25e6;
      cfg.plan = fus::plan_nested_meshes(cfg.transducer, cfg.medium, 6e-3, 3, 3, 0.35);
      cfg.n_harmonics = 3;
      return cfg;
    };
    const fus::CascadeResult r1 = fus::run_cascade(tiny(10.0));
    const fus::CascadeResult r4 = fus::run_cascade(tiny(40.0));
    CHECK(r1.harmonics.size() == 3 && r1.timings.size() == 2);
    CHECK(r1.timings[0].harmonic == 2 && r1.timings[1].harmonic == 3);
    const double s[3] = {2.0, 4.0, 8.0};
    for (int n = 1; n <= 3; ++n)
      CHECK((r4.p(n).values - s[n - 1] * r1.p(n).values).norm() / r1.p(n).values.norm() < 1e-12);
    const fus::CascadeResult again = fus::run_cascade(tiny(10.0));
    CHECK(again.p(2).values == r1.p(2).values && again.p(3).values == r1.p(3).values);
  }
}

// Every declaration of the drop-in headers not exercised above, as a reference user calls it:
// host-side ones always, device-side ones with `all`.
void surface_host_cases() {
  // medium / transducer presets, validation and config-file loaders (src/medium.cpp:47-69,
  // src/transducer.cpp:86-102)
  CHECK(fus::is_medium_preset("liver") && !fus::is_medium_preset("bone"));
  CHECK(fus::is_transducer_preset("H101") && !fus::is_transducer_preset("H999"));
  CHECK(std::fabs(fus::attenuation_np_per_m(kWater, 2.0e6) - 0.2 * 4.0 / fus::kDbPerNeper) < 1e-15);
  {
    const std::string mp = "/tmp/fus_api_medium.cfg", tp = "/tmp/fus_api_bowl.cfg";
    std::ofstream(mp) << "# tissue\nname = tissue\nrho0 = 1050\nc0 = 1540\nbeta = 4.5\nalpha0 = 0.5\neta = 1.1\n";
    std::ofstream(tp) << "name = bowl\nf0 = 1e6\nfocal_length = 0.04\nouter_radius = 0.02\nn_points = 128\n";
    const fus::Medium m = fus::load_medium(mp);
    CHECK(m.name == "tissue" && m.rho0 == 1050.0 && m.c0 == 1540.0 && m.beta == 4.5 && m.alpha0 == 0.5 && m.eta == 1.1);
    CHECK(m.validate().empty());
    const fus::BowlTransducer t = fus::load_transducer(tp, 12.5);
    const fus::BowlTransducer u = fus::make_bowl("bowl", 1e6, 0.04, 0.02, 12.5, 128);
    CHECK(t.name == "bowl" && t.power == 12.5 && t.source_points.size() == 128);
    CHECK(t.source_points[77] == u.source_points[77]);
    CHECK(std::fabs(t.cap_area() - 2.0 * M_PI * 0.04 * t.rim_plane_x()) < 1e-18);
    std::ofstream(mp) << "name = broken\nrho0 = 1050\n";
    CHECK_THROWS_AS(fus::load_medium(mp), std::runtime_error);
    fus::Medium bad = kWater;
    bad.c0 = -1.0;
    CHECK_THROWS_AS(bad.validate(), std::invalid_argument);
  }
  // reference domain and the single-mesh plan (src/grid.cpp:70-79, src/cascade.cpp:109-118)
  {
    const fus::BowlTransducer t = fus::transducer_preset("H131");
    const fus::DomainBox d2 = fus::reference_domain(t, 10.2e-3);
    CHECK(d2.contains(t.focus()) && d2.extent().x() > 0.0);
    const fus::MeshPlan single = fus::plan_single_mesh(t, kWater, 10.2e-3, 6, 3);
    for (int n = 2; n <= 3; ++n) CHECK(single.for_harmonic(n).grid.dims == single.for_harmonic(2).grid.dims);
  }
}

void surface_device_cases() {
  const fus::BowlTransducer t = [] {
    fus::BowlTransducer b = fus::transducer_preset("H131", 20.0, 256);
    b.f0 = 0.25e6;
    return b;
  }();
  const fus::MeshPlan plan = fus::plan_nested_meshes(t, kWater, 6e-3, 3, 3, 0.35);
  const fus::VoxelGrid g2 = plan.for_harmonic(2).grid;
  // source field, power normalisation, first harmonic (src/transducer.cpp:179-206)
  const fus::SourceField sf = fus::evaluate_source_field(t, kWater, g2);
  const fus::Wavenumber k1 = fus::complex_wavenumber(kWater, t.f0, 1);
  const fus::HarmonicField p1 = fus::evaluate_first_harmonic(t, kWater, g2, sf.normalization);
  CHECK((p1.values - sf.field.values).norm() <= 1e-12 * sf.field.values.norm());
  fus::SourceField raw{fus::evaluate_first_harmonic(t, kWater, g2, 1.0), 1.0};
  const fus::SourceField normed = fus::normalize_to_power(raw, t, kWater);
  CHECK(std::fabs(normed.normalization - fus::power_scale_factor(t, kWater, k1)) <= 1e-12 * normed.normalization);
  // direct O(N^2) quadrature vs the FFT apply (tests/test_potential.cpp:75-92)
  {
    const fus::VoxelGrid g = fus::make_grid({{0, 0, 0}, {12e-4, 10e-4, 8e-4}}, 1e-4, 2);
    const fus::Wavenumber k = fus::complex_wavenumber(kWater, 1.1e6, 2);
    const Eigen::VectorXcd f = random_vector(g.count(), 21);
    const Eigen::VectorXcd d = fus::direct_potential_oracle(k, g, f);
    CHECK((fus::GreenKernel(g, k).apply(f) - d).cwiseAbs().maxCoeff() < 1e-12 * max_abs(d));
    CHECK((d - direct(k, g, f)).cwiseAbs().maxCoeff() < 1e-12 * max_abs(d));
    const fus::VoxelGrid big = fus::make_grid({{0, 0, 0}, {60e-4, 50e-4, 40e-4}}, 1e-4, 2);
    CHECK_THROWS_AS(fus::direct_potential_oracle(k, big, Eigen::VectorXcd::Zero(Eigen::Index(big.count()))),
                    std::invalid_argument);
    // apply_device / native on caller-owned device buffers
    fus::GreenKernel K(g, k);
    CHECK(K.native() != nullptr);
    std::complex<double>*fd = nullptr, *ud = nullptr;
    const size_t bytes = g.count() * sizeof(std::complex<double>);
    CHECK(cudaMalloc(&fd, bytes) == cudaSuccess && cudaMalloc(&ud, bytes) == cudaSuccess);
    cudaMemcpy(fd, f.data(), bytes, cudaMemcpyHostToDevice);
    K.apply_device(fd, ud, -1.0);
    cudaDeviceSynchronize();
    Eigen::VectorXcd u(Eigen::Index(g.count()));
    cudaMemcpy(u.data(), ud, bytes, cudaMemcpyDeviceToHost);
    CHECK((u + K.apply(f)).cwiseAbs().maxCoeff() <= 1e-15 * max_abs(u));
    cudaFree(fd);
    cudaFree(ud);
  }
  // on-axis profiles and the shrink diagnostics (src/analysis.cpp:26-90,176-242; src/grid.cpp:114-139)
  {
    const fus::OnAxisProfile a = fus::extract_on_axis(p1);
    CHECK(a.x.size() == a.p.size() && a.x.size() > 2);
    CHECK(fus::on_axis_error(a, a, a) == 0.0);
    const Eigen::VectorXd q = fus::localisedness_map(p1);
    CHECK(q.size() == Eigen::Index(p1.grid.count()) && q.maxCoeff() <= 1.0 + 1e-15);
    const fus::DomainBox box = fus::shrink_domain_by_threshold(p1, 0.5);
    CHECK(p1.grid.box.contains(box, 1e-12));
    CHECK(std::isfinite(fus::error_trend_diagnostic(a, a, 0.5)));
  }
  // VIE pieces on a liver slab (src/vie.cpp:11-323)
  {
    const fus::Medium liver = fus::medium_preset("liver");
    const fus::MediumMap mm = fus::slab_map(g2, kWater, liver, t.focal_length, 2e-3);
    CHECK(!mm.is_homogeneous() && !mm.contrast_support().empty());
    const Eigen::VectorXcd contrast = mm.wavenumber_contrast(t.f0, 2);
    CHECK(contrast.size() == Eigen::Index(g2.count()));
    const fus::MediumMap half = mm.resample(plan.for_harmonic(3).grid);
    CHECK(half.c.size() == Eigen::Index(plan.for_harmonic(3).grid.count()));
    const fus::GreenKernel K(g2, fus::complex_wavenumber(kWater, t.f0, 2));
    const Eigen::VectorXcd lhs = fus::vie_operator_apply(p1.values, contrast, K);
    const Eigen::VectorXcd v = contrast.cwiseProduct(p1.values);
    CHECK((lhs - (p1.values - K.apply(v))).cwiseAbs().maxCoeff() <= 1e-12 * max_abs(lhs));
  }
}

}  // namespace

int main(int argc, char** argv) {
  const bool all = argc > 1 && std::strcmp(argv[1], "all") == 0;
  try {
    host_cases();
    io_cases();
    surface_host_cases();
    if (all) {
      device_cases();
      surface_device_cases();
    }
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught exception: %s\n", e.what());
    ++g_fail;
  }
  std::printf("%s: %d passed, %d failed\n", g_fail ? "FAILED" : "OK", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
