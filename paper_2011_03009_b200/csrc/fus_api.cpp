// namespace fus drop-in (reference signatures, include/fus/*.hpp) over the C-ABI of libfusg.so.
//
// Host arithmetic delegates to the library's bit-exact C++ (make_grid, planner, wavenumbers,
// point layout); numerics run on the GPU through fusg_* calls.  Errors come back as the
// reference's exception types.  Device: FUSG_DEVICE (default 0), one process-wide context.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <cstring>
#include <iostream>
#include <mutex>
#include <sstream>
#include <stdexcept>

#include "fus/cascade.hpp"
#include "fus/grid.hpp"
#include "fus/medium.hpp"
#include "fus/potential.hpp"
#include "fus/transducer.hpp"
#include "fus/vie.hpp"
#include "fus_api_detail.hpp"
#include "fusg.h"

namespace fus {
namespace detail {

void check(fusg_status st) {
  if (st == FUSG_OK) return;
  const std::string msg = fusg_last_error();
  switch (st) {
    case FUSG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FUSG_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

fusg_ctx* ctx() {
  static std::once_flag once;
  static fusg_ctx* c = nullptr;
  std::call_once(once, [] {
    const char* e = std::getenv("FUSG_DEVICE");
    check(fusg_ctx_create(e ? std::atoi(e) : 0, &c));
  });
  return c;
}

DevBuf upload(const Eigen::VectorXcd& v) {
  DevBuf b(size_t(v.size()) * 16);
  if (v.size()) cuda_check(cudaMemcpy(b.p, v.data(), size_t(v.size()) * 16, cudaMemcpyHostToDevice), "upload");
  return b;
}

Eigen::VectorXcd download(const DevBuf& b, size_t n) {
  Eigen::VectorXcd v(static_cast<Eigen::Index>(n));
  if (n) cuda_check(cudaMemcpy(v.data(), b.p, n * 16, cudaMemcpyDeviceToHost), "download");
  return v;
}

fusg_grid to_c(const VoxelGrid& g) {
  fusg_grid c{};
  for (int a = 0; a < 3; ++a) {
    c.lo[a] = g.box.lo[a];
    c.hi[a] = g.box.hi[a];
    c.dims[a] = g.dims[a];
  }
  c.dx = g.dx;
  c.harmonic = g.harmonic;
  return c;
}

VoxelGrid from_c(const fusg_grid& c) {
  VoxelGrid g;
  for (int a = 0; a < 3; ++a) {
    g.box.lo[a] = c.lo[a];
    g.box.hi[a] = c.hi[a];
    g.dims[a] = c.dims[a];
  }
  g.dx = c.dx;
  g.harmonic = c.harmonic;
  return g;
}

fusg_wavenumber to_c(const Wavenumber& k) { return {k.k.real(), k.k.imag(), k.harmonic, k.omega}; }
fusg_medium to_c(const Medium& m) { return {m.rho0, m.c0, m.beta, m.alpha0, m.eta}; }

std::vector<double> flat_points(const std::vector<Eigen::Vector3d>& pts) {
  std::vector<double> f(3 * pts.size());
  for (size_t i = 0; i < pts.size(); ++i)
    for (int a = 0; a < 3; ++a) f[3 * i + a] = pts[i][a];
  return f;
}

}  // namespace detail
using namespace detail;

// ------------------------------------------------------------------------------ medium
std::vector<std::string> Medium::validate() const {  // src/medium.cpp:11-23
  if (rho0 <= 0.0) throw std::invalid_argument("medium '" + name + "': rho0 must be positive");
  if (c0 <= 0.0) throw std::invalid_argument("medium '" + name + "': c0 must be positive");
  if (beta < 0.0) throw std::invalid_argument("medium '" + name + "': beta must be non-negative");
  if (alpha0 < 0.0) throw std::invalid_argument("medium '" + name + "': alpha0 must be non-negative");
  std::vector<std::string> w;
  if (eta < 1.0 || eta > 2.0)
    w.push_back("medium '" + name + "': power-law exponent eta=" + std::to_string(eta) +
                " is outside the typical range [1, 2]");
  return w;
}

double attenuation_np_per_m(const Medium& m, double f_hz) {
  const double f_mhz = f_hz / 1.0e6;
  return m.alpha0 * std::pow(f_mhz, m.eta) / kDbPerNeper;
}

Wavenumber complex_wavenumber(const Medium& m, double f0, int n) {
  const fusg_medium mc = to_c(m);
  fusg_wavenumber k{};
  check(fusg_complex_wavenumber(&mc, f0, n, &k));
  return {{k.k_re, k.k_im}, k.harmonic, k.omega};
}

Medium medium_preset(const std::string& name) {  // src/medium.cpp:47-52
  if (name == "water") return Medium{"water", 1000.0, 1480.0, 3.5, 0.2, 2.0};
  if (name == "liver") return Medium{"liver", 1060.0, 1590.0, 4.4, 90.0, 1.1};
  if (name == "kidney") return Medium{"kidney", 1050.0, 1570.0, 4.7, 10.0, 1.0};
  throw std::invalid_argument("unknown medium preset '" + name + "'");
}

bool is_medium_preset(const std::string& n) { return n == "water" || n == "liver" || n == "kidney"; }

// ------------------------------------------------------------------------------ grid
VoxelGrid make_grid(const DomainBox& request, double dx, int harmonic,
                    const std::optional<Eigen::Vector3d>& anchor) {
  const double lo[3] = {request.lo[0], request.lo[1], request.lo[2]};
  const double hi[3] = {request.hi[0], request.hi[1], request.hi[2]};
  double a[3];
  if (anchor)
    for (int i = 0; i < 3; ++i) a[i] = (*anchor)[i];
  fusg_grid g{};
  check(fusg_make_grid(lo, hi, dx, harmonic, anchor ? a : nullptr, &g));
  return from_c(g);
}

const PlannedGrid& MeshPlan::for_harmonic(int n) const {
  for (const auto& pg : grids)
    if (pg.harmonic == n) return pg;
  throw std::out_of_range("MeshPlan: no grid planned for harmonic " + std::to_string(n));
}

double MeshPlan::reduction_factor(int n) const {
  return double(reference.count()) / double(for_harmonic(n).grid.count());
}

std::string MeshPlan::report() const {
  std::ostringstream os;
  auto gib = [](std::size_t n) { return 16.0 * double(n) / (1024.0 * 1024.0 * 1024.0); };
  os << "nested mesh plan (n_w = " << n_w << ", d = " << d * 1e3 << " mm, w = " << w * 1e3 << " mm)\n";
  os << "  reference mesh (harmonic " << reference.harmonic << "): " << reference.dims.x() << " x "
     << reference.dims.y() << " x " << reference.dims.z() << " = " << double(reference.count())
     << " voxels, dx = " << reference.dx * 1e6 << " um, " << gib(reference.count()) << " GiB/field\n";
  std::size_t total = 0;
  for (const auto& pg : grids) {
    total += pg.grid.count();
    os << "  p" << pg.harmonic << ": " << pg.grid.dims.x() << " x " << pg.grid.dims.y() << " x "
       << pg.grid.dims.z() << " = " << double(pg.grid.count()) << " voxels, dx = " << pg.grid.dx * 1e6
       << " um, " << gib(pg.grid.count()) << " GiB/field, reduction " << reduction_factor(pg.harmonic)
       << "x\n";
  }
  const double single = double(reference.count()) * double(grids.size());
  os << "  total nested voxels: " << double(total) << " (vs " << single
     << " with all harmonics on the reference mesh, reduction " << single / double(total) << "x)\n";
  return os.str();
}

DomainBox reference_domain(const BowlTransducer& t, double d) {  // src/grid.cpp:70-79
  if (d < 0.0) throw std::invalid_argument("reference_domain: d must be >= 0");
  const double l = t.focal_length, R = t.outer_radius;
  const double L = std::sqrt(l * l - R * R) - 0.1e-3;
  DomainBox box;
  box.lo = {l - L, -R, -R};
  box.hi = {l + d, R, R};
  return box;
}

static MeshPlan plan(const BowlTransducer& t, const Medium& m, double d, int n_w, int n_h,
                     double width_scale, bool single) {
  if (n_h < 2) throw std::invalid_argument("plan_nested_meshes: need n_harmonics >= 2");
  const BowlC bc(t);
  const fusg_medium mc = to_c(m);
  std::vector<fusg_grid> grids(n_h - 1);
  std::vector<double> lo(3 * (n_h - 1)), hi(3 * (n_h - 1));
  fusg_grid ref{};
  double w = 0.0;
  check(fusg_plan_nested_meshes(&bc.c, &mc, d, n_w, n_h, width_scale, single ? 1 : 0, grids.data(),
                                lo.data(), hi.data(), &ref, &w));
  MeshPlan p;
  p.d = d;
  p.w = w;
  p.n_w = n_w;
  p.focus = t.focus();
  p.reference = from_c(ref);
  for (int i = 0; i < n_h - 1; ++i) {
    PlannedGrid pg;
    pg.harmonic = i + 2;
    pg.domain.lo = {lo[3 * i], lo[3 * i + 1], lo[3 * i + 2]};
    pg.domain.hi = {hi[3 * i], hi[3 * i + 1], hi[3 * i + 2]};
    pg.grid = from_c(grids[i]);
    p.grids.push_back(pg);
  }
  return p;
}

MeshPlan plan_nested_meshes(const BowlTransducer& t, const Medium& m, double d, int n_w,
                            int n_harmonics, double width_scale) {
  return plan(t, m, d, n_w, n_harmonics, width_scale, false);
}

MeshPlan plan_single_mesh(const BowlTransducer& t, const Medium& m, double d, int n_w,
                          int n_harmonics, double width_scale) {
  return plan(t, m, d, n_w, n_harmonics, width_scale, true);
}

HarmonicField interpolate(const HarmonicField& field, const VoxelGrid& target) {
  if (field.values.size() != Eigen::Index(field.grid.count()))
    throw std::invalid_argument("interpolate: field size does not match its grid");
  const DevBuf src = upload(field.values);
  DevBuf out(target.count() * 16);
  const fusg_grid sg = to_c(field.grid), tg = to_c(target);
  check(fusg_interpolate(ctx(), &sg, src.d(), &tg, out.d(), nullptr));
  check(fusg_ctx_synchronize(ctx()));
  return {target, download(out, target.count()), field.wavenumber};
}

// ------------------------------------------------------------------------------ potential
std::complex<double> green_function(const Eigen::Vector3d& x, const Eigen::Vector3d& y,
                                    const Wavenumber& k) {  // src/potential.cpp:47-53
  const double r = (x - y).norm();
  if (r < 1e-300) throw std::invalid_argument("green_function: singular at x == y");
  const double mag = std::exp(-k.k.imag() * r) / (4.0 * M_PI * r);
  return std::polar(mag, k.k.real() * r);
}

double equivalent_sphere_radius(double dx) { return fusg_equivalent_sphere_radius(dx); }

std::complex<double> self_weight(const Wavenumber& k, double dx) {
  const fusg_wavenumber kc = to_c(k);
  double w[2];
  check(fusg_self_weight(&kc, dx, w));
  return {w[0], w[1]};
}

GreenKernel::GreenKernel(const VoxelGrid& grid, const Wavenumber& k, bool pad_small_primes)
    : grid_(grid), k_(k) {
  const fusg_grid g = to_c(grid);
  const fusg_wavenumber kc = to_c(k);
  fusg_kernel* h = nullptr;
  check(fusg_kernel_create(ctx(), &g, &kc, pad_small_primes ? 1 : 0, &h));
  handle_ = std::shared_ptr<fusg_kernel>(h, [](fusg_kernel* p) { fusg_kernel_destroy(p); });
}

Eigen::VectorXcd GreenKernel::apply(const Eigen::VectorXcd& f) const {
  if (f.size() != Eigen::Index(grid_.count()))
    throw std::invalid_argument("GreenKernel::apply: field size does not match kernel grid");
  Eigen::VectorXcd u(f.size());
  check(fusg_kernel_apply_host(handle_.get(), reinterpret_cast<const double*>(f.data()),
                               reinterpret_cast<double*>(u.data()), 1.0));
  return u;
}

HarmonicField GreenKernel::apply(const HarmonicField& f) const { return {grid_, apply(f.values), k_}; }

void GreenKernel::apply_device(const std::complex<double>* f, std::complex<double>* u, double scale,
                               void* stream) const {
  check(fusg_kernel_apply(handle_.get(), reinterpret_cast<const double*>(f),
                          reinterpret_cast<double*>(u), scale, stream));
}

Eigen::Vector3i GreenKernel::padded() const {
  int32_t p[3];
  check(fusg_kernel_padded(handle_.get(), p));
  return Eigen::Vector3i(p[0], p[1], p[2]);
}

Eigen::VectorXcd evaluate_potential_at(const Wavenumber& k, const VoxelGrid& grid, const Eigen::VectorXcd& f,
                                       const std::vector<Eigen::Vector3d>& points) {
  if (f.size() != Eigen::Index(grid.count()))
    throw std::invalid_argument("evaluate_potential_at: field size mismatch");
  const fusg_grid g = to_c(grid);
  const fusg_wavenumber kc = to_c(k);
  std::vector<double> pts(3 * points.size());
  for (size_t i = 0; i < points.size(); ++i)
    for (int a = 0; a < 3; ++a) pts[3 * i + a] = points[i][a];
  const DevBuf fd = upload(f);
  Eigen::VectorXcd out(static_cast<Eigen::Index>(points.size()));
  check(fusg_evaluate_potential_at(ctx(), &g, &kc, fd.d(), pts.data(), int64_t(points.size()),
                                   reinterpret_cast<double*>(out.data())));
  return out;
}

Eigen::VectorXcd direct_potential_oracle(const Wavenumber& k, const VoxelGrid& grid, const Eigen::VectorXcd& f) {
  if (grid.count() > 100000)
    throw std::invalid_argument("direct_potential_oracle: grid exceeds the 1e5 voxel guard");
  if (f.size() != Eigen::Index(grid.count()))
    throw std::invalid_argument("direct_potential_oracle: field size mismatch");
  std::vector<Eigen::Vector3d> centres(grid.count());
  for (int iz = 0; iz < grid.dims.z(); ++iz)
    for (int iy = 0; iy < grid.dims.y(); ++iy)
      for (int ix = 0; ix < grid.dims.x(); ++ix) centres[grid.index(ix, iy, iz)] = grid.center(ix, iy, iz);
  return evaluate_potential_at(k, grid, f, centres);
}

// ------------------------------------------------------------------------------ transducer
double BowlTransducer::cap_area() const {
  const double l = focal_length, R = outer_radius;
  return 2.0 * M_PI * l * (l - std::sqrt(l * l - R * R));
}

double BowlTransducer::rim_plane_x() const {
  const double l = focal_length, R = outer_radius;
  return l - std::sqrt(l * l - R * R);
}

std::vector<Eigen::Vector3d> distribute_points(double l, double R, int n) {
  std::vector<double> f(3 * size_t(std::max(n, 0)));
  check(fusg_distribute_points(l, R, n, f.data()));
  std::vector<Eigen::Vector3d> pts(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) pts[size_t(i)] = {f[3 * i], f[3 * i + 1], f[3 * i + 2]};
  return pts;
}

BowlTransducer make_bowl(const std::string& name, double f0, double l, double R, double power,
                         int n_points) {  // src/transducer.cpp:72-84
  if (f0 <= 0.0) throw std::invalid_argument("make_bowl: f0 must be positive");
  if (power < 0.0) throw std::invalid_argument("make_bowl: power must be >= 0");
  return BowlTransducer{name, f0, l, R, power, distribute_points(l, R, n_points)};
}

BowlTransducer transducer_preset(const std::string& name, double power, int n_points) {
  if (name == "H101") return make_bowl("H101", 1.1e6, 63.2e-3, 32.0e-3, power, n_points);
  if (name == "H131") return make_bowl("H131", 1.1e6, 35.0e-3, 16.5e-3, power, n_points);
  throw std::invalid_argument("unknown transducer preset '" + name + "'");
}

bool is_transducer_preset(const std::string& n) { return n == "H101" || n == "H131"; }

Eigen::VectorXcd unnormalized_field(const BowlTransducer& t, const std::vector<Eigen::Vector3d>& pts,
                                    const Wavenumber& k) {
  const BowlC bc(t);
  const std::vector<double> fp = flat_points(pts);
  DevBuf dp(fp.size() * sizeof(double)), out(pts.size() * 16);
  if (!fp.empty())
    cuda_check(cudaMemcpy(dp.p, fp.data(), fp.size() * sizeof(double), cudaMemcpyHostToDevice), "upload");
  const double amp = t.cap_area() / double(t.source_points.size());
  check(fusg_monopole_points(ctx(), bc.pts.data(), bc.c.n_points, dp.d(), int64_t(pts.size()),
                             k.k.real(), k.k.imag(), amp, out.d(), nullptr));
  return download(out, pts.size());
}

double radiated_power(const BowlTransducer& t, const Medium& m, const Wavenumber& k,
                      double amplitude_scale, int n_r, int n_theta) {
  const BowlC bc(t);
  const double amp = amplitude_scale * t.cap_area() / double(t.source_points.size());
  double out = 0.0;
  check(fusg_radiated_power(ctx(), bc.pts.data(), bc.c.n_points, t.rim_plane_x(), t.outer_radius,
                            k.k.real(), k.k.imag(), amp, m.rho0, m.c0, n_r, n_theta, &out));
  return out;
}

double power_scale_factor(const BowlTransducer& t, const Medium& m, const Wavenumber& k) {
  if (t.power == 0.0) return 0.0;  // src/transducer.cpp:157-163
  const double pw = radiated_power(t, m, k, 1.0);
  if (pw <= 0.0) throw std::runtime_error("power normalization: degenerate field, Pi(p) = 0");
  return std::sqrt(t.power / pw);
}

SourceField normalize_to_power(const SourceField& field, const BowlTransducer& t, const Medium& m) {
  if (field.normalization <= 0.0)  // src/transducer.cpp:165-177
    throw std::invalid_argument("normalize_to_power: normalization factor must be positive");
  const double factor = power_scale_factor(t, m, field.field.wavenumber);
  SourceField out;
  out.field.grid = field.field.grid;
  out.field.wavenumber = field.field.wavenumber;
  out.field.values = field.field.values * (factor / field.normalization);
  out.normalization = factor > 0.0 ? factor : 1.0;
  if (factor == 0.0) out.field.values.setZero();
  return out;
}

HarmonicField evaluate_first_harmonic(const BowlTransducer& t, const Medium& m, const VoxelGrid& grid,
                                      double amplitude_scale) {
  const Wavenumber k1 = complex_wavenumber(m, t.f0, 1);
  const double amp = amplitude_scale * t.cap_area() / double(t.source_points.size());
  const BowlC bc(t);
  const fusg_grid g = to_c(grid);
  DevBuf out(grid.count() * 16);
  check(fusg_monopole_grid(ctx(), bc.pts.data(), bc.c.n_points, &g, k1.k.real(), k1.k.imag(), amp,
                           out.d(), nullptr));
  return {grid, download(out, grid.count()), k1};
}

SourceField evaluate_source_field(const BowlTransducer& t, const Medium& m, const VoxelGrid& grid) {
  const Wavenumber k1 = complex_wavenumber(m, t.f0, 1);
  const double scale = power_scale_factor(t, m, k1);
  SourceField s;
  s.field = evaluate_first_harmonic(t, m, grid, scale);
  s.normalization = scale > 0.0 ? scale : 1.0;
  return s;
}

// ------------------------------------------------------------------------------ cascade
Eigen::VectorXcd rhs_source(int n, const std::vector<HarmonicField>& lower, const Medium& m,
                            double omega) {  // src/cascade.cpp:21-40
  if (n < 2) throw std::invalid_argument("rhs_source: harmonic index must be >= 2");
  if (int(lower.size()) < n - 1)
    throw std::invalid_argument("rhs_source: missing lower harmonics for n = " + std::to_string(n));
  const Eigen::Index count = lower[0].values.size();
  for (int i = 1; i < n; ++i)
    if (lower[i - 1].values.size() != count)
      throw std::invalid_argument("rhs_source: lower harmonics live on different grids");
  std::vector<std::unique_ptr<DevBuf>> bufs;
  std::vector<const double*> ptrs;
  for (int i = 0; i < n - 1; ++i) {
    bufs.push_back(std::make_unique<DevBuf>(size_t(count) * 16));
    cuda_check(cudaMemcpy(bufs.back()->p, lower[i].values.data(), size_t(count) * 16,
                          cudaMemcpyHostToDevice), "upload");
    ptrs.push_back(bufs.back()->d());
  }
  DevBuf out(size_t(count) * 16);
  const fusg_medium mc = to_c(m);
  check(fusg_rhs_source(ctx(), n, ptrs.data(), count, &mc, omega, out.d(), nullptr));
  check(fusg_ctx_synchronize(ctx()));
  return download(out, size_t(count));
}

CascadeResult run_cascade(const CascadeConfig& cfg) {  // src/cascade.cpp:42-107
  const int n = cfg.n_harmonics;
  if (n < 2) throw std::invalid_argument("run_cascade: n_harmonics must be >= 2");
  std::vector<fusg_grid> grids;
  for (int i = 2; i <= n; ++i) grids.push_back(to_c(cfg.plan.for_harmonic(i).grid));
  const BowlC bc(cfg.transducer);
  fusg_cascade_desc d{to_c(cfg.medium), bc.c, grids.data(), n,
                      cfg.recompute_p1_each_grid ? 1 : 0, cfg.pad_small_primes ? 1 : 0};
  std::vector<std::unique_ptr<DevBuf>> out;
  std::vector<double*> ptrs;
  for (int i = 0; i < n; ++i) {
    const fusg_grid& g = grids[size_t(std::max(i - 1, 0))];
    out.push_back(std::make_unique<DevBuf>(size_t(g.dims[0]) * g.dims[1] * g.dims[2] * 16));
    ptrs.push_back(out.back()->d());
  }
  std::vector<fusg_stage_timing> rows(size_t(n - 1));
  double norm = 1.0;
  check(fusg_run_cascade(ctx(), &d, ptrs.data(), rows.data(), &norm));
  CascadeResult r;
  r.source_normalization = norm;
  for (int i = 0; i < n; ++i) {
    const VoxelGrid g = from_c(grids[size_t(std::max(i - 1, 0))]);
    r.harmonics.push_back({g, download(*out[size_t(i)], g.count()),
                           complex_wavenumber(cfg.medium, cfg.transducer.f0, i + 1)});
  }
  for (const auto& row : rows)
    r.timings.push_back({row.harmonic, std::size_t(row.voxels), row.meshing_s, row.interpolation_s,
                         row.kernel_s, row.potential_s, row.p1_s, row.rhs_s});
  return r;
}

}  // namespace fus
