// namespace fus VIE mode (reference include/fus/vie.hpp, src/vie.cpp) over the C-ABI: the
// contrast, operator, GMRES, solve_vie and the inhomogeneous cascade run on the GPU; the map
// constructors and support queries are host arithmetic like the reference's.
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fus/vie.hpp"
#include "fus_api_detail.hpp"

namespace fus {
using namespace detail;

namespace {

DevBuf upload_map(const MediumMap& m) {  // (c, beta) interleaved: one complex field
  const Eigen::Index n = m.c.size();
  if (m.beta.size() != n || n != Eigen::Index(m.grid.count()))
    throw std::invalid_argument("MediumMap: c / beta sizes do not match the grid");
  Eigen::VectorXcd packed(n);
  for (Eigen::Index i = 0; i < n; ++i) packed[i] = {m.c[i], m.beta[i]};
  return upload(packed);
}

// fusg_status -> exception, with the residual history for non-convergence
void check_vie(fusg_status st, const std::vector<double>& hist) {
  if (st == FUSG_NOT_CONVERGED) throw ConvergenceError(fusg_last_error(), hist);
  check(st);
}

VieSolution finish(fusg_status st, std::vector<double>& hist, int len, int it, const DevBuf& x, std::size_t n) {
  hist.resize(std::min<std::size_t>(hist.size(), std::size_t(std::max(len, 0))));
  check_vie(st, hist);
  VieSolution sol;
  sol.field = download(x, n);
  sol.residual_history = hist;
  sol.iterations = it;
  return sol;
}

int history_capacity(int max_iter, int restart) { return max_iter + max_iter / std::max(1, restart) + 4; }

}  // namespace

Eigen::VectorXcd MediumMap::wavenumber_contrast(double f0, int n) const {  // src/vie.cpp:11-23
  const DevBuf m = upload_map(*this);
  DevBuf out(std::size_t(c.size()) * 16);
  const fusg_medium bg = to_c(background);
  check(fusg_vie_contrast(ctx(), m.d(), c.size(), &bg, f0, n, out.d(), nullptr));
  check(fusg_ctx_synchronize(ctx()));
  return download(out, std::size_t(c.size()));
}

std::vector<std::size_t> MediumMap::contrast_support(double tol) const {  // src/vie.cpp:25-31
  std::vector<std::size_t> support;
  for (Eigen::Index i = 0; i < c.size(); ++i)
    if (std::abs(c[i] - background.c0) > tol || std::abs(beta[i] - background.beta) > tol)
      support.push_back(std::size_t(i));
  return support;
}

bool MediumMap::is_homogeneous() const { return contrast_support().empty(); }

MediumMap MediumMap::resample(const VoxelGrid& target) const {  // src/vie.cpp:35-54
  HarmonicField packed;
  packed.grid = grid;
  packed.values.resize(c.size());
  for (Eigen::Index i = 0; i < c.size(); ++i) packed.values[i] = {c[i], beta[i]};
  const HarmonicField res = interpolate(packed, target);
  MediumMap out;
  out.grid = target;
  out.background = background;
  out.c.resize(res.values.size());
  out.beta.resize(res.values.size());
  for (Eigen::Index i = 0; i < res.values.size(); ++i) {
    out.c[i] = res.values[i].real();
    out.beta[i] = res.values[i].imag();
  }
  return out;
}

MediumMap homogeneous_map(const VoxelGrid& grid, const Medium& background) {  // src/vie.cpp:56-63
  MediumMap m;
  m.grid = grid;
  m.background = background;
  m.c = Eigen::VectorXd::Constant(Eigen::Index(grid.count()), background.c0);
  m.beta = Eigen::VectorXd::Constant(Eigen::Index(grid.count()), background.beta);
  return m;
}

MediumMap slab_map(const VoxelGrid& grid, const Medium& background, const Medium& inclusion, double x_center,
                   double thickness) {  // src/vie.cpp:65-81
  MediumMap m = homogeneous_map(grid, background);
  const double lo = x_center - thickness / 2.0, hi = x_center + thickness / 2.0;
  for (int iz = 0; iz < grid.dims.z(); ++iz)
    for (int iy = 0; iy < grid.dims.y(); ++iy)
      for (int ix = 0; ix < grid.dims.x(); ++ix) {
        const double x = grid.center(ix, iy, iz).x();
        if (x >= lo && x <= hi) {
          const Eigen::Index i = Eigen::Index(grid.index(ix, iy, iz));
          m.c[i] = inclusion.c0;
          m.beta[i] = inclusion.beta;
        }
      }
  return m;
}

Eigen::VectorXcd vie_operator_apply(const Eigen::VectorXcd& field, const Eigen::VectorXcd& contrast,
                                    const GreenKernel& kernel) {  // src/vie.cpp:133-139
  if (field.size() != contrast.size() || field.size() != Eigen::Index(kernel.grid().count()))
    throw std::invalid_argument("vie_operator_apply: grid mismatch");
  const DevBuf p = upload(field), c = upload(contrast);
  DevBuf out(std::size_t(field.size()) * 16);
  check(fusg_vie_operator_apply(kernel.native(), c.d(), p.d(), out.d(), nullptr));
  check(fusg_ctx_synchronize(ctx()));
  return download(out, std::size_t(field.size()));
}

namespace {
struct HostOp {
  const std::function<Eigen::VectorXcd(const Eigen::VectorXcd&)>* op;
  std::size_t n;
  std::string error;
};
fusg_status host_op_trampoline(void* user, const double* in_dev, double* out_dev) {
  auto* h = static_cast<HostOp*>(user);
  try {
    Eigen::VectorXcd x(static_cast<Eigen::Index>(h->n));
    cuda_check(cudaMemcpy(x.data(), in_dev, h->n * 16, cudaMemcpyDeviceToHost), "gmres operator input");
    const Eigen::VectorXcd y = (*h->op)(x);
    if (std::size_t(y.size()) != h->n) throw std::invalid_argument("gmres: operator changed the vector size");
    cuda_check(cudaMemcpy(out_dev, y.data(), h->n * 16, cudaMemcpyHostToDevice), "gmres operator output");
    return FUSG_OK;
  } catch (const std::exception& e) {
    h->error = e.what();
    return FUSG_RUNTIME;
  }
}
}  // namespace

VieSolution gmres(const std::function<Eigen::VectorXcd(const Eigen::VectorXcd&)>& op, const Eigen::VectorXcd& rhs,
                  double tol, int max_iter, int restart) {  // src/vie.cpp:141-236, Krylov basis on the GPU
  const std::size_t n = std::size_t(rhs.size());
  const DevBuf b = upload(rhs);
  DevBuf x(n * 16);
  HostOp h{&op, n, {}};
  std::vector<double> hist(std::size_t(history_capacity(max_iter, restart)));
  int len = 0, it = 0;
  const fusg_status st = fusg_gmres(ctx(), host_op_trampoline, &h, b.d(), int64_t(n), tol, max_iter, restart,
                                    x.d(), hist.data(), int(hist.size()), &len, &it);
  if (st != FUSG_OK && !h.error.empty()) throw std::runtime_error(h.error);
  return finish(st, hist, len, it, x, n);
}

VieSolution solve_vie(const Eigen::VectorXcd& rhs, const Eigen::VectorXcd& contrast, const GreenKernel& kernel,
                      double tol, int max_iter, int restart) {  // src/vie.cpp:238-242
  if (rhs.size() != contrast.size() || rhs.size() != Eigen::Index(kernel.grid().count()))
    throw std::invalid_argument("solve_vie: grid mismatch");
  const std::size_t n = std::size_t(rhs.size());
  const DevBuf b = upload(rhs), c = upload(contrast);
  DevBuf x(n * 16);
  std::vector<double> hist(std::size_t(history_capacity(max_iter, restart)));
  int len = 0, it = 0;
  const fusg_status st = fusg_solve_vie(kernel.native(), b.d(), c.d(), tol, max_iter, restart, x.d(),
                                        hist.data(), int(hist.size()), &len, &it);
  return finish(st, hist, len, it, x, n);
}

CascadeResult run_cascade_inhomogeneous(const CascadeConfig& cfg, const MediumMap& master_map,
                                        const VieConfig& vie) {  // src/vie.cpp:244-323
  const int n = cfg.n_harmonics;
  if (n < 1) throw std::invalid_argument("run_cascade_inhomogeneous: n_harmonics must be >= 1");
  std::vector<fusg_grid> grids;
  for (int i = 2; i <= std::max(n, 2); ++i) grids.push_back(to_c(cfg.plan.for_harmonic(i).grid));
  const BowlC bc(cfg.transducer);
  fusg_cascade_desc d{to_c(cfg.medium), bc.c, grids.data(), n, cfg.recompute_p1_each_grid ? 1 : 0,
                      cfg.pad_small_primes ? 1 : 0};
  std::vector<std::unique_ptr<DevBuf>> out;
  std::vector<double*> ptrs;
  for (int i = 0; i < n; ++i) {
    const fusg_grid& g = grids[std::size_t(std::max(i - 1, 0))];
    out.push_back(std::make_unique<DevBuf>(std::size_t(g.dims[0]) * g.dims[1] * g.dims[2] * 16));
    ptrs.push_back(out.back()->d());
  }
  std::vector<double> raster(std::size_t(2 * master_map.c.size()));
  for (Eigen::Index i = 0; i < master_map.c.size(); ++i) {
    raster[std::size_t(2 * i)] = master_map.c[i];
    raster[std::size_t(2 * i + 1)] = master_map.beta[i];
  }
  const fusg_grid mg = to_c(master_map.grid);
  const fusg_medium bg = to_c(master_map.background);
  const fusg_vie_config vc{vie.tol, vie.max_iter, vie.restart};
  std::vector<fusg_stage_timing> rows(std::size_t(std::max(n - 1, 1)));
  double norm = 1.0;
  check(fusg_run_cascade_inhomogeneous(ctx(), &d, &mg, raster.data(), &bg, &vc, ptrs.data(), rows.data(), &norm));
  CascadeResult r;
  r.source_normalization = norm;
  for (int i = 0; i < n; ++i) {
    const VoxelGrid g = from_c(grids[std::size_t(std::max(i - 1, 0))]);
    r.harmonics.push_back({g, download(*out[std::size_t(i)], g.count()),
                           complex_wavenumber(master_map.background, cfg.transducer.f0, i + 1)});
  }
  for (int i = 0; i + 1 < n; ++i) {
    StageTiming st;
    st.harmonic = rows[std::size_t(i)].harmonic;
    st.voxels = std::size_t(rows[std::size_t(i)].voxels);
    r.timings.push_back(st);
  }
  return r;
}

}  // namespace fus
