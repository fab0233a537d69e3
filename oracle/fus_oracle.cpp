// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into or called by the product path.
//
// CPU restatement of the fus-harmonics reference (arXiv 2011.03009 C++ tree under
// /root/reference/proj) for the volume-potential hot path. Each function follows the cited
// reference function statement by statement, in the reference's expression order, so the
// oracle rounds the way the reference does (compile with -O2 -ffp-contract=off, like the
// reference's default x86-64 GCC build which has no FMA).
//
// The reference itself cannot be built here (Eigen3, FFTW3 and vendor/ are absent; see
// DESIGN.md), so this file is the "port" oracle. It is pinned against the reference's own
// known-answer tests and recorded goldens (tests/test_oracle_*.py).
//
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load it.
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

using cd = std::complex<double>;

namespace {

thread_local char g_err[512];

int fail(const char* msg) {
  std::snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

struct Grid {
  double lo[3], hi[3], dx;
  int dims[3];
  std::size_t count() const { return std::size_t(dims[0]) * dims[1] * dims[2]; }
  std::size_t index(int ix, int iy, int iz) const {
    return std::size_t(ix) + std::size_t(dims[0]) * (std::size_t(iy) + std::size_t(dims[1]) * iz);
  }
  // include/fus/grid.hpp:44-46  center = lo + ((i+0.5)dx, ...)
  double center(int a, int i) const { return lo[a] + (i + 0.5) * dx; }
};

Grid to_grid(const double* lo, const double* hi, double dx, const int* dims) {
  Grid g;
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = lo[a];
    g.hi[a] = hi[a];
    g.dims[a] = dims[a];
  }
  g.dx = dx;
  return g;
}

// src/transducer.cpp:107-119 monopole_sum (throws on coincidence -> returns false)
bool monopole_sum(const double* src, int n_src, double x, double y, double z, cd k, cd* out) {
  cd acc = 0.0;
  for (int i = 0; i < n_src; ++i) {
    const double ddx = x - src[3 * i + 0], ddy = y - src[3 * i + 1], ddz = z - src[3 * i + 2];
    // Eigen's (x - r).norm() = sqrt(dx*dx + dy*dy + dz*dz) summed left to right
    const double dist = std::sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    if (dist < 1e-12) return false;
    const double mag = std::exp(-k.imag() * dist) / (4.0 * M_PI * dist);
    acc += std::polar(mag, k.real() * dist);
  }
  *out = acc;
  return true;
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err; }

int orc_num_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

// tests/acceptance.cpp:30-36 random_vector: std::mt19937(seed) +
// uniform_real_distribution<double>(-1,1), real then imaginary per element.
void orc_random_vector(std::int64_t n, unsigned seed, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (std::int64_t i = 0; i < n; ++i) {
    const double re = u(rng);
    const double im = u(rng);
    out[2 * i] = re;
    out[2 * i + 1] = im;
  }
}

// src/grid.cpp:12-34 make_grid
int orc_make_grid(const double* req_lo, const double* req_hi, double dx, const double* anchor,
                  double* out_lo, double* out_hi, int* out_dims) {
  if (dx <= 0.0) return fail("make_grid: dx must be positive");
  for (int a = 0; a < 3; ++a)
    if (req_hi[a] - req_lo[a] <= 0.0) return fail("make_grid: degenerate domain box");
  for (int a = 0; a < 3; ++a) {
    double lo = req_lo[a];
    if (anchor) {
      const double m = std::ceil((anchor[a] - lo) / dx - 0.5 - 1e-12);
      lo = anchor[a] - (m + 0.5) * dx;
    }
    const int n = std::max(1, int(std::ceil((req_hi[a] - lo) / dx - 1e-9)));
    out_lo[a] = lo;
    out_hi[a] = lo + n * dx;
    out_dims[a] = n;
  }
  return 0;
}

// src/potential.cpp:55-70 equivalent_sphere_radius / self_weight
double orc_equivalent_sphere_radius(double dx) { return dx * std::cbrt(3.0 / (4.0 * M_PI)); }

int orc_self_weight(double k_re, double k_im, double dx, double* out) {
  if (dx <= 0.0) return fail("self_weight: delta_x must be positive");
  const cd k(k_re, k_im);
  const double a = orc_equivalent_sphere_radius(dx);
  const cd ka = k * a;
  cd w;
  if (std::abs(ka) < 1e-3) {
    w = a * a / 2.0 + cd(0.0, 1.0) * k * (a * a * a) / 3.0 - k * k * (a * a * a * a) / 8.0;
  } else {
    const cd i(0.0, 1.0);
    w = (std::exp(i * ka) * (1.0 - i * ka) - 1.0) / (k * k);
  }
  out[0] = w.real();
  out[1] = w.imag();
  return 0;
}

// src/potential.cpp:47-53 green_function at distance r (x != y)
void orc_green(double k_re, double k_im, double r, double* out) {
  const double mag = std::exp(-k_im * r) / (4.0 * M_PI * r);
  const cd g = std::polar(mag, k_re * r);
  out[0] = g.real();
  out[1] = g.imag();
}

// src/potential.cpp:72-115 GreenKernel constructor: embedded kernel tensor on the padded
// box (x fastest), before its forward DFT (done by the Python glue with numpy).
int orc_kernel_fill(const int* n, const int* p, double dx, double k_re, double k_im,
                    double* out /* 2*Px*Py*Pz */) {
  const cd k(k_re, k_im);
  const double vol = dx * dx * dx;
  double sw[2];
  if (orc_self_weight(k_re, k_im, dx, sw)) return 1;
  const cd self(sw[0], sw[1]);
  auto offset_of = [](int m, int count, int padded) -> int {
    if (m < count) return m;
    if (m > padded - count) return m - padded;
    return INT32_MIN;
  };
  const std::size_t total = std::size_t(p[0]) * p[1] * p[2];
  std::memset(out, 0, 2 * sizeof(double) * total);
#pragma omp parallel for collapse(2) schedule(static)
  for (int iz = 0; iz < p[2]; ++iz)
    for (int iy = 0; iy < p[1]; ++iy) {
      const int oz = offset_of(iz, n[2], p[2]);
      const int oy = offset_of(iy, n[1], p[1]);
      if (oz == INT32_MIN || oy == INT32_MIN) continue;
      for (int ix = 0; ix < p[0]; ++ix) {
        const int ox = offset_of(ix, n[0], p[0]);
        if (ox == INT32_MIN) continue;
        const std::size_t idx =
            std::size_t(ix) + std::size_t(p[0]) * (std::size_t(iy) + std::size_t(p[1]) * iz);
        cd v;
        if (ox == 0 && oy == 0 && oz == 0) {
          v = self;
        } else {
          const double r = dx * std::sqrt(double(ox) * ox + double(oy) * oy + double(oz) * oz);
          const double mag = std::exp(-k.imag() * r) / (4.0 * M_PI * r);
          v = vol * std::polar(mag, k.real() * r);
        }
        out[2 * idx] = v.real();
        out[2 * idx + 1] = v.imag();
      }
    }
  return 0;
}

// src/potential.cpp:203-238 direct_potential_oracle (O(N^2)); the 1e5 guard is kept.
int orc_direct_potential(const double* lo, const double* hi, double dx, const int* dims,
                         double k_re, double k_im, const double* f, double* out) {
  const Grid g = to_grid(lo, hi, dx, dims);
  if (g.count() > 100000) return fail("direct_potential_oracle: grid exceeds the 1e5 voxel guard");
  const cd k(k_re, k_im);
  const double vol = dx * dx * dx;
  double sw[2];
  if (orc_self_weight(k_re, k_im, dx, sw)) return 1;
  const cd self(sw[0], sw[1]);
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const cd* fc = reinterpret_cast<const cd*>(f);
  cd* oc = reinterpret_cast<cd*>(out);
#pragma omp parallel for collapse(2) schedule(static)
  for (int iz = 0; iz < nz; ++iz)
    for (int iy = 0; iy < ny; ++iy)
      for (int ix = 0; ix < nx; ++ix) {
        cd acc = 0.0;
        for (int jz = 0; jz < nz; ++jz)
          for (int jy = 0; jy < ny; ++jy)
            for (int jx = 0; jx < nx; ++jx) {
              const cd fj = fc[g.index(jx, jy, jz)];
              if (ix == jx && iy == jy && iz == jz) {
                acc += self * fj;
              } else {
                const double r = dx * std::sqrt(double(ix - jx) * (ix - jx) +
                                                double(iy - jy) * (iy - jy) +
                                                double(iz - jz) * (iz - jz));
                const double mag = std::exp(-k.imag() * r) / (4.0 * M_PI * r);
                acc += vol * std::polar(mag, k.real() * r) * fj;
              }
            }
        oc[g.index(ix, iy, iz)] = acc;
      }
  return 0;
}

// direct_potential_oracle (src/potential.cpp:203-238) evaluated only at the output voxels idx[]:
// the same per-pair formula, O(N) per output, no voxel guard.  Each output sums plane by
// plane (plane partial sums in source order, then planes in order), so the result does not
// depend on the thread count.  Used to check full-size applies at sampled voxels.
int orc_direct_potential_at(const double* lo, const double* hi, double dx, const int* dims,
                            double k_re, double k_im, const double* f, const std::int64_t* idx,
                            std::int64_t n_idx, double* out) {
  const Grid g = to_grid(lo, hi, dx, dims);
  const cd k(k_re, k_im);
  const double vol = dx * dx * dx;
  double sw[2];
  if (orc_self_weight(k_re, k_im, dx, sw)) return 1;
  const cd self(sw[0], sw[1]);
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const cd* fc = reinterpret_cast<const cd*>(f);
  cd* oc = reinterpret_cast<cd*>(out);
  std::vector<cd> planes(nz);
  for (std::int64_t q = 0; q < n_idx; ++q) {
    const std::int64_t i = idx[q];
    if (i < 0 || i >= std::int64_t(g.count())) return fail("direct_potential_at: voxel index out of range");
    const int ix = int(i % nx), iy = int((i / nx) % ny), iz = int(i / (std::int64_t(nx) * ny));
#pragma omp parallel for schedule(dynamic)
    for (int jz = 0; jz < nz; ++jz) {
      cd acc = 0.0;
      for (int jy = 0; jy < ny; ++jy)
        for (int jx = 0; jx < nx; ++jx) {
          const cd fj = fc[g.index(jx, jy, jz)];
          if (ix == jx && iy == jy && iz == jz) {
            acc += self * fj;
          } else {
            const double r = dx * std::sqrt(double(ix - jx) * (ix - jx) + double(iy - jy) * (iy - jy) +
                                            double(iz - jz) * (iz - jz));
            const double mag = std::exp(-k.imag() * r) / (4.0 * M_PI * r);
            acc += vol * std::polar(mag, k.real() * r) * fj;
          }
        }
      planes[jz] = acc;
    }
    cd total = 0.0;
    for (int jz = 0; jz < nz; ++jz) total += planes[jz];
    oc[q] = total;
  }
  return 0;
}

// src/potential.cpp:161-201 evaluate_potential_at
int orc_evaluate_potential_at(double k_re, double k_im, const double* lo, const double* hi,
                              double dx, const int* dims, const double* f, const double* pts,
                              std::int64_t n_pts, double* out) {
  const Grid g = to_grid(lo, hi, dx, dims);
  const cd k(k_re, k_im);
  const double vol = dx * dx * dx;
  double sw[2];
  if (orc_self_weight(k_re, k_im, dx, sw)) return 1;
  const cd self(sw[0], sw[1]);
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const double coincident = 1e-9 * dx;
  const cd* fc = reinterpret_cast<const cd*>(f);
  cd* oc = reinterpret_cast<cd*>(out);
#pragma omp parallel for schedule(static)
  for (std::int64_t pi = 0; pi < n_pts; ++pi) {
    const double x0 = pts[3 * pi], x1 = pts[3 * pi + 1], x2 = pts[3 * pi + 2];
    cd acc = 0.0;
    for (int jz = 0; jz < nz; ++jz)
      for (int jy = 0; jy < ny; ++jy) {
        const double cy = g.lo[1] + (jy + 0.5) * dx - x1;
        const double cz = g.lo[2] + (jz + 0.5) * dx - x2;
        const double ryz2 = cy * cy + cz * cz;
        const std::size_t row = g.index(0, jy, jz);
        for (int jx = 0; jx < nx; ++jx) {
          const cd fj = fc[row + jx];
          if (fj == cd(0.0, 0.0)) continue;
          const double cx = g.lo[0] + (jx + 0.5) * dx - x0;
          const double r = std::sqrt(cx * cx + ryz2);
          if (r < coincident) {
            acc += self * fj;
          } else {
            const double mag = std::exp(-k.imag() * r) / (4.0 * M_PI * r);
            acc += vol * std::polar(mag, k.real() * r) * fj;
          }
        }
      }
    oc[pi] = acc;
  }
  return 0;
}

// src/transducer.cpp:22-70 distribute_points
int orc_distribute_points(double focal_length, double outer_radius, int n_points, double* out) {
  const double l = focal_length, R = outer_radius;
  if (n_points < 1) return fail("distribute_points: n_points must be >= 1");
  if (!(R > 0.0 && R < l)) return fail("distribute_points: need 0 < R < l (non-degenerate cap)");
  auto cap_point = [&](double theta, double phi, double* o) {
    // focus + l * (-cos t, sin t cos p, sin t sin p)
    o[0] = l + l * -std::cos(theta);
    o[1] = 0.0 + l * (std::sin(theta) * std::cos(phi));
    o[2] = 0.0 + l * (std::sin(theta) * std::sin(phi));
  };
  if (n_points == 1) {
    cap_point(0.0, 0.0, out);
    return 0;
  }
  const double theta_max = std::asin(R / l);
  const double area = 2.0 * M_PI * l * (l - std::sqrt(l * l - R * R));
  const double spacing = std::sqrt(area / n_points);
  const int n_rings = std::max(1, int(std::lround(theta_max * l / spacing)));
  std::vector<double> theta(n_rings), weight(n_rings);
  double total_weight = 0.0;
  for (int m = 0; m < n_rings; ++m) {
    theta[m] = theta_max * (m + 0.5) / n_rings;
    weight[m] = std::sin(theta[m]);
    total_weight += weight[m];
  }
  double cum = 0.0;
  long assigned = 0;
  int w = 0;
  for (int m = 0; m < n_rings; ++m) {
    cum += weight[m];
    const long upto = std::lround(n_points * cum / total_weight);
    const long in_ring = upto - assigned;
    assigned = upto;
    if (in_ring <= 0) continue;
    const double offset = 2.0 * M_PI * std::fmod(m * 0.618033988749895, 1.0);
    for (long j = 0; j < in_ring; ++j) {
      const double phi = 2.0 * M_PI * (j + 0.5) / double(in_ring) + offset;
      if (w >= n_points) return fail("distribute_points: layout overflow");
      cap_point(theta[m], phi, out + 3 * w);
      ++w;
    }
  }
  if (w != n_points) return fail("distribute_points: layout count mismatch");
  return 0;
}

// src/transducer.cpp:123-132 unnormalized_field (amp = 1 there; amp passed explicitly here)
int orc_monopole_points(const double* src, int n_src, const double* pts, std::int64_t n_pts,
                        double k_re, double k_im, double amp, double* out) {
  const cd k(k_re, k_im);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (std::int64_t i = 0; i < n_pts; ++i) {
    cd s;
    if (!monopole_sum(src, n_src, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], k, &s)) {
      bad = 1;
      continue;
    }
    const cd v = amp * s;
    out[2 * i] = v.real();
    out[2 * i + 1] = v.imag();
  }
  if (bad) return fail("evaluation point coincides with a monopole source");
  return 0;
}

// src/transducer.cpp:179-196 evaluate_first_harmonic on voxel centres
int orc_monopole_grid(const double* src, int n_src, const double* lo, const double* hi, double dx,
                      const int* dims, double k_re, double k_im, double amp, double* out) {
  const Grid g = to_grid(lo, hi, dx, dims);
  const cd k(k_re, k_im);
  int bad = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(| : bad)
  for (int iz = 0; iz < dims[2]; ++iz)
    for (int iy = 0; iy < dims[1]; ++iy)
      for (int ix = 0; ix < dims[0]; ++ix) {
        cd s;
        if (!monopole_sum(src, n_src, g.center(0, ix), g.center(1, iy), g.center(2, iz), k, &s)) {
          bad = 1;
          continue;
        }
        const cd v = amp * s;
        const std::size_t idx = g.index(ix, iy, iz);
        out[2 * idx] = v.real();
        out[2 * idx + 1] = v.imag();
      }
  if (bad) return fail("evaluation point coincides with a monopole source");
  return 0;
}

// src/transducer.cpp:134-155 radiated_power. amp = amplitude_scale * A / n_p.
// The reference reduces over rings with an OpenMP reduction; here rings are summed in
// ascending order (the 1-thread order).
int orc_radiated_power(const double* src, int n_src, double x_disc, double R, double k_re,
                       double k_im, double amp, double rho0, double c0, int n_r, int n_theta,
                       double* out) {
  const cd k(k_re, k_im);
  const double dr = R / n_r;
  const double dth = 2.0 * M_PI / n_theta;
  std::vector<double> rings(n_r);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int j = 0; j < n_r; ++j) {
    const double r = (j + 0.5) * dr;
    double ring = 0.0;
    for (int m = 0; m < n_theta; ++m) {
      const double th = (m + 0.5) * dth;
      cd s;
      if (!monopole_sum(src, n_src, x_disc, r * std::cos(th), r * std::sin(th), k, &s)) {
        bad = 1;
        break;
      }
      ring += std::norm(amp * s);
    }
    rings[j] = ring * r;
  }
  if (bad) return fail("evaluation point coincides with a monopole source");
  double total = 0.0;
  for (int j = 0; j < n_r; ++j) total += rings[j];
  *out = total * dr * dth / (2.0 * rho0 * c0);
  return 0;
}

// src/grid.cpp:141-195 interpolate
int orc_interpolate(const double* s_lo, const double* s_hi, double s_dx, const int* s_dims,
                    const double* f, const double* t_lo, const double* t_hi, double t_dx,
                    const int* t_dims, double* out) {
  const Grid src = to_grid(s_lo, s_hi, s_dx, s_dims);
  const Grid tgt = to_grid(t_lo, t_hi, t_dx, t_dims);
  for (int a = 0; a < 3; ++a)
    if (tgt.lo[a] < src.lo[a] - src.dx || tgt.hi[a] > src.hi[a] + src.dx)
      return fail(
          "interpolate: target extends more than one source voxel beyond the source domain");
  const int* n = s_dims;
  auto clampi = [](int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); };
  const cd* fc = reinterpret_cast<const cd*>(f);
  cd* oc = reinterpret_cast<cd*>(out);
#pragma omp parallel for collapse(2) schedule(static)
  for (int iz = 0; iz < t_dims[2]; ++iz)
    for (int iy = 0; iy < t_dims[1]; ++iy)
      for (int ix = 0; ix < t_dims[0]; ++ix) {
        const double p[3] = {tgt.center(0, ix), tgt.center(1, iy), tgt.center(2, iz)};
        int i0[3];
        double t[3];
        for (int a = 0; a < 3; ++a) {
          const double q = (p[a] - src.lo[a]) / src.dx - 0.5;
          int base = int(std::floor(q));
          base = clampi(base, 0, std::max(0, n[a] - 2));
          double frac = q - base;
          if (frac < 0.0) frac = 0.0;
          if (frac > 1.0) frac = n[a] > 1 ? 1.0 : 0.0;
          i0[a] = base;
          t[a] = frac;
        }
        cd acc = 0.0;
        for (int cz = 0; cz < 2; ++cz)
          for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx) {
              const double wgt = (cx ? t[0] : 1.0 - t[0]) * (cy ? t[1] : 1.0 - t[1]) *
                                 (cz ? t[2] : 1.0 - t[2]);
              if (wgt == 0.0) continue;
              const int jx = clampi(i0[0] + cx, 0, n[0] - 1);
              const int jy = clampi(i0[1] + cy, 0, n[1] - 1);
              const int jz = clampi(i0[2] + cz, 0, n[2] - 1);
              acc += wgt * fc[src.index(jx, jy, jz)];
            }
        oc[tgt.index(ix, iy, iz)] = acc;
      }
  return 0;
}

// src/cascade.cpp:21-40 rhs_source. lower: n-1 pointers to fields of `count` elements.
void orc_rhs_source(int n, const double* const* lower, std::int64_t count, double beta,
                    double omega, double rho0, double c0, double* out) {
  const double coeff =
      beta * omega * omega * double(n) * double(n) / (2.0 * rho0 * std::pow(c0, 4));
  cd* oc = reinterpret_cast<cd*>(out);
  for (std::int64_t i = 0; i < count; ++i) oc[i] = 0.0;
  for (int m = 1; m <= n - 1; ++m) {
    const cd* a = reinterpret_cast<const cd*>(lower[m - 1]);
    const cd* b = reinterpret_cast<const cd*>(lower[n - m - 1]);
    for (std::int64_t i = 0; i < count; ++i) oc[i] += a[i] * b[i];
  }
  for (std::int64_t i = 0; i < count; ++i) oc[i] = coeff * oc[i];
}

}  // extern "C"
