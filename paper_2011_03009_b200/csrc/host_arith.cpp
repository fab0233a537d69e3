// Host-side arithmetic of the drop-in boundary: grid construction, nested-mesh planning,
// wavenumbers, self weight and the bowl point layout.  These are scalar, microsecond-scale
// computations whose results must be bit-identical to the reference (they fix voxel counts,
// grid origins and crop indices), so they stay on the host and are compiled with
// -ffp-contract=off in the reference's expression order.
#include <cmath>
#include <complex>
#include <cstdio>
#include <iostream>
#include <random>
#include <string>
#include <vector>

#include "internal.hpp"

namespace fusg {

static thread_local std::string g_error;

fusg_status set_error(fusg_status st, const std::string& msg) {
  g_error = msg;
  return st;
}

fusg_status cuda_error(cudaError_t e, const char* what) {
  const fusg_status st = (e == cudaErrorMemoryAllocation) ? FUSG_OOM : FUSG_CUDA;
  return set_error(st, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace fusg

using fusg::set_error;

extern "C" {

const char* fusg_last_error(void) { return fusg::g_error.c_str(); }
const char* fusg_version(void) { return "fusg 0.1 (sm_100a)"; }

// src/grid.cpp:12-34
fusg_status fusg_make_grid(const double req_lo[3], const double req_hi[3], double dx,
                           int32_t harmonic, const double* anchor, fusg_grid* out) {
  if (!out || !req_lo || !req_hi) return set_error(FUSG_INVALID_ARGUMENT, "make_grid: null argument");
  if (dx <= 0.0) return set_error(FUSG_INVALID_ARGUMENT, "make_grid: dx must be positive");
  for (int a = 0; a < 3; ++a)
    if (req_hi[a] - req_lo[a] <= 0.0)
      return set_error(FUSG_INVALID_ARGUMENT, "make_grid: degenerate domain box");
  fusg_grid g{};
  g.dx = dx;
  g.harmonic = harmonic;
  for (int a = 0; a < 3; ++a) {
    double lo = req_lo[a];
    if (anchor) {
      const double m = std::ceil((anchor[a] - lo) / dx - 0.5 - 1e-12);
      lo = anchor[a] - (m + 0.5) * dx;
    }
    const int n = std::max(1, int(std::ceil((req_hi[a] - lo) / dx - 1e-9)));
    g.lo[a] = lo;
    g.hi[a] = lo + n * dx;
    g.dims[a] = n;
  }
  *out = g;
  return FUSG_OK;
}

// src/medium.cpp:25-45
fusg_status fusg_complex_wavenumber(const fusg_medium* m, double f0, int32_t n,
                                    fusg_wavenumber* out) {
  if (f0 <= 0.0) return set_error(FUSG_INVALID_ARGUMENT, "complex_wavenumber: f0 must be positive");
  if (n < 1)
    return set_error(FUSG_INVALID_ARGUMENT, "complex_wavenumber: harmonic index must be >= 1");
  const double omega = 2.0 * M_PI * f0;
  const double f_mhz = (n * f0) / 1.0e6;
  const double alpha = m->alpha0 * std::pow(f_mhz, m->eta) / 8.685889638065035;
  if (alpha * m->c0 / (n * omega) >= 0.1)
    std::cerr << "warning: power-law attenuation bound alpha*c0/omega < 0.1 violated at harmonic "
              << n << "\n";
  out->k_re = n * omega / m->c0;
  out->k_im = alpha;
  out->harmonic = n;
  out->omega = omega;
  return FUSG_OK;
}

// src/potential.cpp:55-57
double fusg_equivalent_sphere_radius(double dx) { return dx * std::cbrt(3.0 / (4.0 * M_PI)); }

// src/potential.cpp:59-70
fusg_status fusg_self_weight(const fusg_wavenumber* kw, double dx, double out[2]) {
  if (dx <= 0.0) return set_error(FUSG_INVALID_ARGUMENT, "self_weight: delta_x must be positive");
  using cd = std::complex<double>;
  const cd k(kw->k_re, kw->k_im);
  const double a = fusg_equivalent_sphere_radius(dx);
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
  return FUSG_OK;
}

// src/potential.cpp:36-43
int32_t fusg_next_fast_size(int32_t n) {
  for (;; ++n) {
    int m = n;
    for (int p : {2, 3, 5, 7})
      while (m % p == 0) m /= p;
    if (m == 1) return n;
  }
}

fusg_status fusg_padded_dims(const fusg_grid* g, int32_t pad_small_primes, int32_t out[3]) {
  for (int a = 0; a < 3; ++a) {
    if (g->dims[a] < 1) return set_error(FUSG_INVALID_ARGUMENT, "padded_dims: empty grid");
    out[a] = pad_small_primes ? fusg::smooth_padded_size(g->dims[a], true)
                              : fusg::device_padded_size(g->dims[a], a);
  }
  return FUSG_OK;
}

// src/transducer.cpp:22-70
fusg_status fusg_distribute_points(double focal_length, double outer_radius, int32_t n_points,
                                   double* out) {
  const double l = focal_length, R = outer_radius;
  if (n_points < 1)
    return set_error(FUSG_INVALID_ARGUMENT, "distribute_points: n_points must be >= 1");
  if (!(R > 0.0 && R < l))
    return set_error(FUSG_INVALID_ARGUMENT, "distribute_points: need 0 < R < l (non-degenerate cap)");
  auto cap_point = [&](double theta, double phi, double* o) {
    o[0] = l + l * -std::cos(theta);
    o[1] = 0.0 + l * (std::sin(theta) * std::cos(phi));
    o[2] = 0.0 + l * (std::sin(theta) * std::sin(phi));
  };
  if (n_points == 1) {
    cap_point(0.0, 0.0, out);
    return FUSG_OK;
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
      if (w >= n_points) return set_error(FUSG_RUNTIME, "distribute_points: layout overflow");
      cap_point(theta[m], phi, out + 3 * w);
      ++w;
    }
  }
  if (w != n_points) return set_error(FUSG_RUNTIME, "distribute_points: layout count mismatch");
  return FUSG_OK;
}

// src/grid.cpp:70-112 (reference_domain + plan_nested_meshes); src/cascade.cpp:109-118
fusg_status fusg_plan_nested_meshes(const fusg_bowl* t, const fusg_medium* med, double d,
                                    int32_t n_w, int32_t n_harmonics, double width_scale,
                                    int32_t single_mesh, fusg_grid* out_grids, double* dlo,
                                    double* dhi, fusg_grid* reference, double* w_out) {
  if (n_harmonics < 2)
    return set_error(FUSG_INVALID_ARGUMENT, "plan_nested_meshes: need n_harmonics >= 2");
  if (n_w < 1) return set_error(FUSG_INVALID_ARGUMENT, "plan_nested_meshes: need n_w >= 1");
  if (d < 0.0) return set_error(FUSG_INVALID_ARGUMENT, "reference_domain: d must be >= 0");
  const double lambda1 = med->c0 / t->f0;
  const double focus[3] = {t->focal_length, 0.0, 0.0};
  const double l = t->focal_length, R = t->outer_radius;
  const double Lref = std::sqrt(l * l - R * R) - 0.1e-3;
  const double ref_lo_x = l - Lref;
  const double L = focus[0] - ref_lo_x;
  const double w = 2.0 * t->outer_radius * width_scale;
  const double d2lo[3] = {focus[0] - L, -w / 2.0, -w / 2.0};
  const double d2hi[3] = {focus[0] + d, w / 2.0, w / 2.0};
  fusg_grid ref{};
  fusg_status st = fusg_make_grid(d2lo, d2hi, lambda1 / (n_harmonics * n_w), n_harmonics, focus, &ref);
  if (st != FUSG_OK) return st;
  if (reference) *reference = ref;
  if (w_out) *w_out = w;
  for (int i = 2; i <= n_harmonics; ++i) {
    const double s = 2.0 / double(i);
    double lo[3] = {focus[0] - s * L, -s * w / 2.0, -s * w / 2.0};
    double hi[3] = {focus[0] + d, s * w / 2.0, s * w / 2.0};
    fusg_grid g{};
    if (single_mesh) {
      // plan_single_mesh: every harmonic on the reference mesh with the D_2 domain
      for (int a = 0; a < 3; ++a) {
        lo[a] = d2lo[a];
        hi[a] = d2hi[a];
      }
      g = ref;
      g.harmonic = i;
    } else {
      st = fusg_make_grid(lo, hi, lambda1 / (i * n_w), i, focus, &g);
      if (st != FUSG_OK) return st;
    }
    if (out_grids) out_grids[i - 2] = g;
    for (int a = 0; a < 3; ++a) {
      if (dlo) dlo[3 * (i - 2) + a] = lo[a];
      if (dhi) dhi[3 * (i - 2) + a] = hi[a];
    }
  }
  return FUSG_OK;
}

// src/cascade.cpp:32-34
double fusg_rhs_coefficient(const fusg_medium* m, double omega, int32_t n) {
  return m->beta * omega * omega * double(n) * double(n) / (2.0 * m->rho0 * std::pow(m->c0, 4));
}

// tests/acceptance.cpp:30-36
fusg_status fusg_random_vector(int64_t n, uint32_t seed, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int64_t i = 0; i < n; ++i) {
    const double re = u(rng);
    const double im = u(rng);
    out[2 * i] = re;
    out[2 * i + 1] = im;
  }
  return FUSG_OK;
}

}  // extern "C"
