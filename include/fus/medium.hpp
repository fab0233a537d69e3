// fus drop-in: medium and wavenumbers (reference: include/fus/medium.hpp, src/medium.cpp).
// Implemented over the C-ABI in include/fusg.h (libfus.so -> libfusg.so).
#pragma once
#include <complex>
#include <string>
#include <vector>

namespace fus {

/// Acoustic constants with power-law attenuation alpha0 * (f / MHz)^eta dB/m.
struct Medium {
  std::string name;
  double rho0;
  double c0;
  double beta;
  double alpha0;
  double eta;

  // Throws std::invalid_argument for non-physical constants; returns warnings otherwise.
  std::vector<std::string> validate() const;
};

/// k = n omega / c0 + i alpha(n f0)
struct Wavenumber {
  std::complex<double> k;
  int harmonic;
  double omega;
};

inline constexpr double kDbPerNeper = 8.685889638065035;

double attenuation_np_per_m(const Medium& medium, double f_hz);
Wavenumber complex_wavenumber(const Medium& medium, double f0, int n);
Medium medium_preset(const std::string& name);
bool is_medium_preset(const std::string& name);
// key=value config file with keys name, rho0, c0, beta, alpha0, eta (src/medium.cpp:58-69)
Medium load_medium(const std::string& path);

}  // namespace fus
