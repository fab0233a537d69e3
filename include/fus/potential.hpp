// fus drop-in: volume potential (reference: include/fus/potential.hpp, src/potential.cpp).
// GreenKernel keeps its spectrum on the GPU (octant of the even kernel, libfusg.so); copies
// share it.  apply() takes and returns host vectors like the reference; apply_device() is the
// device-resident variant.
#pragma once
#include <Eigen/Dense>
#include <complex>
#include <memory>
#include <vector>

#include "fus/grid.hpp"
#include "fus/medium.hpp"

struct fusg_kernel;

namespace fus {

std::complex<double> green_function(const Eigen::Vector3d& x, const Eigen::Vector3d& y,
                                    const Wavenumber& k);
std::complex<double> self_weight(const Wavenumber& k, double delta_x);
double equivalent_sphere_radius(double delta_x);

class GreenKernel {
 public:
  GreenKernel(const VoxelGrid& grid, const Wavenumber& k, bool pad_small_primes = false);

  Eigen::VectorXcd apply(const Eigen::VectorXcd& f) const;
  HarmonicField apply(const HarmonicField& f) const;
  // u = scale * apply(f) on device pointers (N complex128 each), on `stream` (nullptr: default).
  void apply_device(const std::complex<double>* f, std::complex<double>* u, double scale = 1.0,
                    void* stream = nullptr) const;

  const VoxelGrid& grid() const { return grid_; }
  const Wavenumber& wavenumber() const { return k_; }
  Eigen::Vector3i padded() const;
  // the device kernel (C-ABI handle) behind this GreenKernel
  fusg_kernel* native() const { return handle_.get(); }

 private:
  VoxelGrid grid_;
  Wavenumber k_;
  std::shared_ptr<fusg_kernel> handle_;
};

// Off-grid potential (src/potential.cpp:161-201): sum over voxels of vol G(|x - c_j|) f_j
// (self weight for |x - c_j| < 1e-9 dx, zero-f voxels skipped) at each point; on the GPU.
Eigen::VectorXcd evaluate_potential_at(const Wavenumber& k, const VoxelGrid& grid,
                                       const Eigen::VectorXcd& f,
                                       const std::vector<Eigen::Vector3d>& points);
// The O(N^2) quadrature the FFT path is checked against (src/potential.cpp:203-238), guarded to
// grids of at most 1e5 voxels; here it runs on the device (the off-grid kernel at every voxel
// centre, where the coincident point takes the self term).
Eigen::VectorXcd direct_potential_oracle(const Wavenumber& k, const VoxelGrid& grid,
                                         const Eigen::VectorXcd& f);

}  // namespace fus
