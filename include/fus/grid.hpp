// fus drop-in: voxel grids, nested-mesh planner, transfer (reference: include/fus/grid.hpp,
// src/grid.cpp).  Host arithmetic is bit-identical to the reference; interpolate runs on the GPU.
#pragma once
#include <Eigen/Dense>
#include <optional>
#include <string>
#include <vector>

#include "fus/medium.hpp"

namespace fus {

struct BowlTransducer;

struct DomainBox {
  Eigen::Vector3d lo;
  Eigen::Vector3d hi;

  Eigen::Vector3d extent() const { return hi - lo; }
  bool contains(const Eigen::Vector3d& p, double tol = 0.0) const {
    for (int a = 0; a < 3; ++a)
      if (p[a] < lo[a] - tol || p[a] > hi[a] + tol) return false;
    return true;
  }
  bool contains(const DomainBox& other, double tol = 0.0) const {
    return contains(other.lo, tol) && contains(other.hi, tol);
  }
};

struct VoxelGrid {
  DomainBox box;
  double dx = 0.0;
  Eigen::Vector3i dims;
  int harmonic = 1;

  std::size_t count() const {
    return std::size_t(dims.x()) * std::size_t(dims.y()) * std::size_t(dims.z());
  }
  std::size_t index(int ix, int iy, int iz) const {
    return std::size_t(ix) + std::size_t(dims.x()) * (std::size_t(iy) + std::size_t(dims.y()) * iz);
  }
  Eigen::Vector3d center(int ix, int iy, int iz) const {
    return box.lo + Eigen::Vector3d((ix + 0.5) * dx, (iy + 0.5) * dx, (iz + 0.5) * dx);
  }
};

VoxelGrid make_grid(const DomainBox& request, double dx, int harmonic,
                    const std::optional<Eigen::Vector3d>& anchor = std::nullopt);

struct HarmonicField {
  VoxelGrid grid;
  Eigen::VectorXcd values;
  Wavenumber wavenumber;
};

struct PlannedGrid {
  int harmonic;
  DomainBox domain;
  VoxelGrid grid;
};

struct MeshPlan {
  std::vector<PlannedGrid> grids;
  VoxelGrid reference;
  double d = 0.0;
  double w = 0.0;
  Eigen::Vector3d focus;
  int n_w = 0;

  const PlannedGrid& for_harmonic(int n) const;  // std::out_of_range if absent
  double reduction_factor(int n) const;
  std::string report() const;
};

DomainBox reference_domain(const BowlTransducer& transducer, double d);
MeshPlan plan_nested_meshes(const BowlTransducer& transducer, const Medium& medium, double d,
                            int n_w, int n_harmonics, double width_scale = 1.0);
HarmonicField interpolate(const HarmonicField& field, const VoxelGrid& target);

}  // namespace fus
