// Internal helpers of the fus C++ shim (fus_api.cpp, fus_vie.cpp): status -> exception
// mapping, the shared context, device buffers and C-ABI struct conversions.
#pragma once
#include <cuda_runtime.h>

#include <Eigen/Dense>
#include <string>
#include <vector>

#include "fus/grid.hpp"
#include "fus/medium.hpp"
#include "fus/transducer.hpp"
#include "fusg.h"

namespace fus {
namespace detail {

void check(fusg_status st);
void cuda_check(cudaError_t e, const char* what);
fusg_ctx* ctx();

// RAII device buffer
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  double* d() const { return static_cast<double*>(p); }
};

DevBuf upload(const Eigen::VectorXcd& v);
Eigen::VectorXcd download(const DevBuf& b, size_t n);
fusg_grid to_c(const VoxelGrid& g);
VoxelGrid from_c(const fusg_grid& c);
fusg_wavenumber to_c(const Wavenumber& k);
fusg_medium to_c(const Medium& m);
std::vector<double> flat_points(const std::vector<Eigen::Vector3d>& pts);

struct BowlC {
  std::vector<double> pts;
  fusg_bowl c{};
  explicit BowlC(const BowlTransducer& t) : pts(flat_points(t.source_points)) {
    c = {t.f0, t.focal_length, t.outer_radius, t.power, int32_t(t.source_points.size()), pts.data()};
  }
};

}  // namespace detail
}  // namespace fus
