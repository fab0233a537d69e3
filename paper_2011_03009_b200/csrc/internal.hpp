// Internal (non-ABI) declarations shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <map>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fusg.h"
#include "plan.hpp"

namespace fusg {

fusg_status set_error(fusg_status st, const std::string& msg);
fusg_status cuda_error(cudaError_t e, const char* what);

#define FUSG_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t e_ = (expr);                                  \
    if (e_ != cudaSuccess) return ::fusg::cuda_error(e_, #expr); \
  } while (0)

#define FUSG_TRY(expr)            \
  do {                            \
    fusg_status s_ = (expr);      \
    if (s_ != FUSG_OK) return s_; \
  } while (0)

// Reports the first launch error of the preceding kernel(s).
#define FUSG_LAUNCH_CHECK(what)                               \
  do {                                                        \
    cudaError_t e_ = cudaGetLastError();                      \
    if (e_ != cudaSuccess) return ::fusg::cuda_error(e_, what); \
  } while (0)

int smooth_padded_size(int n, bool pad_small_primes);
int device_padded_size(int n, int axis);  // the kernel's padded length on axis (z may prefer a warp length)
bool make_plan_radices(int L, AxisPlan& pl);

}  // namespace fusg

namespace fusg {
// Destinations of a fused-transpose store (sharded apply): the element
// (line i, outer k, position pos) of a pass goes to the rank q owning key = by_pos ? pos : i
// (ranks own contiguous key ranges starting at begin[q]) at
//   base[q] + off[q] + i * out_si + k * sk[q] + pos * out_sp.
// n = 0: plain store to the pass's own output.  Pass A keys by kx (into the owners' x-slabs),
// pass D by z (into the owners' A slabs); base[q] is the peer buffer (CUDA IPC mapping, or a
// buffer of another in-process rank for the loopback).
constexpr int kMaxPeers = 8;
struct PeerMap {
  int n = 0;
  int by_pos = 0;
  int begin[kMaxPeers] = {};
  double2* base[kMaxPeers] = {};
  int64_t off[kMaxPeers] = {};
  int64_t sk[kMaxPeers] = {};
#ifdef __CUDACC__
  __host__ __device__ __forceinline__ int owner(int key) const {
    int q = 0;
#pragma unroll
    for (int j = 1; j < kMaxPeers; ++j)
      if (j < n && key >= begin[j]) q = j;
    return q;
  }
#endif
};
}  // namespace fusg

struct fusg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int* dev_flag = nullptr;  // device error flag (monopole coincidence)
  double2* phase_tab = nullptr;  // e^{2 pi i j / 1024} / (4 pi), built on first use (fields.cu)
  std::atomic<uint64_t> launches{0};
  void* nccl = nullptr;  // ncclComm_t of a sharded job (fusg_ctx_attach_nccl)
  int nranks = 1, rank = 0;
  std::mutex mu;
  // twiddle tables e^{-2 pi i m / L} per padded length, uploaded once per context and shared by
  // its kernels (a build then needs no synchronous cudaMalloc / cudaMemcpy / cudaFree)
  std::map<int, double2*> tw_cache;
  std::mutex tw_mu;
  cudaStream_t pick(void* s) const { return s ? static_cast<cudaStream_t>(s) : stream; }
  // the owner's reference plus one per live kernel: a context outlives its kernels whatever
  // order their owners release them in (fusg_ctx_destroy drops the owner's reference)
  std::atomic<int> refs{1};
};

struct fusg_kernel {
  fusg_ctx* ctx = nullptr;
  fusg_grid grid{};
  fusg_wavenumber k{};
  int P[3] = {0, 0, 0};  // padded box
  int H[3] = {0, 0, 0};  // octant extents P/2 + 1
  fusg::AxisPlan plan[3]{};
  double2* tw[3] = {nullptr, nullptr, nullptr};
  double2* koct = nullptr;  // kernel spectrum octant [kx][ky][kz]  (Hx x Hy x Hz)
  // folded kx rows of the octant held here: [kf0, kf0 + knf) (unsharded: all Hx rows; slab
  // kernels keep only the rows their kx columns fold to, SURVEY.md 8(e) "octant per x-slab")
  int kf0 = 0, knf = 0;
  double2* bufA = nullptr;  // [kx][z][y]  (Px x Nz x Ny)
  double2* bufB = nullptr;  // [kx][ky][z]  (Px x Py x Nz)
  double2* stage_f = nullptr;  // host-vector apply staging (lazily allocated)
  double2* stage_u = nullptr;
  cudaStream_t copy_stream = nullptr;  // host-vector apply: chunked H2D / D2H beside the compute
  std::vector<cudaEvent_t> chunk_ev;   // one per z-chunk: copied in, then computed out
  void* ring = nullptr;                // fusg::PinnedRing for pageable host vectors (host_stage.hpp)
  // the workspace's last user: an apply on another stream waits for it (applies sharing one
  // kernel are ordered, as the reference's reentrant const apply is safe to call concurrently)
  cudaEvent_t last_ev = nullptr;
  cudaStream_t last_stream = nullptr;
  // slab decomposition (unsharded: G = 1, rank 0 owns everything)
  int G = 1, rank = 0;
  bool slab = false;   // created by fusg_kernel_create_slab: owns exchange buffers even at G = 1
  // layout of the x-transformed intermediate A (and X): [kx][z][y] (az = Ny, akx = Nz Ny), or
  // [z][kx][y] for unsharded kernels with FUSG_A_ZKY (az = Px Ny, akx = Ny)
  int64_t az = 0, akx = 0;
  // z pitch of the spectral intermediate B [kx][ky][z] (>= Nz): rounded up to 8 elements so every
  // ky row starts on a 128-byte line (FUSG_B_PITCH=0: Nz)
  int64_t bz = 0;
  int z0 = 0, nz = 0;  // this rank's z-planes of f/u
  int x0 = 0, nx = 0;  // this rank's spectral kx columns
  std::vector<int> zs, nzs, xs, nxs;  // all ranks' ranges (exchange offsets)
  double2* xbuf = nullptr;  // x-slab X [nx][Nz][Ny] (G > 1; aliases bufA when G = 1)
  double2* rbuf = nullptr;  // all-to-all staging [p][nx][nz_p][Ny] (G > 1)
  std::vector<int64_t> aoff, acnt, roff, rcnt;  // exchange plan (fusg_slab_exchange_plan)
  // fused peer-memory transposes: xbuf and bufA are cudaMalloc'd (IPC-exportable) for slab
  // kernels; peerX/peerA[q] = rank q's x-slab / A slab (own buffers for q == rank)
  bool ipc_bufs = false;
  std::vector<double2*> peerX, peerA;
  std::vector<bool> peer_opened;  // IPC mappings to close on destroy
  int* bar = nullptr;             // 1-int NCCL barrier buffer
  int* absync = nullptr;          // fused A+B pass: ticket and per-slab completion counters
  cudaStream_t ab_stream = nullptr;        // z-chunked A/B: pass-B stream (pass A on the caller's)
  std::vector<cudaEvent_t> ab_ev;          // [2 * chunk + 0]: A done, [2 * chunk + 1]: B done
  uint64_t bytes = 0;
  std::mutex mu;  // serialises applies sharing the workspace
};

namespace fusg {
void ctx_retain(fusg_ctx* ctx);
void ctx_release(fusg_ctx* ctx);  // frees the context with its last reference
// Function attributes are per device: run `set` once for each device this process uses
// (a mask over device ordinals 0..63; the current device is the one being launched on).
template <class F>
inline bool once_per_device(std::atomic<uint64_t>& mask, F&& set) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return set();
  const uint64_t bit = uint64_t(1) << dev;
  if (mask.load(std::memory_order_acquire) & bit) return true;
  if (!set()) return false;
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return true;
}
// Padded sizes, FFT plans, twiddles and the slab decomposition (G ranks, this is `rank`).
fusg_status kernel_init_geometry(fusg_kernel* K, int G, int rank);
void slab_split(int n, int G, int r, int* begin, int* count);
fusg_status volume_potential_build(fusg_kernel* K, double2 self);
fusg_status apply_phase_A(fusg_kernel* K, const double2* f, cudaStream_t s);
fusg_status apply_phase_BCD(fusg_kernel* K, double2* X, cudaStream_t s, cudaEvent_t* ev = nullptr);
fusg_status apply_phase_E(fusg_kernel* K, double2* u, double scale, cudaStream_t s);
// z-chunked unsharded apply (host-vector pipeline): planes [z0, z0 + nzc) of f (device pointer
// to plane z0) through passes A and B; pass C on the whole box; planes [z0, z0 + nzc) through
// passes D and E into u (device pointer to plane z0)
fusg_status apply_chunk_AB(fusg_kernel* K, const double2* f_z0, int z0, int nzc, cudaStream_t s);
fusg_status apply_phase_C(fusg_kernel* K, cudaStream_t s);
fusg_status apply_chunk_DE(fusg_kernel* K, double2* u_z0, int z0, int nzc, double scale, cudaStream_t s);
// fused peer-memory transposes (shard.cu): pass A storing into the x-slabs owned by each kx,
// passes B and C, pass D storing into the A slabs owned by each z
fusg_status apply_phase_A_peers(fusg_kernel* K, const double2* f, const PeerMap& pm, cudaStream_t s);
fusg_status apply_phase_BC(fusg_kernel* K, double2* X, cudaStream_t s);
fusg_status apply_phase_D_peers(fusg_kernel* K, const PeerMap& pm, cudaStream_t s);
void destroy_nccl(fusg_ctx* ctx);
// ev (optional): 6 events recorded before passes A..E and after E
fusg_status volume_potential_apply(fusg_kernel* K, const double2* f, double2* u, double scale,
                                   cudaStream_t st, cudaEvent_t* ev = nullptr);
}  // namespace fusg

namespace fusg {
// device helpers of fields.cu / api.cu shared by the cascades (api.cu, vie.cu)
fusg_status upload_sources(const double* src_host, int n_src, double** dev, cudaStream_t s);
fusg_status monopole_grid(fusg_ctx* ctx, const double* src_dev, int n_src, const fusg_grid& g,
                          double kre, double kim, double amp, double2* out, cudaStream_t s,
                          double dmax, int z0 = 0, int nz = -1);
double distance_bound(const double* src_host, int n_src, const double lo[3], const double hi[3]);
fusg_status interpolate_dev(fusg_ctx* ctx, const fusg_grid& src, const double2* f,
                            const fusg_grid& tgt, double2* out, cudaStream_t s);
fusg_status rhs_dev(fusg_ctx* ctx, int n, const double2* const* lower, int64_t count, double coeff,
                    double2* out, cudaStream_t s);
fusg_status max_abs_dev(fusg_ctx* ctx, const double2* v, int64_t n, double* out, cudaStream_t s);
fusg_status radiated_power_dev(fusg_ctx* ctx, const double* src_dev, int n_src, double x_disc,
                               double R, double kre, double kim, double amp, double rho0, double c0,
                               int n_r, int n_theta, double* out_host, cudaStream_t s, double dmax);
fusg_status check_monopole_flag(fusg_ctx* ctx, cudaStream_t s);
fusg_status source_field_dev(fusg_ctx* ctx, const fusg_bowl& t, const fusg_medium& med, const double* src,
                             const fusg_grid& grid, double2* out, fusg_wavenumber* k1, double* norm,
                             double* amp1, cudaStream_t s);
}  // namespace fusg
