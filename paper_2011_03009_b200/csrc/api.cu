// C-ABI entry points for the device context, the GreenKernel (volume potential) and the
// device-resident harmonic recursion (run_cascade, src/cascade.cpp:42-107).
#include <chrono>
#include <cstring>
#include <iostream>
#include <memory>
#include <vector>

#include "internal.hpp"
#include "host_stage.hpp"


namespace fusg {
void ctx_retain(fusg_ctx* ctx) { ctx->refs.fetch_add(1); }

void ctx_release(fusg_ctx* ctx) {
  if (ctx->refs.fetch_sub(1) != 1) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  destroy_nccl(ctx);
  cudaFree(ctx->dev_flag);
  if (ctx->phase_tab) cudaFree(ctx->phase_tab);
  for (auto& kv : ctx->tw_cache) cudaFree(kv.second);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

}  // namespace fusg

using namespace fusg;

namespace {

int64_t count_of(const fusg_grid& g) { return int64_t(g.dims[0]) * g.dims[1] * g.dims[2]; }

bool same_grid(const fusg_grid& a, const fusg_grid& b) {  // src/cascade.cpp:15-17
  return a.dims[0] == b.dims[0] && a.dims[1] == b.dims[1] && a.dims[2] == b.dims[2] &&
         a.dx == b.dx && a.lo[0] == b.lo[0] && a.lo[1] == b.lo[1] && a.lo[2] == b.lo[2];
}

// Kernel workspaces come from the context's stream-ordered pool; work on other streams
// using this kernel must be complete before destruction (as with any GreenKernel owner).
void free_kernel(fusg_kernel* K) {
  if (!K) return;
  cudaSetDevice(K->ctx->device);
  cudaStream_t s = K->ctx->stream;
  for (size_t q = 0; q < K->peer_opened.size(); ++q)
    if (K->peer_opened[q]) {
      cudaIpcCloseMemHandle(K->peerX[q]);
      cudaIpcCloseMemHandle(K->peerA[q]);
    }
  if (K->bar) cudaFree(K->bar);
  if (K->absync) cudaFree(K->absync);
  for (cudaEvent_t e : K->ab_ev) cudaEventDestroy(e);
  if (K->ab_stream) cudaStreamDestroy(K->ab_stream);
  if (K->ipc_bufs) {
    cudaStreamSynchronize(s);
    cudaFree(K->bufA);
    if (K->xbuf) cudaFree(K->xbuf);
  } else {
    cudaFreeAsync(K->bufA, s);
    if (K->xbuf) cudaFreeAsync(K->xbuf, s);
  }
  cudaFreeAsync(K->bufB, s);
  cudaFreeAsync(K->koct, s);
  if (K->rbuf) cudaFreeAsync(K->rbuf, s);
  if (K->stage_f) cudaFree(K->stage_f);
  if (K->stage_u) cudaFree(K->stage_u);
  if (K->ring) {
    static_cast<PinnedRing*>(K->ring)->destroy();
    delete static_cast<PinnedRing*>(K->ring);
  }
  if (K->last_ev) cudaEventDestroy(K->last_ev);
  for (cudaEvent_t e : K->chunk_ev) cudaEventDestroy(e);
  if (K->copy_stream) cudaStreamDestroy(K->copy_stream);
  fusg_ctx* ctx = K->ctx;
  delete K;  // (twiddle tables belong to the context's cache)
  ctx_release(ctx);
}

// Applies of one kernel share its workspace: an apply enqueued on a stream other than the last
// user's waits for the last user's work (an event), then records its own.  Callers hold K->mu.
cudaError_t workspace_acquire(fusg_kernel* K, cudaStream_t s) {
  if (!K->last_ev) {
    cudaError_t e = cudaEventCreateWithFlags(&K->last_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  } else if (K->last_stream != s) {
    cudaError_t e = cudaStreamWaitEvent(s, K->last_ev, 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
cudaError_t workspace_release(fusg_kernel* K, cudaStream_t s) {
  K->last_stream = s;
  return cudaEventRecord(K->last_ev, s);
}

// CUDA-event stopwatch on a stream
struct EvTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit EvTimer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~EvTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  void start() { cudaEventRecord(a, s); }
  double stop() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
  }
};

}  // namespace

namespace fusg {
// evaluate_source_field (src/transducer.cpp:198-206) into out on `grid`, sources already on
// the device: power normalisation (power_scale_factor, :157-163) then the monopole sum, with
// the coincidence check.  Returns k1, the normalisation (1 when power = 0) and the amplitude.
fusg_status source_field_dev(fusg_ctx* ctx, const fusg_bowl& t, const fusg_medium& med, const double* src,
                             const fusg_grid& grid, double2* out, fusg_wavenumber* k1, double* norm,
                             double* amp1, cudaStream_t s) {
  const double l = t.focal_length, R = t.outer_radius;
  const double cap_area = 2.0 * M_PI * l * (l - std::sqrt(l * l - R * R));
  const double x_disc = l - std::sqrt(l * l - R * R);
  FUSG_TRY(fusg_complex_wavenumber(&med, t.f0, 1, k1));
  double scale = 0.0;
  if (t.power != 0.0) {
    double pw = 0.0;
    const double dlo[3] = {x_disc, -R, -R}, dhi[3] = {x_disc, R, R};
    FUSG_TRY(radiated_power_dev(ctx, src, t.n_points, x_disc, R, k1->k_re, k1->k_im,
                                1.0 * cap_area / double(t.n_points), med.rho0, med.c0, 384, 256, &pw, s,
                                distance_bound(t.points_host, t.n_points, dlo, dhi)));
    if (pw <= 0.0) return set_error(FUSG_RUNTIME, "power normalization: degenerate field, Pi(p) = 0");
    scale = std::sqrt(t.power / pw);
  }
  *norm = scale > 0.0 ? scale : 1.0;
  *amp1 = scale * cap_area / double(t.n_points);
  FUSG_TRY(monopole_grid(ctx, src, t.n_points, grid, k1->k_re, k1->k_im, *amp1, out, s,
                         distance_bound(t.points_host, t.n_points, grid.lo, grid.hi)));
  return check_monopole_flag(ctx, s);
}
}  // namespace fusg

extern "C" {

fusg_status fusg_ctx_create(int32_t device, fusg_ctx** out) {
  if (!out) return set_error(FUSG_INVALID_ARGUMENT, "ctx_create: null out");
  int n = 0;
  FUSG_CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return set_error(FUSG_INVALID_ARGUMENT, "ctx_create: no such device");
  FUSG_CUDA_TRY(cudaSetDevice(device));
  auto ctx = std::make_unique<fusg_ctx>();
  ctx->device = device;
  FUSG_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  FUSG_CUDA_TRY(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
  FUSG_CUDA_TRY(cudaMalloc(&ctx->dev_flag, sizeof(int)));
  {  // keep freed stream-ordered memory in the pool (kernels/cascade temporaries are reused)
    cudaMemPool_t pool;
    FUSG_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    FUSG_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  }
  FUSG_CUDA_TRY(cudaMemset(ctx->dev_flag, 0, sizeof(int)));
  *out = ctx.release();
  return FUSG_OK;
}

fusg_status fusg_ctx_destroy(fusg_ctx* ctx) {
  if (ctx) ctx_release(ctx);
  return FUSG_OK;
}

void* fusg_ctx_stream(fusg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

fusg_status fusg_ctx_synchronize(fusg_ctx* ctx) {
  if (!ctx) return set_error(FUSG_INVALID_ARGUMENT, "ctx_synchronize: null ctx");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  FUSG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return FUSG_OK;
}

uint64_t fusg_ctx_launch_count(fusg_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

// GreenKernel::GreenKernel (src/potential.cpp:72-118)
fusg_status fusg_kernel_create(fusg_ctx* ctx, const fusg_grid* grid, const fusg_wavenumber* k,
                               int32_t pad_small_primes, fusg_kernel** out) {
  if (!ctx || !grid || !k || !out) return set_error(FUSG_INVALID_ARGUMENT, "kernel_create: null argument");
  for (int a = 0; a < 3; ++a)
    if (grid->dims[a] < 1) return set_error(FUSG_INVALID_ARGUMENT, "kernel_create: empty grid");
  if (grid->dx <= 0.0) return set_error(FUSG_INVALID_ARGUMENT, "self_weight: delta_x must be positive");
  (void)pad_small_primes;  // any smooth P >= 2N-1 is the same operator; see fusg_padded_dims
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  double w0[2];
  fusg_status st = fusg_self_weight(k, grid->dx, w0);
  if (st != FUSG_OK) return st;
  auto* K = new fusg_kernel;
  K->ctx = ctx;
  ctx_retain(ctx);
  K->grid = *grid;
  K->k = *k;
  st = kernel_init_geometry(K, 1, 0);
  if (st == FUSG_OK) st = volume_potential_build(K, make_double2(w0[0], w0[1]));
  if (st != FUSG_OK) {
    free_kernel(K);
    return st;
  }
  *out = K;
  return FUSG_OK;
}

fusg_status fusg_kernel_destroy(fusg_kernel* K) {
  free_kernel(K);
  return FUSG_OK;
}

fusg_status fusg_kernel_padded(const fusg_kernel* K, int32_t out[3]) {
  if (!K) return set_error(FUSG_INVALID_ARGUMENT, "kernel_padded: null kernel");
  for (int a = 0; a < 3; ++a) out[a] = K->P[a];
  return FUSG_OK;
}

uint64_t fusg_kernel_device_bytes(const fusg_kernel* K) { return K ? K->bytes : 0; }

// GreenKernel::apply (src/potential.cpp:120-151)
fusg_status fusg_kernel_apply(fusg_kernel* K, const double* f_dev, double* u_dev, double scale,
                              void* stream) {
  if (!K || !f_dev || !u_dev) return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply: null argument");
  if (static_cast<const void*>(f_dev) == static_cast<const void*>(u_dev))
    return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply: output aliases input");
  FUSG_CUDA_TRY(cudaSetDevice(K->ctx->device));
  std::lock_guard<std::mutex> lock(K->mu);
  cudaStream_t s = K->ctx->pick(stream);
  FUSG_CUDA_TRY(workspace_acquire(K, s));
  fusg_status st = volume_potential_apply(K, reinterpret_cast<const double2*>(f_dev),
                                          reinterpret_cast<double2*>(u_dev), scale, s);
  FUSG_CUDA_TRY(workspace_release(K, s));
  return st;
}

fusg_status fusg_kernel_apply_timed(fusg_kernel* K, const double* f_dev, double* u_dev,
                                    double scale, int32_t reps, double pass_ms[5]) {
  if (!K || !f_dev || !u_dev || !pass_ms || reps < 1)
    return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply_timed: bad argument");
  FUSG_CUDA_TRY(cudaSetDevice(K->ctx->device));
  std::lock_guard<std::mutex> lock(K->mu);
  cudaStream_t s = K->ctx->stream;
  FUSG_CUDA_TRY(workspace_acquire(K, s));
  std::vector<cudaEvent_t> ev(6 * size_t(reps));
  for (auto& e : ev) FUSG_CUDA_TRY(cudaEventCreate(&e));
  fusg_status st = FUSG_OK;
  for (int r = 0; r < reps && st == FUSG_OK; ++r)
    st = volume_potential_apply(K, reinterpret_cast<const double2*>(f_dev),
                                reinterpret_cast<double2*>(u_dev), scale, s, &ev[6 * size_t(r)]);
  if (st == FUSG_OK) {
    FUSG_CUDA_TRY(cudaStreamSynchronize(s));
    for (int p = 0; p < 5; ++p) {
      double acc = 0.0;
      for (int r = 0; r < reps; ++r) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[6 * size_t(r) + p], ev[6 * size_t(r) + p + 1]);
        acc += ms;
      }
      pass_ms[p] = acc / reps;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  FUSG_CUDA_TRY(workspace_release(K, s));
  return st;
}

fusg_status fusg_kernel_apply_host(fusg_kernel* K, const double* f_host, double* u_host,
                                   double scale) {
  if (!K || !f_host || !u_host) return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply: null argument");
  if (K->G != 1) return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply_host: sharded kernel needs a slab apply");
  FUSG_CUDA_TRY(cudaSetDevice(K->ctx->device));
  const size_t bytes = size_t(count_of(K->grid)) * 16;
  cudaStream_t s = K->ctx->stream;
  std::lock_guard<std::mutex> lock(K->mu);
  if (!K->stage_f || !K->stage_u) {  // device staging for host-vector applies, allocated once per kernel
    if (K->stage_f) cudaFree(K->stage_f);
    if (K->stage_u) cudaFree(K->stage_u);
    K->stage_f = K->stage_u = nullptr;
    if (cudaMalloc(&K->stage_f, bytes) != cudaSuccess || cudaMalloc(&K->stage_u, bytes) != cudaSuccess) {
      cudaGetLastError();
      if (K->stage_f) cudaFree(K->stage_f);
      K->stage_f = K->stage_u = nullptr;
      return set_error(FUSG_OOM, "kernel_apply_host: staging allocation failed");
    }
    K->bytes += 2 * bytes;
  }
  // Pageable host vectors (the VectorXcd case) go through the library's pinned staging ring;
  // pinned ones are copied directly.
  const bool pinned = host_pinned(f_host) && host_pinned(u_host);
  PinnedRing* ring = nullptr;
  if (!pinned) {
    if (!K->ring) {
      auto* r = new PinnedRing;
      // FUSG_HOST_THREADS: copy threads (default: every hardware thread, up to 32);
      // FUSG_HOST_SLOT_MB / FUSG_HOST_SLOTS: pinned slot size and count (16 MB x 3)
      const char* env_t = getenv("FUSG_HOST_THREADS");
      const char* env_s = getenv("FUSG_HOST_SLOT_MB");
      const int hw = int(std::thread::hardware_concurrency());
      const int nt = env_t ? std::max(1, atoi(env_t)) : std::max(1, std::min(32, hw));
      // 3 slots of 16 MB: a thread's 1 MB share of a slot is still in the host caches when the
      // DMA reads it, and the ring (48 MB) stays inside the box's 60 MB L3 (cfg5 pageable apply:
      // 4 x 64 MB 368-414 ms, 4 x 16 MB 308-389 ms, 3 x 16 MB 307-312 ms, 4 x 4 MB 458 ms;
      // pinned buffers 287 ms)
      const size_t slot_mb = env_s ? size_t(std::max(1, atoi(env_s))) : 16;
      const char* env_n = getenv("FUSG_HOST_SLOTS");
      const int nslots = env_n ? std::max(2, atoi(env_n)) : 3;
      if (r->init(nslots, slot_mb << 20, nt) != cudaSuccess) {
        cudaGetLastError();
        r->destroy();
        delete r;
        return set_error(FUSG_OOM, "kernel_apply_host: pinned staging allocation failed");
      }
      K->ring = r;
    }
    ring = static_cast<PinnedRing*>(K->ring);
  }
  // z-chunk pipeline: chunk c is copied in on the copy stream while the compute stream runs
  // passes A+B on chunk c-1; after pass C, passes D+E of chunk c overlap the copy-out of c-1.
  const int Nz = K->grid.dims[2];
  const size_t plane = bytes / size_t(Nz);
  // FUSG_HOST_CHUNKS overrides the chunk count (any size); default 8 above 8 MB, else 1
  const char* env_chunks = getenv("FUSG_HOST_CHUNKS");
  const int nchunks = env_chunks ? std::min(std::max(1, atoi(env_chunks)), Nz)
                                 : (bytes < (size_t(8) << 20) ? 1 : std::min(8, Nz));
  if (!K->copy_stream) FUSG_CUDA_TRY(cudaStreamCreateWithFlags(&K->copy_stream, cudaStreamNonBlocking));
  while (int(K->chunk_ev.size()) < 2 * nchunks + 1) {
    cudaEvent_t e;
    FUSG_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    K->chunk_ev.push_back(e);
  }
  FUSG_CUDA_TRY(workspace_acquire(K, s));
  cudaStream_t cs = K->copy_stream;
  auto z_of = [&](int c) { return int(int64_t(Nz) * c / nchunks); };
  auto* hf = reinterpret_cast<const char*>(f_host);
  auto* hu = reinterpret_cast<char*>(u_host);
  auto* df = reinterpret_cast<char*>(K->stage_f);
  auto* du = reinterpret_cast<char*>(K->stage_u);
  // the copy stream starts after the compute stream's earlier work (a previous apply's reads of
  // the staging buffers)
  FUSG_CUDA_TRY(cudaEventRecord(K->chunk_ev[2 * nchunks], s));
  FUSG_CUDA_TRY(cudaStreamWaitEvent(cs, K->chunk_ev[2 * nchunks], 0));
  fusg_status st = FUSG_OK;
  // host -> device, chunk by chunk; with the ring the host thread stages chunk c + 1 while the
  // device computes passes A+B of chunk c, so the compute launches are interleaved with it
  for (int c = 0; c < nchunks && st == FUSG_OK; ++c) {
    const int z0 = z_of(c), nzc = z_of(c + 1) - z0;
    if (ring)
      FUSG_CUDA_TRY(ring->h2d(df + z0 * plane, hf + z0 * plane, nzc * plane, cs));
    else
      FUSG_CUDA_TRY(cudaMemcpyAsync(df + z0 * plane, hf + z0 * plane, nzc * plane, cudaMemcpyHostToDevice, cs));
    FUSG_CUDA_TRY(cudaEventRecord(K->chunk_ev[c], cs));
    FUSG_CUDA_TRY(cudaStreamWaitEvent(s, K->chunk_ev[c], 0));
    st = apply_chunk_AB(K, K->stage_f + int64_t(z0) * (plane / 16), z0, nzc, s);
  }
  if (st == FUSG_OK) st = apply_phase_C(K, s);
  for (int c = 0; c < nchunks && st == FUSG_OK; ++c) {
    const int z0 = z_of(c), nzc = z_of(c + 1) - z0;
    st = apply_chunk_DE(K, K->stage_u + int64_t(z0) * (plane / 16), z0, nzc, scale, s);
    if (st != FUSG_OK) break;
    FUSG_CUDA_TRY(cudaEventRecord(K->chunk_ev[nchunks + c], s));
    FUSG_CUDA_TRY(cudaStreamWaitEvent(cs, K->chunk_ev[nchunks + c], 0));
    if (!ring)
      FUSG_CUDA_TRY(cudaMemcpyAsync(hu + z0 * plane, du + z0 * plane, nzc * plane, cudaMemcpyDeviceToHost, cs));
  }
  // with the ring the host drains chunk by chunk (each chunk's DMA waits for its passes D+E)
  for (int c = 0; ring && c < nchunks && st == FUSG_OK; ++c) {
    const int z0 = z_of(c), nzc = z_of(c + 1) - z0;
    FUSG_CUDA_TRY(ring->d2h(hu + z0 * plane, du + z0 * plane, nzc * plane, cs));
  }
  // the compute stream's later work must not overwrite the staging buffers under the copies
  FUSG_CUDA_TRY(cudaEventRecord(K->chunk_ev[2 * nchunks], cs));
  FUSG_CUDA_TRY(cudaStreamWaitEvent(s, K->chunk_ev[2 * nchunks], 0));
  FUSG_CUDA_TRY(workspace_release(K, s));
  FUSG_CUDA_TRY(cudaStreamSynchronize(cs));
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return st;
}

// run_cascade (src/cascade.cpp:42-107), device resident.
fusg_status fusg_run_cascade(fusg_ctx* ctx, const fusg_cascade_desc* d, double* const* out_dev,
                             fusg_stage_timing* timings, double* source_normalization) {
  if (!ctx || !d || !out_dev) return set_error(FUSG_INVALID_ARGUMENT, "run_cascade: null argument");
  const int n = d->n_harmonics;
  if (n < 2) return set_error(FUSG_INVALID_ARGUMENT, "run_cascade: n_harmonics must be >= 2");
  if (!d->grids) return set_error(FUSG_INVALID_ARGUMENT, "run_cascade: no planned grids");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const fusg_bowl& t = d->transducer;
  const fusg_medium& med = d->medium;
  auto grid_of = [&](int harmonic) -> const fusg_grid& {  // p1 lives on D_2's grid
    return d->grids[harmonic <= 2 ? 0 : harmonic - 2];
  };

  double* src = nullptr;
  fusg_status st = upload_sources(t.points_host, t.n_points, &src, s);
  if (st != FUSG_OK) return st;
  std::unique_ptr<double, void (*)(double*)> src_guard(src, [](double* p) { cudaFree(p); });

  // Reserve the stream-ordered pool once for the largest stage (its kernel's buffers, the
  // lower fields brought onto its grid and its source term): the per-harmonic allocations then
  // come from memory the pool already maps, instead of growing it (and stalling) stage by stage.
  {
    size_t peak = 0;
    for (int i = 2; i <= n; ++i) {
      const fusg_grid& gi = grid_of(i);
      size_t P[3], H[3];
      for (int a = 0; a < 3; ++a) {
        P[a] = size_t(fusg::device_padded_size(gi.dims[a], a));
        H[a] = P[a] / 2 + 1;
      }
      const size_t cnt = size_t(count_of(gi));
      const size_t e = P[0] * gi.dims[1] * gi.dims[2] + P[0] * P[1] * gi.dims[2] + H[0] * H[1] * H[2] + size_t(i) * cnt;
      peak = std::max(peak, e * 16);
    }
    void* r = nullptr;
    if (cudaMallocAsync(&r, peak + peak / 8, s) == cudaSuccess) cudaFreeAsync(r, s);
    cudaGetLastError();
  }

  // p1 on the D_2 grid: evaluate_source_field (src/transducer.cpp:198-206)
  EvTimer tm(s);
  tm.start();
  fusg_wavenumber k1{};
  double norm = 1.0, amp1 = 0.0;
  st = source_field_dev(ctx, t, med, src, grid_of(1), reinterpret_cast<double2*>(out_dev[0]), &k1, &norm,
                        &amp1, s);
  if (st != FUSG_OK) return st;
  if (source_normalization) *source_normalization = norm;
  const double p1_s = tm.stop();
  double peak = 0.0;
  st = max_abs_dev(ctx, reinterpret_cast<const double2*>(out_dev[0]), count_of(grid_of(1)), &peak, s);
  if (st != FUSG_OK) return st;
  if (peak > 15e6)
    std::cerr << "warning: peak pressure " << peak / 1e6
              << " MPa exceeds the 15 MPa weakly-nonlinear bound; the truncated cascade"
                 " may be inaccurate\n";

  for (int i = 2; i <= n; ++i) {
    fusg_stage_timing row{};
    row.harmonic = i;
    auto t0 = std::chrono::steady_clock::now();
    const fusg_grid& grid = grid_of(i);
    const int64_t count = count_of(grid);
    row.voxels = uint64_t(count);
    row.meshing_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (i == 2) row.p1_s = p1_s;

    // bring p_1 .. p_{i-1} onto this grid
    tm.start();
    std::vector<double2*> temps;
    std::vector<const double2*> lower;
    for (int m = 1; m <= i - 1; ++m) {
      const fusg_grid& gm = grid_of(m);
      const double2* pm = reinterpret_cast<const double2*>(out_dev[m - 1]);
      if (same_grid(gm, grid)) {
        lower.push_back(pm);
        continue;
      }
      double2* tmp = nullptr;
      if (cudaMallocAsync(&tmp, size_t(count) * 16, s) != cudaSuccess) {
        for (auto* p : temps) cudaFreeAsync(p, s);
        cudaGetLastError();
        return set_error(FUSG_OOM, "run_cascade: temporary field allocation failed");
      }
      temps.push_back(tmp);
      if (m == 1 && d->recompute_p1_each_grid)
        st = monopole_grid(ctx, src, t.n_points, grid, k1.k_re, k1.k_im, amp1, tmp, s,
                           distance_bound(t.points_host, t.n_points, grid.lo, grid.hi));
      else
        st = interpolate_dev(ctx, gm, pm, grid, tmp, s);
      if (st != FUSG_OK) break;
      lower.push_back(tmp);
    }
    if (st == FUSG_OK) row.interpolation_s = tm.stop();

    // rhs_source (untimed in the reference; timed separately here)
    fusg_wavenumber ki{};
    double2* f = nullptr;
    if (st == FUSG_OK) st = fusg_complex_wavenumber(&med, t.f0, i, &ki);
    if (st == FUSG_OK) {
      if (cudaMallocAsync(&f, size_t(count) * 16, s) != cudaSuccess) {
        cudaGetLastError();
        st = set_error(FUSG_OOM, "run_cascade: source allocation failed");
      } else {
        cudaStreamSynchronize(s);  // keep first-touch pool growth out of the rhs timing
        tm.start();
        st = rhs_dev(ctx, i, lower.data(), count, fusg_rhs_coefficient(&med, ki.omega, i), f, s);
        if (st == FUSG_OK) row.rhs_s = tm.stop();
      }
    }
    for (auto* p : temps) cudaFreeAsync(p, s);

    // GreenKernel(grid_i, k_i) -> "Evaluate G_k"
    fusg_kernel* K = nullptr;
    if (st == FUSG_OK) {
      tm.start();
      fusg_grid gi = grid;
      gi.harmonic = i;
      st = fusg_kernel_create(ctx, &gi, &ki, d->pad_small_primes, &K);
      if (st == FUSG_OK) row.kernel_s = tm.stop();
    }
    // p_i = -apply(f)
    if (st == FUSG_OK) {
      tm.start();
      st = volume_potential_apply(K, f, reinterpret_cast<double2*>(out_dev[i - 1]), -1.0, s);
      if (st == FUSG_OK) row.potential_s = tm.stop();
    }
    if (f) cudaFreeAsync(f, s);
    if (K) fusg_kernel_destroy(K);
    if (st != FUSG_OK) return st;
    if (timings) timings[i - 2] = row;
  }
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return FUSG_OK;
}

}  // extern "C"
