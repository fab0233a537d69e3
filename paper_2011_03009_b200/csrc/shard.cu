// Slab-sharded volume-potential apply: one exchange step each way.
//
// Rank r of G owns z-planes [z0_r, z0_r + nz_r) of f/u and spectral kx columns [x0_r, x0_r + nx_r).
//   phase A on the z-slab writes A_r [Px][nz_r][Ny]; A_r's kx-range slices ARE the send blocks
//   exchange 1: rank r receives [nx_r][nz_p][Ny] from every p into rbuf, unpacked (2D copy) into
//              the x-slab X_r [nx_r][Nz][Ny]
//   phases B, C, D run locally on X_r (K^ octant rows held per x-slab: the folded kx window
//              [kf0, kf0 + knf) of this rank's columns, built without a collective)
//   exchange 2: X_r rows of z-slab q are packed (2D copy) into rbuf and sent to q, which
//              receives them straight into its A_q kx-slice
//   phase E on the z-slab.
// Transports: NCCL grouped send/recv (one process per GPU; NCCL 2.27 has no ncclAlltoAll) and a
// loopback that runs every rank of the decomposition in one process on one device, exchanging
// with device copies — the same blocks, offsets and kernels, so G = 2/4/8 decompositions are
// testable on a single GPU and must reproduce the unsharded apply bit for bit.
#include <nccl.h>

#include <cstring>
#include <vector>

#include "internal.hpp"

namespace fusg {
namespace {

constexpr size_t kC = sizeof(double2);

int64_t row(const fusg_kernel* K) { return K->grid.dims[1]; }  // Ny: elements per (kx, z) row

// The all-to-all staging buffer [p][nx][nz_p][Ny] of the NCCL transport, allocated on first use.
fusg_status ensure_rbuf(fusg_kernel* K, cudaStream_t s) {
  if (K->rbuf) return FUSG_OK;
  const size_t n = size_t(K->nx) * K->grid.dims[2] * K->grid.dims[1];
  if (cudaMallocAsync(&K->rbuf, std::max<size_t>(n, 1) * sizeof(double2), s) != cudaSuccess) {
    cudaGetLastError();
    K->rbuf = nullptr;
    return set_error(FUSG_OOM, "slab apply: exchange buffer allocation failed");
  }
  K->bytes += n * sizeof(double2);
  return FUSG_OK;
}

// The exchange plan (element offsets/counts per peer), shared by the NCCL and loopback
// transports and exported as fusg_slab_exchange_plan:
//   a_off/a_cnt[q]: block of A_r [Px][nz_r][Ny] holding rank q's kx columns (send in exchange 1,
//                   receive in exchange 2) = [x0_q, x0_q + nx_q) x nz_r x Ny
//   r_off/r_cnt[p]: block of rbuf [p][nx_r][nz_p][Ny] from/to rank p (receive in exchange 1,
//                   send in exchange 2) = nx_r x [z0_p, z0_p + nz_p) x Ny
void exchange_plan(const int dims[3], int Px, int G, int r, int64_t* aoff, int64_t* acnt, int64_t* roff,
                   int64_t* rcnt) {
  int z0r, nzr, x0r, nxr;
  slab_split(dims[2], G, r, &z0r, &nzr);
  slab_split(Px, G, r, &x0r, &nxr);
  const int64_t Ny = dims[1];
  for (int q = 0; q < G; ++q) {
    int zq, nzq, xq, nxq;
    slab_split(dims[2], G, q, &zq, &nzq);
    slab_split(Px, G, q, &xq, &nxq);
    aoff[q] = int64_t(xq) * nzr * Ny;
    acnt[q] = int64_t(nxq) * nzr * Ny;
    roff[q] = int64_t(nxr) * zq * Ny;
    rcnt[q] = int64_t(nxr) * nzq * Ny;
  }
}

size_t a_off(const fusg_kernel* K, int q) { return size_t(K->aoff[q]); }
size_t a_cnt(const fusg_kernel* K, int q) { return size_t(K->acnt[q]); }
size_t r_off(const fusg_kernel* K, int p) { return size_t(K->roff[p]); }
size_t r_cnt(const fusg_kernel* K, int p) { return size_t(K->rcnt[p]); }

// rbuf [p][nx][nz_p][Ny] <-> X [nx][Nz][Ny]
fusg_status unpack(fusg_kernel* K, cudaStream_t s) {
  const int64_t Ny = row(K), Nz = K->grid.dims[2];
  for (int p = 0; p < K->G; ++p) {
    if (K->nzs[p] == 0 || K->nx == 0) continue;
    FUSG_CUDA_TRY(cudaMemcpy2DAsync(K->xbuf + K->zs[p] * Ny, Nz * Ny * kC, K->rbuf + r_off(K, p),
                                    K->nzs[p] * Ny * kC, K->nzs[p] * Ny * kC, K->nx,
                                    cudaMemcpyDeviceToDevice, s));
  }
  return FUSG_OK;
}

fusg_status pack(fusg_kernel* K, cudaStream_t s) {
  const int64_t Ny = row(K), Nz = K->grid.dims[2];
  for (int q = 0; q < K->G; ++q) {
    if (K->nzs[q] == 0 || K->nx == 0) continue;
    FUSG_CUDA_TRY(cudaMemcpy2DAsync(K->rbuf + r_off(K, q), K->nzs[q] * Ny * kC, K->xbuf + K->zs[q] * Ny,
                                    Nz * Ny * kC, K->nzs[q] * Ny * kC, K->nx,
                                    cudaMemcpyDeviceToDevice, s));
  }
  return FUSG_OK;
}

fusg_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FUSG_OK;
  return set_error(FUSG_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

// one all-to-all(v) over the context's communicator: send block q from `sb + so(q)`, receive
// block p into `rb + ro(p)` (counts in complex128 elements)
template <class SO, class SC, class RO, class RC>
fusg_status nccl_alltoallv(fusg_ctx* ctx, const double2* sb, SO so, SC sc, double2* rb, RO ro, RC rc,
                           int G, cudaStream_t s) {
  auto comm = static_cast<ncclComm_t>(ctx->nccl);
  FUSG_TRY(nccl_check(ncclGroupStart(), "ncclGroupStart"));
  for (int q = 0; q < G; ++q) {
    if (sc(q)) FUSG_TRY(nccl_check(ncclSend(sb + so(q), 2 * sc(q), ncclDouble, q, comm, s), "ncclSend"));
    if (rc(q)) FUSG_TRY(nccl_check(ncclRecv(rb + ro(q), 2 * rc(q), ncclDouble, q, comm, s), "ncclRecv"));
  }
  return nccl_check(ncclGroupEnd(), "ncclGroupEnd");
}

fusg_status create_slab(fusg_ctx* ctx, const fusg_grid* grid, const fusg_wavenumber* k, int G, int r,
                        fusg_kernel** out) {
  double w0[2];
  fusg_status st = fusg_self_weight(k, grid->dx, w0);
  if (st != FUSG_OK) return st;
  auto* K = new fusg_kernel;
  K->ctx = ctx;
  ctx_retain(ctx);
  K->grid = *grid;
  K->k = *k;
  K->slab = true;
  st = kernel_init_geometry(K, G, r);
  if (st == FUSG_OK) {
    K->aoff.resize(G);
    K->acnt.resize(G);
    K->roff.resize(G);
    K->rcnt.resize(G);
    exchange_plan(K->grid.dims, K->P[0], G, r, K->aoff.data(), K->acnt.data(), K->roff.data(),
                  K->rcnt.data());
    st = volume_potential_build(K, make_double2(w0[0], w0[1]));
  }
  if (st != FUSG_OK) {
    fusg_kernel_destroy(K);
    return st;
  }
  *out = K;
  return FUSG_OK;
}

// Peer-store plan of the fused transposes for rank r (exported as fusg_slab_peer_plan):
//   pass A (owner by kx): element (y, z_local, kx) -> X_q[kx - x0_q][z0_r + z_local][y]
//     flat index a_off[q] + y + z_local * a_sk[q] + kx * Nz * Ny
//   pass D (owner by z):  element (z, kx_local, y) -> A_q[x0_r + kx_local][z - z0_q][y]
//     flat index d_off[q] + z * Ny + kx_local * d_sk[q] + y
void peer_plan(const int dims[3], int Px, int G, int r, int64_t* a_begin, int64_t* a_off, int64_t* a_sk,
               int64_t* d_begin, int64_t* d_off, int64_t* d_sk) {
  const int64_t Ny = dims[1], Nz = dims[2];
  int z0r, nzr, x0r, nxr;
  slab_split(dims[2], G, r, &z0r, &nzr);
  slab_split(Px, G, r, &x0r, &nxr);
  for (int q = 0; q < G; ++q) {
    int zq, nzq, xq, nxq;
    slab_split(dims[2], G, q, &zq, &nzq);
    slab_split(Px, G, q, &xq, &nxq);
    a_begin[q] = xq;
    a_off[q] = int64_t(z0r) * Ny - int64_t(xq) * Nz * Ny;
    a_sk[q] = Ny;
    d_begin[q] = zq;
    d_off[q] = int64_t(x0r) * nzq * Ny - int64_t(zq) * Ny;
    d_sk[q] = int64_t(nzq) * Ny;
  }
}

// the plan plus every rank's x-slab / A buffer -> the kernels' peer maps
void peer_maps(const fusg_kernel* K, double2* const* X, double2* const* A, PeerMap* pa, PeerMap* pd) {
  const int G = K->G;
  int64_t ab[kMaxPeers], ao[kMaxPeers], as[kMaxPeers], db[kMaxPeers], dof[kMaxPeers], ds[kMaxPeers];
  peer_plan(K->grid.dims, K->P[0], G, K->rank, ab, ao, as, db, dof, ds);
  pa->n = pd->n = G;
  pa->by_pos = 1;
  pd->by_pos = 0;
  for (int q = 0; q < G; ++q) {
    pa->begin[q] = int(ab[q]);
    pa->base[q] = X[q];
    pa->off[q] = ao[q];
    pa->sk[q] = as[q];
    pd->begin[q] = int(db[q]);
    pd->base[q] = A[q];
    pd->off[q] = dof[q];
    pd->sk[q] = ds[q];
  }
}

fusg_status nccl_barrier(fusg_kernel* K, cudaStream_t s) {
  if (K->G == 1) return FUSG_OK;
  auto comm = static_cast<ncclComm_t>(K->ctx->nccl);
  return nccl_check(ncclAllReduce(K->bar, K->bar, 1, ncclInt, ncclMax, comm, s), "ncclAllReduce (barrier)");
}

}  // namespace

void destroy_nccl(fusg_ctx* ctx) {
  if (ctx && ctx->nccl) ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl));
  if (ctx) ctx->nccl = nullptr;
}

}  // namespace fusg

using namespace fusg;

extern "C" {

fusg_status fusg_slab_range(int32_t n, int32_t nranks, int32_t rank, int32_t* begin, int32_t* count) {
  if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks || !begin || !count)
    return set_error(FUSG_INVALID_ARGUMENT, "slab_range: bad arguments");
  int b, c;
  slab_split(n, nranks, rank, &b, &c);
  *begin = b;
  *count = c;
  return FUSG_OK;
}

fusg_status fusg_slab_exchange_plan(const fusg_grid* global_grid, int32_t nranks, int32_t rank,
                                    int64_t* a_off, int64_t* a_cnt, int64_t* r_off, int64_t* r_cnt) {
  if (!global_grid || nranks < 1 || rank < 0 || rank >= nranks || !a_off || !a_cnt || !r_off || !r_cnt)
    return set_error(FUSG_INVALID_ARGUMENT, "slab_exchange_plan: bad arguments");
  int32_t P[3];
  FUSG_TRY(fusg_padded_dims(global_grid, 0, P));
  if (nranks > global_grid->dims[2] || nranks > P[0])
    return set_error(FUSG_INVALID_ARGUMENT, "more ranks than z-planes or kx columns");
  exchange_plan(global_grid->dims, P[0], nranks, rank, a_off, a_cnt, r_off, r_cnt);
  return FUSG_OK;
}

fusg_status fusg_slab_peer_plan(const fusg_grid* global_grid, int32_t nranks, int32_t rank, int64_t* a_begin,
                                int64_t* a_off, int64_t* a_sk, int64_t* d_begin, int64_t* d_off,
                                int64_t* d_sk) {
  if (!global_grid || nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks || !a_begin || !a_off ||
      !a_sk || !d_begin || !d_off || !d_sk)
    return set_error(FUSG_INVALID_ARGUMENT, "slab_peer_plan: bad arguments");
  int32_t P[3];
  FUSG_TRY(fusg_padded_dims(global_grid, 0, P));
  if (nranks > global_grid->dims[2] || nranks > P[0])
    return set_error(FUSG_INVALID_ARGUMENT, "more ranks than z-planes or kx columns");
  peer_plan(global_grid->dims, P[0], nranks, rank, a_begin, a_off, a_sk, d_begin, d_off, d_sk);
  return FUSG_OK;
}

fusg_status fusg_nccl_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  FUSG_TRY(nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId"));
  std::memcpy(id, &u, 128);
  return FUSG_OK;
}

fusg_status fusg_ctx_attach_nccl(fusg_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[128]) {
  if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(FUSG_INVALID_ARGUMENT, "ctx_attach_nccl: bad arguments");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t comm;
  FUSG_TRY(nccl_check(ncclCommInitRank(&comm, nranks, u, rank), "ncclCommInitRank"));
  ctx->nccl = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  return FUSG_OK;
}

fusg_status fusg_kernel_create_slab(fusg_ctx* ctx, const fusg_grid* global_grid, const fusg_wavenumber* k,
                                    int32_t pad_small_primes, int32_t nranks, int32_t rank,
                                    fusg_kernel** out) {
  (void)pad_small_primes;
  if (!ctx || !global_grid || !k || !out) return set_error(FUSG_INVALID_ARGUMENT, "kernel_create_slab: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  return create_slab(ctx, global_grid, k, nranks, rank, out);
}

fusg_status fusg_kernel_octant_rows(const fusg_kernel* K, int32_t* kf0, int32_t* knf) {
  if (!K) return set_error(FUSG_INVALID_ARGUMENT, "kernel_octant_rows: null kernel");
  if (kf0) *kf0 = K->kf0;
  if (knf) *knf = K->knf;
  return FUSG_OK;
}

fusg_status fusg_kernel_slab(const fusg_kernel* K, int32_t* z0, int32_t* nz, int32_t* x0, int32_t* nx) {
  if (!K) return set_error(FUSG_INVALID_ARGUMENT, "kernel_slab: null kernel");
  if (z0) *z0 = K->z0;
  if (nz) *nz = K->nz;
  if (x0) *x0 = K->x0;
  if (nx) *nx = K->nx;
  return FUSG_OK;
}

// One process per GPU: f_dev/u_dev hold this rank's z-slab [nz][Ny][Nx].
fusg_status fusg_kernel_apply_slab(fusg_kernel* K, const double* f_dev, double* u_dev, double scale,
                                   void* stream) {
  if (!K || !f_dev || !u_dev) return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply_slab: null argument");
  // G = 1 still takes the full exchange path (NCCL send/recv to self): it is the one-GPU
  // test of the code the multi-GPU job runs.
  fusg_ctx* ctx = K->ctx;
  if (!ctx->nccl || ctx->nranks != K->G || ctx->rank != K->rank)
    return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply_slab: context has no matching NCCL communicator");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  std::lock_guard<std::mutex> lock(K->mu);
  cudaStream_t s = ctx->pick(stream);
  FUSG_TRY(ensure_rbuf(K, s));
  FUSG_TRY(apply_phase_A(K, reinterpret_cast<const double2*>(f_dev), s));
  FUSG_TRY(nccl_alltoallv(ctx, K->bufA, [&](int q) { return a_off(K, q); }, [&](int q) { return a_cnt(K, q); },
                          K->rbuf, [&](int p) { return r_off(K, p); }, [&](int p) { return r_cnt(K, p); },
                          K->G, s));
  FUSG_TRY(unpack(K, s));
  FUSG_TRY(apply_phase_BCD(K, K->xbuf, s));
  FUSG_TRY(pack(K, s));
  FUSG_TRY(nccl_alltoallv(ctx, K->rbuf, [&](int q) { return r_off(K, q); }, [&](int q) { return r_cnt(K, q); },
                          K->bufA, [&](int p) { return a_off(K, p); }, [&](int p) { return a_cnt(K, p); },
                          K->G, s));
  return apply_phase_E(K, reinterpret_cast<double2*>(u_dev), scale, s);
}

// Every rank of a G-way decomposition in this process, one device: exchanges are device copies.
fusg_status fusg_kernel_apply_slab_loopback(fusg_kernel* const* ranks, int32_t nranks,
                                            const double* const* f_dev, double* const* u_dev,
                                            double scale) {
  if (!ranks || nranks < 1 || !f_dev || !u_dev) return set_error(FUSG_INVALID_ARGUMENT, "apply_slab_loopback: null argument");
  for (int r = 0; r < nranks; ++r)
    if (!ranks[r] || ranks[r]->G != nranks || ranks[r]->rank != r || ranks[r]->ctx != ranks[0]->ctx)
      return set_error(FUSG_INVALID_ARGUMENT, "apply_slab_loopback: kernels must be ranks 0..G-1 of one decomposition on one context");
  fusg_ctx* ctx = ranks[0]->ctx;
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  for (int r = 0; r < nranks; ++r) FUSG_TRY(ensure_rbuf(ranks[r], s));
  const int G = nranks;
  for (int r = 0; r < G; ++r) FUSG_TRY(apply_phase_A(ranks[r], reinterpret_cast<const double2*>(f_dev[r]), s));
  for (int r = 0; r < G; ++r)  // exchange 1: p's A slice for r -> r's rbuf block p
    for (int p = 0; p < G; ++p)
      if (r_cnt(ranks[r], p))
        FUSG_CUDA_TRY(cudaMemcpyAsync(ranks[r]->rbuf + r_off(ranks[r], p), ranks[p]->bufA + a_off(ranks[p], r),
                                      r_cnt(ranks[r], p) * kC, cudaMemcpyDeviceToDevice, s));
  for (int r = 0; r < G; ++r) {
    FUSG_TRY(unpack(ranks[r], s));
    FUSG_TRY(apply_phase_BCD(ranks[r], ranks[r]->xbuf, s));
    FUSG_TRY(pack(ranks[r], s));
  }
  for (int r = 0; r < G; ++r)  // exchange 2: q's packed block for r -> r's A slice q
    for (int q = 0; q < G; ++q)
      if (a_cnt(ranks[r], q))
        FUSG_CUDA_TRY(cudaMemcpyAsync(ranks[r]->bufA + a_off(ranks[r], q), ranks[q]->rbuf + r_off(ranks[q], r),
                                      a_cnt(ranks[r], q) * kC, cudaMemcpyDeviceToDevice, s));
  for (int r = 0; r < G; ++r) FUSG_TRY(apply_phase_E(ranks[r], reinterpret_cast<double2*>(u_dev[r]), scale, s));
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return FUSG_OK;
}

// ---- fused peer-memory transposes (the transposes fused into passes A and D)
fusg_status fusg_kernel_slab_ipc_handles(const fusg_kernel* K, uint8_t out[128]) {
  if (!K || !out) return set_error(FUSG_INVALID_ARGUMENT, "slab_ipc_handles: null argument");
  if (!K->ipc_bufs || !K->xbuf) return set_error(FUSG_INVALID_ARGUMENT, "slab_ipc_handles: not a slab kernel");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  FUSG_CUDA_TRY(cudaSetDevice(K->ctx->device));
  cudaIpcMemHandle_t hx, ha;
  FUSG_CUDA_TRY(cudaIpcGetMemHandle(&hx, K->xbuf));
  FUSG_CUDA_TRY(cudaIpcGetMemHandle(&ha, K->bufA));
  std::memcpy(out, &hx, 64);
  std::memcpy(out + 64, &ha, 64);
  return FUSG_OK;
}

fusg_status fusg_kernel_slab_attach_peers(fusg_kernel* K, const uint8_t* handles) {
  if (!K || !handles) return set_error(FUSG_INVALID_ARGUMENT, "slab_attach_peers: null argument");
  if (!K->ipc_bufs || !K->xbuf) return set_error(FUSG_INVALID_ARGUMENT, "slab_attach_peers: not a slab kernel");
  if (K->G > kMaxPeers) return set_error(FUSG_INVALID_ARGUMENT, "slab_attach_peers: more than 8 ranks");
  FUSG_CUDA_TRY(cudaSetDevice(K->ctx->device));
  std::lock_guard<std::mutex> lock(K->mu);
  if (!K->peerX.empty()) return set_error(FUSG_INVALID_ARGUMENT, "slab_attach_peers: peers already attached");
  K->peerX.assign(K->G, nullptr);
  K->peerA.assign(K->G, nullptr);
  K->peer_opened.assign(K->G, false);
  for (int q = 0; q < K->G; ++q) {
    if (q == K->rank) {
      K->peerX[q] = K->xbuf;
      K->peerA[q] = K->bufA;
      continue;
    }
    cudaIpcMemHandle_t hx, ha;
    std::memcpy(&hx, handles + 128 * q, 64);
    std::memcpy(&ha, handles + 128 * q + 64, 64);
    void *px = nullptr, *pa = nullptr;
    FUSG_CUDA_TRY(cudaIpcOpenMemHandle(&px, hx, cudaIpcMemLazyEnablePeerAccess));
    if (cudaIpcOpenMemHandle(&pa, ha, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaIpcCloseMemHandle(px);
      return set_error(FUSG_CUDA, "slab_attach_peers: cannot map a peer A slab");
    }
    K->peerX[q] = static_cast<double2*>(px);
    K->peerA[q] = static_cast<double2*>(pa);
    K->peer_opened[q] = true;
  }
  if (!K->bar) {
    FUSG_CUDA_TRY(cudaMalloc(&K->bar, sizeof(int)));
    FUSG_CUDA_TRY(cudaMemset(K->bar, 0, sizeof(int)));
  }
  return FUSG_OK;
}

// One process per GPU, peers attached: pass A stores straight into the owners' x-slabs, a
// stream barrier (1-int NCCL all-reduce), passes B, C, pass D stores straight into the owners'
// A slabs, a barrier, pass E.  No exchange buffers, no pack/unpack copies.
fusg_status fusg_kernel_apply_slab_p2p(fusg_kernel* K, const double* f_dev, double* u_dev, double scale,
                                       void* stream) {
  if (!K || !f_dev || !u_dev) return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply_slab_p2p: null argument");
  fusg_ctx* ctx = K->ctx;
  if (int(K->peerX.size()) != K->G)
    return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply_slab_p2p: peers not attached (fusg_kernel_slab_attach_peers)");
  if (K->G > 1 && (!ctx->nccl || ctx->nranks != K->G || ctx->rank != K->rank))
    return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply_slab_p2p: context has no matching NCCL communicator");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  std::lock_guard<std::mutex> lock(K->mu);
  cudaStream_t s = ctx->pick(stream);
  PeerMap pa, pd;
  peer_maps(K, K->peerX.data(), K->peerA.data(), &pa, &pd);
  FUSG_TRY(apply_phase_A_peers(K, reinterpret_cast<const double2*>(f_dev), pa, s));
  FUSG_TRY(nccl_barrier(K, s));
  FUSG_TRY(apply_phase_BC(K, K->xbuf, s));
  FUSG_TRY(apply_phase_D_peers(K, pd, s));
  FUSG_TRY(nccl_barrier(K, s));
  return apply_phase_E(K, reinterpret_cast<double2*>(u_dev), scale, s);
}

// The fused path for all G ranks in this process on one device (the peers are the other
// in-process ranks' buffers; stream order stands in for the barriers).
fusg_status fusg_kernel_apply_slab_loopback_p2p(fusg_kernel* const* ranks, int32_t nranks,
                                                const double* const* f_dev, double* const* u_dev,
                                                double scale) {
  if (!ranks || nranks < 1 || !f_dev || !u_dev)
    return set_error(FUSG_INVALID_ARGUMENT, "apply_slab_loopback_p2p: null argument");
  if (nranks > kMaxPeers) return set_error(FUSG_INVALID_ARGUMENT, "apply_slab_loopback_p2p: more than 8 ranks");
  for (int r = 0; r < nranks; ++r)
    if (!ranks[r] || ranks[r]->G != nranks || ranks[r]->rank != r || ranks[r]->ctx != ranks[0]->ctx ||
        !ranks[r]->ipc_bufs)
      return set_error(FUSG_INVALID_ARGUMENT, "apply_slab_loopback_p2p: kernels must be ranks 0..G-1 of one decomposition on one context");
  fusg_ctx* ctx = ranks[0]->ctx;
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const int G = nranks;
  std::vector<double2*> X(G), A(G);
  for (int q = 0; q < G; ++q) {
    X[q] = ranks[q]->xbuf;
    A[q] = ranks[q]->bufA;
  }
  std::vector<PeerMap> pa(G), pd(G);
  for (int r = 0; r < G; ++r) peer_maps(ranks[r], X.data(), A.data(), &pa[r], &pd[r]);
  for (int r = 0; r < G; ++r)
    FUSG_TRY(apply_phase_A_peers(ranks[r], reinterpret_cast<const double2*>(f_dev[r]), pa[r], s));
  for (int r = 0; r < G; ++r) {
    FUSG_TRY(apply_phase_BC(ranks[r], ranks[r]->xbuf, s));
    FUSG_TRY(apply_phase_D_peers(ranks[r], pd[r], s));
  }
  for (int r = 0; r < G; ++r) FUSG_TRY(apply_phase_E(ranks[r], reinterpret_cast<double2*>(u_dev[r]), scale, s));
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return FUSG_OK;
}

}  // extern "C"
