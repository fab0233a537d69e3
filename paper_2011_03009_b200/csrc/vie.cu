// VIE mode on the device (reference src/vie.cpp): the wavenumber
// contrast of a medium map, the VIE operator p - V[(k^2 - kbar^2) p], restarted GMRES with the
// reference's modified Gram-Schmidt Arnoldi and Givens rotations, solve_vie, and the
// inhomogeneous-medium cascade.
//
// GMRES keeps the Krylov basis (restart + 1 vectors) and every vector operation on the device.
// Dot products are deterministic: 1024 fixed blocks, each summing a fixed grid-stride slice and
// tree-reducing in shared memory, then one block adding the 1024 partials in order.  The
// results stay on the device, so a whole Arnoldi step (operator, k+1 dot/axpy pairs, the norm)
// runs without host round trips; the host reads the new Hessenberg column once per iteration
// and runs the (m+1) x m Givens/back-substitution logic exactly as src/vie.cpp:141-236.
#include <cmath>
#include <complex>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "internal.hpp"

namespace fusg {
namespace {

constexpr int kRedBlocks = 1024, kRedThreads = 256;

unsigned blocks_for(int64_t n) { return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }

// k^2 - kbar^2 with k = (n omega / c, Im kbar) where c != c0, else 0 (src/vie.cpp:11-23); the
// complex products round like std::complex's (ac - bd, ad + bc)
__global__ void contrast_kernel(const double2* __restrict__ map, int64_t n, double c0, double n_omega,
                                double2 kbar, double2* __restrict__ out) {
  const double kb_re = __dsub_rn(__dmul_rn(kbar.x, kbar.x), __dmul_rn(kbar.y, kbar.y));
  const double kb_im = __dadd_rn(__dmul_rn(kbar.x, kbar.y), __dmul_rn(kbar.y, kbar.x));
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double c = map[i].x;
    if (c == c0) {
      out[i] = make_double2(0.0, 0.0);
      continue;
    }
    const double kr = __ddiv_rn(n_omega, c), ki = kbar.y;
    const double re = __dsub_rn(__dmul_rn(kr, kr), __dmul_rn(ki, ki));
    const double im = __dadd_rn(__dmul_rn(kr, ki), __dmul_rn(ki, kr));
    out[i] = make_double2(__dsub_rn(re, kb_re), __dsub_rn(im, kb_im));
  }
}

// rhs_j = -(beta_j omega^2 n^2 / (2 rho0 c_j^4)) conv_j   (src/vie.cpp:305-311)
__global__ void vie_rhs_kernel(const double2* __restrict__ map, const double2* __restrict__ conv, int64_t n,
                               double omega, double n2, double rho0, double2* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double c = map[i].x, beta = map[i].y;
    const double c2 = __dmul_rn(c, c);
    const double coeff = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(beta, omega), omega), n2),
                                   __dmul_rn(2.0 * rho0, __dmul_rn(c2, c2)));
    const double2 v = conv[i];
    out[i] = make_double2(__dmul_rn(-coeff, v.x), __dmul_rn(-coeff, v.y));
  }
}

// out = a .* b (complex, non-fused like std::complex)
__global__ void cmul_kernel(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                            double2* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double2 x = a[i], y = b[i];
    out[i] = make_double2(__dsub_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)),
                          __dadd_rn(__dmul_rn(x.x, y.y), __dmul_rn(x.y, y.x)));
  }
}

// out = a + sa * b  (sa = +-1: sums and differences of whole vectors)
__global__ void axpb_kernel(const double2* __restrict__ a, double sb, const double2* __restrict__ b, int64_t n,
                            double2* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double2 x = a[i], y = b[i];
    out[i] = sb > 0.0 ? make_double2(x.x + y.x, x.y + y.y) : make_double2(x.x - y.x, x.y - y.y);
  }
}

// partial[b] = sum over block b's fixed slice of conj(a_i) b_i (Eigen's dot convention)
__global__ void __launch_bounds__(kRedThreads) dot_partial_kernel(const double2* __restrict__ a,
                                                                  const double2* __restrict__ b, int64_t n,
                                                                  double2* __restrict__ partial) {
  __shared__ double2 red[kRedThreads];
  double sr = 0.0, si = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; i < n; i += int64_t(kRedBlocks) * kRedThreads) {
    const double2 x = a[i], y = b[i];
    sr = fma(x.x, y.x, fma(x.y, y.y, sr));
    si = fma(x.x, y.y, fma(-x.y, y.x, si));
  }
  red[threadIdx.x] = make_double2(sr, si);
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      red[threadIdx.x] = make_double2(red[threadIdx.x].x + red[threadIdx.x + w].x,
                                      red[threadIdx.x].y + red[threadIdx.x + w].y);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// MGS step fused: w -= (*s_prev) v_prev, then partial[b] = sum conj(v_next_i) w_i over the same
// fixed slices as dot_partial_kernel (v_next == w gives |w|^2).  One pass over w instead of two.
__global__ void __launch_bounds__(kRedThreads) axpy_dot_partial_kernel(double2* __restrict__ w,
                                                                       const double2* __restrict__ v_prev,
                                                                       const double2* __restrict__ s_prev,
                                                                       const double2* v_next, int64_t n,
                                                                       double2* __restrict__ partial) {
  __shared__ double2 red[kRedThreads];
  const double2 c = *s_prev;
  double sr = 0.0, si = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; i < n; i += int64_t(kRedBlocks) * kRedThreads) {
    const double2 x = v_prev[i];
    const double2 y = make_double2(w[i].x - (c.x * x.x - c.y * x.y), w[i].y - (c.x * x.y + c.y * x.x));
    w[i] = y;
    const double2 a = v_next == w ? y : v_next[i];
    sr = fma(a.x, y.x, fma(a.y, y.y, sr));
    si = fma(a.x, y.y, fma(-a.y, y.x, si));
  }
  red[threadIdx.x] = make_double2(sr, si);
  __syncthreads();
  for (int t = kRedThreads / 2; t > 0; t >>= 1) {
    if (threadIdx.x < t)
      red[threadIdx.x] = make_double2(red[threadIdx.x].x + red[threadIdx.x + t].x,
                                      red[threadIdx.x].y + red[threadIdx.x + t].y);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(kRedThreads) dot_final_kernel(const double2* __restrict__ partial,
                                                                double2* __restrict__ result) {
  __shared__ double2 red[kRedThreads];
  double2 t = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < kRedBlocks; i += kRedThreads) t = make_double2(t.x + partial[i].x, t.y + partial[i].y);
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      red[threadIdx.x] = make_double2(red[threadIdx.x].x + red[threadIdx.x + w].x,
                                      red[threadIdx.x].y + red[threadIdx.x + w].y);
    __syncthreads();
  }
  if (threadIdx.x == 0) *result = red[0];
}

// x += y v (host coefficient)
__global__ void axpy_host_kernel(double2* __restrict__ x, const double2* __restrict__ v, double2 y, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double2 a = v[i];
    x[i] = make_double2(x[i].x + (y.x * a.x - y.y * a.y), x[i].y + (y.x * a.y + y.y * a.x));
  }
}

// out = w / d (d a real host scalar)
__global__ void div_kernel(const double2* __restrict__ w, double d, int64_t n, double2* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = make_double2(w[i].x / d, w[i].y / d);
}

struct DevBufs {
  std::vector<void*> p;
  cudaStream_t s;
  ~DevBufs() {
    for (void* q : p) cudaFreeAsync(q, s);
  }
  template <class T>
  fusg_status alloc(T** out, size_t n) {
    void* q = nullptr;
    if (cudaMallocAsync(&q, n * sizeof(T), s) != cudaSuccess) {
      cudaGetLastError();
      return set_error(FUSG_OOM, "VIE: device workspace allocation failed");
    }
    p.push_back(q);
    *out = static_cast<T*>(q);
    return FUSG_OK;
  }
};

struct Reducer {
  fusg_ctx* ctx;
  double2* partial;
  cudaStream_t s;
  // result[0] = sum conj(a) b, left on the device
  fusg_status dot(const double2* a, const double2* b, int64_t n, double2* result) {
    dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a, b, n, partial);
    dot_final_kernel<<<1, kRedThreads, 0, s>>>(partial, result);
    ctx->launches += 2;
    FUSG_LAUNCH_CHECK("dot kernels");
    return FUSG_OK;
  }
};

// gmres (src/vie.cpp:141-236) on device vectors; `op` computes out = A in on the device.
fusg_status gmres_dev(fusg_ctx* ctx, const std::function<fusg_status(const double2*, double2*)>& op,
                      const double2* rhs, int64_t n, double tol, int max_iter, int restart, double2* x,
                      std::vector<double>& hist, int* iterations, cudaStream_t s) {
  using cd = std::complex<double>;
  if (tol <= 0.0) return set_error(FUSG_INVALID_ARGUMENT, "gmres: tol must be positive");
  if (restart < 1) return set_error(FUSG_INVALID_ARGUMENT, "gmres: restart must be >= 1");
  DevBufs ws{{}, s};
  double2 *V = nullptr, *w = nullptr, *r = nullptr, *partial = nullptr, *hcol = nullptr;
  FUSG_TRY(ws.alloc(&partial, kRedBlocks));
  FUSG_TRY(ws.alloc(&hcol, size_t(restart) + 2));
  Reducer red{ctx, partial, s};
  auto host_dot = [&](const double2* a, const double2* b, cd* out) -> fusg_status {
    FUSG_TRY(red.dot(a, b, n, hcol));
    double2 h;
    FUSG_CUDA_TRY(cudaMemcpyAsync(&h, hcol, sizeof(h), cudaMemcpyDeviceToHost, s));
    FUSG_CUDA_TRY(cudaStreamSynchronize(s));
    *out = cd(h.x, h.y);
    return FUSG_OK;
  };
  hist.clear();
  *iterations = 0;
  FUSG_CUDA_TRY(cudaMemsetAsync(x, 0, size_t(n) * sizeof(double2), s));
  cd rr;
  FUSG_TRY(host_dot(rhs, rhs, &rr));
  const double rhs_norm = std::sqrt(rr.real());
  if (rhs_norm == 0.0) return FUSG_OK;
  FUSG_TRY(ws.alloc(&V, size_t(restart + 1) * size_t(n)));
  FUSG_TRY(ws.alloc(&w, size_t(n)));
  FUSG_TRY(ws.alloc(&r, size_t(n)));
  auto vec = [&](int j) { return V + size_t(j) * size_t(n); };
  const unsigned nb = blocks_for(n);
  int total = 0;
  bool x_zero = true;
  while (true) {
    if (x_zero) {  // op(0) = 0 exactly: r = rhs
      FUSG_CUDA_TRY(cudaMemcpyAsync(r, rhs, size_t(n) * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    } else {
      FUSG_TRY(op(x, w));
      axpb_kernel<<<nb, 256, 0, s>>>(rhs, -1.0, w, n, r);
      ctx->launches++;
    }
    FUSG_TRY(host_dot(r, r, &rr));
    const double beta = std::sqrt(rr.real());
    double rel = beta / rhs_norm;
    if (hist.empty()) hist.push_back(rel);
    if (rel <= tol) {
      *iterations = total;
      return FUSG_OK;
    }
    if (total >= max_iter)
      return set_error(FUSG_NOT_CONVERGED, "gmres: no convergence within " + std::to_string(max_iter) +
                                                " iterations (residual " + std::to_string(rel) + ")");
    const int m = restart;
    div_kernel<<<nb, 256, 0, s>>>(r, beta, n, vec(0));
    ctx->launches++;
    std::vector<cd> h(size_t(m + 1) * m, cd(0.0)), g(m + 1, cd(0.0)), cs(m), sn(m);
    auto H = [&](int i, int j) -> cd& { return h[size_t(i) * m + j]; };
    g[0] = beta;
    int k = 0;
    std::vector<double2> col(m + 2);
    while (k < m && total < max_iter) {
      // Arnoldi with modified Gram-Schmidt, on the device
      FUSG_TRY(op(vec(k), w));
      // h_j = <v_j, w>; w -= h_j v_j, each axpy fused with the next dot (and the last with |w|^2)
      FUSG_TRY(red.dot(vec(0), w, n, hcol));
      for (int j = 1; j <= k + 1; ++j) {
        axpy_dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(w, vec(j - 1), hcol + j - 1,
                                                                   j <= k ? vec(j) : w, n, partial);
        dot_final_kernel<<<1, kRedThreads, 0, s>>>(partial, hcol + j);
        ctx->launches += 2;
      }
      FUSG_LAUNCH_CHECK("arnoldi kernels");
      FUSG_CUDA_TRY(cudaMemcpyAsync(col.data(), hcol, sizeof(double2) * (k + 2), cudaMemcpyDeviceToHost, s));
      FUSG_CUDA_TRY(cudaStreamSynchronize(s));
      for (int j = 0; j <= k; ++j) H(j, k) = cd(col[j].x, col[j].y);
      const double wnorm = std::sqrt(col[k + 1].x);
      H(k + 1, k) = wnorm;
      // previous Givens rotations, then the new one annihilating h(k+1, k)
      for (int j = 0; j < k; ++j) {
        const cd tmp = std::conj(cs[j]) * H(j, k) + std::conj(sn[j]) * H(j + 1, k);
        H(j + 1, k) = -sn[j] * H(j, k) + cs[j] * H(j + 1, k);
        H(j, k) = tmp;
      }
      const double denom = std::sqrt(std::norm(H(k, k)) + std::norm(H(k + 1, k)));
      if (denom == 0.0) {
        cs[k] = 1.0;
        sn[k] = 0.0;
      } else {
        cs[k] = H(k, k) / denom;
        sn[k] = H(k + 1, k) / denom;
      }
      H(k, k) = std::conj(cs[k]) * H(k, k) + std::conj(sn[k]) * H(k + 1, k);
      H(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = std::conj(cs[k]) * g[k];
      rel = std::abs(g[k + 1]) / rhs_norm;
      hist.push_back(rel);
      // (src/vie.cpp:213-221: the two early exits advance k but not the iteration count)
      if (rel <= tol) {
        ++k;
        break;
      }
      if (wnorm == 0.0) {
        ++k;
        break;  // invariant subspace reached
      }
      div_kernel<<<nb, 256, 0, s>>>(w, wnorm, n, vec(k + 1));
      ctx->launches++;
      ++k;
      ++total;
    }
    // back-substitute y and update x
    std::vector<cd> y(k);
    for (int i = k - 1; i >= 0; --i) {
      cd sum = g[i];
      for (int j = i + 1; j < k; ++j) sum -= H(i, j) * y[j];
      y[i] = sum / H(i, i);
    }
    for (int i = 0; i < k; ++i) {
      axpy_host_kernel<<<nb, 256, 0, s>>>(x, vec(i), make_double2(y[i].real(), y[i].imag()), n);
      ctx->launches++;
    }
    FUSG_LAUNCH_CHECK("gmres update");
    x_zero = false;
    if (rel <= tol) {
      *iterations = total;
      return FUSG_OK;
    }
  }
}

void copy_history(const std::vector<double>& hist, double* out, int cap, int* len) {
  if (len) *len = int(hist.size());
  if (out)
    for (int i = 0; i < cap && i < int(hist.size()); ++i) out[i] = hist[i];
}

// p - V[contrast p] into out (tmp: N-element workspace)
fusg_status vie_op(fusg_kernel* K, const double2* contrast, const double2* p, double2* out, double2* tmp,
                   cudaStream_t s) {
  const int64_t n = int64_t(K->grid.dims[0]) * K->grid.dims[1] * K->grid.dims[2];
  const unsigned nb = blocks_for(n);
  cmul_kernel<<<nb, 256, 0, s>>>(contrast, p, n, tmp);
  K->ctx->launches++;
  FUSG_LAUNCH_CHECK("cmul_kernel");
  FUSG_TRY(volume_potential_apply(K, tmp, out, -1.0, s));  // out = -V[contrast p]
  axpb_kernel<<<nb, 256, 0, s>>>(p, 1.0, out, n, out);     // p + (-V[..]) == p - V[..]
  K->ctx->launches++;
  FUSG_LAUNCH_CHECK("axpb_kernel");
  return FUSG_OK;
}

fusg_status solve_vie_dev(fusg_kernel* K, const double2* rhs, const double2* contrast, double tol, int max_iter,
                          int restart, double2* x, std::vector<double>& hist, int* iterations, cudaStream_t s) {
  const int64_t n = int64_t(K->grid.dims[0]) * K->grid.dims[1] * K->grid.dims[2];
  DevBufs ws{{}, s};
  double2* tmp = nullptr;
  FUSG_TRY(ws.alloc(&tmp, size_t(n)));
  auto op = [&](const double2* in, double2* out) { return vie_op(K, contrast, in, out, tmp, s); };
  return gmres_dev(K->ctx, op, rhs, n, tol, max_iter, restart, x, hist, iterations, s);
}

bool all_zero_dev(const double2* v, int64_t n, fusg_ctx* ctx, cudaStream_t s, fusg_status* st) {
  double m = 0.0;
  *st = max_abs_dev(ctx, v, n, &m, s);
  return m == 0.0;
}

}  // namespace
}  // namespace fusg

using namespace fusg;

extern "C" {

fusg_status fusg_vie_contrast(fusg_ctx* ctx, const double* map_dev, int64_t count, const fusg_medium* background,
                              double f0, int32_t n, double* out_dev, void* stream) {
  if (!ctx || !background || (count > 0 && (!map_dev || !out_dev)))
    return set_error(FUSG_INVALID_ARGUMENT, "vie_contrast: null argument");
  if (count == 0) return FUSG_OK;
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  fusg_wavenumber kbar{};
  FUSG_TRY(fusg_complex_wavenumber(background, f0, n, &kbar));
  cudaStream_t s = ctx->pick(stream);
  contrast_kernel<<<blocks_for(count), 256, 0, s>>>(reinterpret_cast<const double2*>(map_dev), count,
                                                    background->c0, double(n) * kbar.omega,
                                                    make_double2(kbar.k_re, kbar.k_im),
                                                    reinterpret_cast<double2*>(out_dev));
  ctx->launches++;
  FUSG_LAUNCH_CHECK("contrast_kernel");
  return FUSG_OK;
}

fusg_status fusg_vie_operator_apply(fusg_kernel* K, const double* contrast_dev, const double* p_dev, double* out_dev,
                                    void* stream) {
  if (!K || !contrast_dev || !p_dev || !out_dev)
    return set_error(FUSG_INVALID_ARGUMENT, "vie_operator_apply: null argument");
  if (K->G != 1) return set_error(FUSG_INVALID_ARGUMENT, "vie_operator_apply: sharded kernel");
  FUSG_CUDA_TRY(cudaSetDevice(K->ctx->device));
  std::lock_guard<std::mutex> lock(K->mu);
  cudaStream_t s = K->ctx->pick(stream);
  const int64_t n = int64_t(K->grid.dims[0]) * K->grid.dims[1] * K->grid.dims[2];
  DevBufs ws{{}, s};
  double2* tmp = nullptr;
  FUSG_TRY(ws.alloc(&tmp, size_t(n)));
  return vie_op(K, reinterpret_cast<const double2*>(contrast_dev), reinterpret_cast<const double2*>(p_dev),
                reinterpret_cast<double2*>(out_dev), tmp, s);
}

fusg_status fusg_gmres(fusg_ctx* ctx, fusg_operator_fn op, void* user, const double* rhs_dev, int64_t count,
                       double tol, int32_t max_iter, int32_t restart, double* x_dev, double* history_host,
                       int32_t history_capacity, int32_t* history_len, int32_t* iterations) {
  if (!ctx || !op || !x_dev || (count > 0 && !rhs_dev)) return set_error(FUSG_INVALID_ARGUMENT, "gmres: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  std::vector<double> hist;
  int it = 0;
  auto f = [&](const double2* in, double2* out) -> fusg_status {
    FUSG_CUDA_TRY(cudaStreamSynchronize(s));
    return op(user, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(out));
  };
  const fusg_status st = gmres_dev(ctx, f, reinterpret_cast<const double2*>(rhs_dev), count, tol, max_iter, restart,
                                   reinterpret_cast<double2*>(x_dev), hist, &it, s);
  copy_history(hist, history_host, history_capacity, history_len);
  if (iterations) *iterations = it;
  cudaStreamSynchronize(s);
  return st;
}

fusg_status fusg_solve_vie(fusg_kernel* K, const double* rhs_dev, const double* contrast_dev, double tol,
                           int32_t max_iter, int32_t restart, double* x_dev, double* history_host,
                           int32_t history_capacity, int32_t* history_len, int32_t* iterations) {
  if (!K || !rhs_dev || !contrast_dev || !x_dev) return set_error(FUSG_INVALID_ARGUMENT, "solve_vie: null argument");
  if (K->G != 1) return set_error(FUSG_INVALID_ARGUMENT, "solve_vie: sharded kernel");
  FUSG_CUDA_TRY(cudaSetDevice(K->ctx->device));
  std::lock_guard<std::mutex> lock(K->mu);
  cudaStream_t s = K->ctx->stream;
  std::vector<double> hist;
  int it = 0;
  const fusg_status st = solve_vie_dev(K, reinterpret_cast<const double2*>(rhs_dev),
                                       reinterpret_cast<const double2*>(contrast_dev), tol, max_iter, restart,
                                       reinterpret_cast<double2*>(x_dev), hist, &it, s);
  copy_history(hist, history_host, history_capacity, history_len);
  if (iterations) *iterations = it;
  cudaStreamSynchronize(s);
  return st;
}

fusg_status fusg_device_copy(fusg_ctx* ctx, void* dst_dev, const void* src_dev, uint64_t bytes) {
  if (!ctx || (bytes && (!dst_dev || !src_dev))) return set_error(FUSG_INVALID_ARGUMENT, "device_copy: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  FUSG_CUDA_TRY(cudaMemcpyAsync(dst_dev, src_dev, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  FUSG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return FUSG_OK;
}

// run_cascade_inhomogeneous (src/vie.cpp:244-323), device resident
fusg_status fusg_run_cascade_inhomogeneous(fusg_ctx* ctx, const fusg_cascade_desc* d, const fusg_grid* map_grid,
                                           const double* map_host, const fusg_medium* background,
                                           const fusg_vie_config* vie, double* const* out_dev,
                                           fusg_stage_timing* timings, double* source_normalization) {
  if (!ctx || !d || !map_grid || !map_host || !background || !vie || !out_dev)
    return set_error(FUSG_INVALID_ARGUMENT, "run_cascade_inhomogeneous: null argument");
  const int nh = d->n_harmonics;
  if (nh < 1) return set_error(FUSG_INVALID_ARGUMENT, "run_cascade_inhomogeneous: n_harmonics must be >= 1");
  if (!d->grids) return set_error(FUSG_INVALID_ARGUMENT, "run_cascade_inhomogeneous: no planned grids");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const fusg_bowl& t = d->transducer;
  const fusg_medium& bg = *background;
  const double f0 = t.f0;
  auto grid_of = [&](int harmonic) -> const fusg_grid& { return d->grids[harmonic <= 2 ? 0 : harmonic - 2]; };
  auto count_of = [](const fusg_grid& g) { return int64_t(g.dims[0]) * g.dims[1] * g.dims[2]; };
  auto same_grid = [](const fusg_grid& a, const fusg_grid& b) {
    return a.dims[0] == b.dims[0] && a.dims[1] == b.dims[1] && a.dims[2] == b.dims[2] && a.lo[0] == b.lo[0] &&
           a.lo[1] == b.lo[1] && a.lo[2] == b.lo[2];
  };
  DevBufs ws{{}, s};
  // master map (c, beta) as one complex field; resample = one trilinear pass (src/vie.cpp:35-54)
  double2* master = nullptr;
  FUSG_TRY(ws.alloc(&master, size_t(count_of(*map_grid))));
  FUSG_CUDA_TRY(cudaMemcpyAsync(master, map_host, size_t(count_of(*map_grid)) * 16, cudaMemcpyHostToDevice, s));
  auto resample = [&](const fusg_grid& target, double2* out) -> fusg_status {
    if (same_grid(*map_grid, target) && map_grid->dx == target.dx) {
      FUSG_CUDA_TRY(cudaMemcpyAsync(out, master, size_t(count_of(target)) * 16, cudaMemcpyDeviceToDevice, s));
      return FUSG_OK;  // (interpolate onto the same grid is the identity)
    }
    return interpolate_dev(ctx, *map_grid, master, target, out, s);
  };
  // incident field and the first-harmonic scattering solve on the D_2 grid
  const fusg_grid& g2 = grid_of(1);
  const int64_t n2c = count_of(g2);
  double* src = nullptr;
  FUSG_TRY(upload_sources(t.points_host, t.n_points, &src, s));
  std::unique_ptr<double, void (*)(double*)> src_guard(src, [](double* p) { cudaFree(p); });
  double2 *inc = nullptr, *map2 = nullptr, *contrast = nullptr;
  FUSG_TRY(ws.alloc(&inc, size_t(n2c)));
  FUSG_TRY(ws.alloc(&map2, size_t(n2c)));
  fusg_wavenumber k1{};
  double norm = 1.0, amp1 = 0.0;
  FUSG_TRY(source_field_dev(ctx, t, bg, src, g2, inc, &k1, &norm, &amp1, s));
  if (source_normalization) *source_normalization = norm;
  FUSG_TRY(resample(g2, map2));
  FUSG_TRY(ws.alloc(&contrast, size_t(n2c)));
  FUSG_TRY(fusg_vie_contrast(ctx, reinterpret_cast<const double*>(map2), n2c, &bg, f0, 1,
                             reinterpret_cast<double*>(contrast), nullptr));
  fusg_status st = FUSG_OK;
  double2* p1 = reinterpret_cast<double2*>(out_dev[0]);
  std::vector<double> hist;
  int it = 0;
  if (all_zero_dev(contrast, n2c, ctx, s, &st)) {
    FUSG_TRY(st);
    FUSG_CUDA_TRY(cudaMemcpyAsync(p1, inc, size_t(n2c) * 16, cudaMemcpyDeviceToDevice, s));
  } else {
    FUSG_TRY(st);
    fusg_kernel* K1 = nullptr;
    fusg_grid gk = g2;
    gk.harmonic = 1;
    FUSG_TRY(fusg_kernel_create(ctx, &gk, &k1, d->pad_small_primes, &K1));
    st = solve_vie_dev(K1, inc, contrast, vie->tol, vie->max_iter, vie->restart, p1, hist, &it, s);
    fusg_kernel_destroy(K1);
    FUSG_TRY(st);
  }
  for (int i = 2; i <= nh; ++i) {
    fusg_stage_timing row{};
    row.harmonic = i;
    const fusg_grid& grid = grid_of(i);
    const int64_t count = count_of(grid);
    row.voxels = uint64_t(count);
    DevBufs stage{{}, s};
    std::vector<const double2*> lower;
    for (int m = 1; m <= i - 1; ++m) {
      const double2* pm = reinterpret_cast<const double2*>(out_dev[m - 1]);
      if (same_grid(grid_of(m), grid)) {
        lower.push_back(pm);
        continue;
      }
      double2* tmp = nullptr;
      FUSG_TRY(stage.alloc(&tmp, size_t(count)));
      FUSG_TRY(interpolate_dev(ctx, grid_of(m), pm, grid, tmp, s));
      lower.push_back(tmp);
    }
    double2 *map_i = nullptr, *products = nullptr, *conv = nullptr, *rhs = nullptr, *ci = nullptr;
    FUSG_TRY(stage.alloc(&map_i, size_t(count)));
    FUSG_TRY(resample(grid, map_i));
    fusg_wavenumber ki{};
    FUSG_TRY(fusg_complex_wavenumber(&bg, f0, i, &ki));
    // quadratic products without the material prefactor (sum_m p_m p_{i-m}, coefficient 1)
    FUSG_TRY(stage.alloc(&products, size_t(count)));
    FUSG_TRY(rhs_dev(ctx, i, lower.data(), count, 1.0, products, s));
    fusg_kernel* K = nullptr;
    fusg_grid gi = grid;
    gi.harmonic = i;
    FUSG_TRY(fusg_kernel_create(ctx, &gi, &ki, d->pad_small_primes, &K));
    std::unique_ptr<fusg_kernel, fusg_status (*)(fusg_kernel*)> kguard(K, fusg_kernel_destroy);
    FUSG_TRY(stage.alloc(&conv, size_t(count)));
    FUSG_TRY(volume_potential_apply(K, products, conv, 1.0, s));
    double2* pi = reinterpret_cast<double2*>(out_dev[i - 1]);
    FUSG_TRY(stage.alloc(&rhs, size_t(count)));
    vie_rhs_kernel<<<blocks_for(count), 256, 0, s>>>(map_i, conv, count, ki.omega, double(i) * double(i), bg.rho0, rhs);
    ctx->launches++;
    FUSG_LAUNCH_CHECK("vie_rhs_kernel");
    FUSG_TRY(stage.alloc(&ci, size_t(count)));
    FUSG_TRY(fusg_vie_contrast(ctx, reinterpret_cast<const double*>(map_i), count, &bg, f0, i,
                               reinterpret_cast<double*>(ci), nullptr));
    if (all_zero_dev(ci, count, ctx, s, &st)) {
      FUSG_TRY(st);
      FUSG_CUDA_TRY(cudaMemcpyAsync(pi, rhs, size_t(count) * 16, cudaMemcpyDeviceToDevice, s));
    } else {
      FUSG_TRY(st);
      FUSG_TRY(solve_vie_dev(K, rhs, ci, vie->tol, vie->max_iter, vie->restart, pi, hist, &it, s));
    }
    if (timings) timings[i - 2] = row;
  }
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return FUSG_OK;
}

}  // extern "C"
