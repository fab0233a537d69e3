// Pass C of the apply at padded z length 768 = 3 x 256 (the nested cascade's z for Nz <= 384):
// one CTA of three warps runs two lines; warp r owns residue r of both, its half-warp h line h,
// and each half-warp computes a 256-point sub-transform as 16 x 16 (16 values per lane, one
// shared-memory exchange per direction, no shuffles).
//
// Forward (decimation in frequency by 3; x[n] = 0 for n >= 384, the zero padding):
//   X[3k' + r] = DFT256_k'( y_r ),  y_r[m] = W768^(m r) (x[m] + W3^r x[m + 256]),  m < 256
// (x[m + 256] only for m < 128, x[m + 512] is padding).  With m = 16 n1 + l (l = lane & 15):
// stage A is a radix 16 over n1 in registers, the twiddle W768^(l r) W256^(l k1) (r16_twiddle_u),
// the exchange hands lane k1 the 16 values Y[k1][l], stage B a radix 16 over l, so lane k1 holds
// X[3 (k1 + 16 k2) + r] in register k2; the slot part W48^(n1 r) of the input twiddle is a
// constant-bank value (residue 0 skips it).  The spectrum is multiplied by the folded K^ row
// (index j or 768 - j), the inverse retraces the steps (decimation in time by 3, cropped to
// n < 384), and the three t_r rows of each line meet in shared memory:
//   x[n'] = t0 + t1 + t2,  x[n' + 256] = t0 + W3^-1 t1 + W3^-2 t2  (n' < 128).
#include <algorithm>
#include <cstdlib>

#include "r16.cuh"

namespace fusg {

__constant__ double2 c_w48h[48];  // W48^j = W768^(16 j) (the twiddle table's long-double values)

// exchange buffers as 16 rows of 17 entries (conflict-free for both patterns, every offset an
// immediate) instead of the XOR-swizzled [16][16] (FUSG_H3_PAD=0)
#ifndef FUSG_H3_PAD
#define FUSG_H3_PAD 1
#endif
struct H3Smem {
  static constexpr int XH = FUSG_H3_PAD ? 16 * 17 : 256;  // exchange buffer of one half-warp
  static constexpr int XB = 0;            // [2 r + h][XH] exchange buffers, then the t_r rows
  static constexpr int KB = 6 * XH;       // folded K^ rows of the two lines (385 each, stride 386)
  static constexpr int TW = KB + 2 * 386; // [4][16] W256^(l 2^j)
  static constexpr int US = TW + 64;      // [3][16] W768^(l r)
  static constexpr int SB = US + 48;      // staged input rows of the two lines (<= 384 each)
  static constexpr int END = SB + 2 * 384;
  // + 2 mbarriers + [2][2] output-row offsets (the staging thread leaves them for the pair it stages:
  // the other threads skip the line -> (ky, kx) divisions)
  static constexpr size_t BYTES = size_t(END) * sizeof(double2) + 6 * sizeof(uint64_t);
};

__device__ __forceinline__ int ex16(int row, int col) { return FUSG_H3_PAD ? row * 17 + col : row * 16 + (col ^ (row & 7)); }

__global__ void __launch_bounds__(96, 4) conv_r16x3h(WArgs a) {
  constexpr int HZ = 385;
  extern __shared__ double2 sm[];
  const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = lane & 15, h = lane >> 4;
  double2* const xb = sm + H3Smem::XB;
  double2* const xr = xb + H3Smem::XH * (2 * r + h);  // this half-warp's exchange buffer / t_r row
  double2* const kb = sm + H3Smem::KB + 386 * h;
  double2* const sb = sm + H3Smem::SB;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + H3Smem::END);
  for (int e = threadIdx.x; e < 64; e += 96) sm[H3Smem::TW + e] = __ldg(a.tw + (((3 * (e & 15)) << (e >> 4)) % 768));
  for (int e = threadIdx.x; e < 48; e += 96) sm[H3Smem::US + e] = __ldg(a.tw + (e & 15) * (e >> 4));
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    mbar_init_fence();
  }
  __syncthreads();
  const double2 u = sm[H3Smem::US + 16 * r + l];
  const double2 w1 = sm[H3Smem::TW + l], w2 = sm[H3Smem::TW + 16 + l];
  const double2 w4 = sm[H3Smem::TW + 32 + l], w8 = sm[H3Smem::TW + 48 + l];
  const double c3 = r == 0 ? 1.0 : -0.5;
  const double s3 = r == 0 ? 0.0 : r == 1 ? -0.8660254037844386467637 : 0.8660254037844386467637;
  const int64_t nlines = int64_t(a.n_inner) * a.n_outer;
  const int64_t npairs = (nlines + 1) / 2;
  const int64_t stride = gridDim.x;
  const bool mirror = a.n_outer == a.ko.Px;
  auto coords = [&](int64_t line, int& ky, int& kx) { conv_line_coords(unsigned(line), a.ko, a.n_inner, mirror, ky, kx); };
  const int nv = a.in_nvalid, onv = a.out_nvalid;
  auto prefetch_in = [&](int64_t pr, unsigned slot) {  // thread 0: both rows of pair pr, one barrier
    int64_t* const orow = reinterpret_cast<int64_t*>(bars + 2);  // [slot][t] output-row offsets
    if (pr < npairs) {
      const int nl = (2 * pr + 1 < nlines) ? 2 : 1;
      const unsigned row = unsigned(nv) * sizeof(double2);
      refill_fence();
      mbar_expect_tx(bars, row * nl);
      for (int t = 0; t < nl; ++t) {
        int ky, kx;
        coords(2 * pr + t, ky, kx);
        orow[2 * slot + t] = ky * a.out_si + int64_t(kx) * a.out_sk;
        bulk_g2s(sb + 384 * t, a.in + ky * a.in_si + int64_t(kx) * a.in_sk, row, bars);
      }
    }
  };
  auto prefetch_k = [&](int64_t pr) {
    if (pr < npairs) {
      const int nl = (2 * pr + 1 < nlines) ? 2 : 1;
      refill_fence();
      mbar_expect_tx(bars + 1, unsigned(HZ * sizeof(double2)) * nl);
      for (int t = 0; t < nl; ++t) {
        int ky, kx;
        coords(2 * pr + t, ky, kx);
        bulk_g2s(sm + H3Smem::KB + 386 * t, a.ko.line(ky, kx), HZ * sizeof(double2), bars + 1);
      }
    }
  };
  int64_t pr = blockIdx.x;
  if (threadIdx.x == 0) {
    prefetch_in(pr, 0);
    prefetch_k(pr);
  }
  unsigned ph = 0;
  for (; pr < npairs; pr += stride, ph ^= 1) {
    const bool ok1 = 2 * pr + 1 < nlines;  // the pair's second line exists
    double2 v[16];
    mbar_wait(bars, ph);
    {  // y_r[16 n1 + l] without its lane twiddle (half-warp h: line h; a missing line reads zeros)
      const double2* row = sb + 384 * h;
      const bool live = h == 0 || ok1;
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) {
        const int m = 16 * n1 + l;
        double2 x0 = (live && m < nv) ? row[m] : make_double2(0.0, 0.0);
        if (n1 < 8) {
          const double2 x1 = (live && m + 256 < nv) ? row[m + 256] : make_double2(0.0, 0.0);
          x0 = make_double2(fma(c3, x1.x, fma(-s3, x1.y, x0.x)), fma(c3, x1.y, fma(s3, x1.x, x0.y)));
        }
        v[n1] = x0;
      }
    }
    __syncthreads();  // both staged rows read by all three warps: refill
    if (threadIdx.x == 0) prefetch_in(pr + stride, ph ^ 1u);
    // forward: slot twiddle, stage A, lane twiddle, exchange, stage B
    if (r == 1) {
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) v[n1] = cmul(v[n1], c_w48h[n1]);
    } else if (r == 2) {
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) v[n1] = cmul(v[n1], c_w48h[2 * n1]);
    }
    dft16<false>(v);
    r16_twiddle_u<false>(v, u, w1, w2, w4, w8);
#pragma unroll
    for (int k = 0; k < 16; ++k) xr[ex16(k, l)] = v[k];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = xr[ex16(l, q)];
    dft16<false>(v);
    // lane l (= k1) register k2 holds X[3 (l + 16 k2) + r]: times the folded K^ row
    mbar_wait(bars + 1, ph);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const int j = 3 * (l + 16 * k2) + r;
      v[k2] = cmul(v[k2], kb[j <= 384 ? j : 768 - j]);
    }
    __syncthreads();  // both K^ rows read: refill
    if (threadIdx.x == 0) prefetch_k(pr + stride);
    // inverse: stage B, exchange back, conjugate lane twiddle, stage A, conjugate slot twiddle
    dft16<true>(v);
#pragma unroll
    for (int q = 0; q < 16; ++q) xr[ex16(l, q)] = v[q];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xr[ex16(k, l)];
    r16_twiddle_u<true>(v, u, w1, w2, w4, w8);
    dft16<true>(v);
    if (r == 1) {
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) v[n1] = cmulc(v[n1], c_w48h[n1]);
    } else if (r == 2) {
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) v[n1] = cmulc(v[n1], c_w48h[2 * n1]);
    }
    __syncwarp();  // every lane has read its exchange slots
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) xr[16 * n1 + l] = v[n1];
    __syncthreads();
    // recombination: 2 lines x 256 positions over the CTA's 96 threads
    constexpr double kS3 = 0.8660254037844386467637;
    double2* outs[2];
#pragma unroll
    for (int t = 0; t < 2; ++t)  // offsets left by thread 0 when it staged this pair (barriers in between)
      outs[t] = a.out + ((t == 0 || ok1) ? reinterpret_cast<const int64_t*>(bars + 2)[2 * ph + t] : 0);
    for (int e = threadIdx.x; e < 512; e += 96) {
      const int t = e >> 8, n = e & 255;
      if (t == 1 && !ok1) break;
      double2* out = outs[t];
      const double2 t0 = xb[H3Smem::XH * t + n], t1 = xb[H3Smem::XH * (2 + t) + n], t2 = xb[H3Smem::XH * (4 + t) + n];
      const double2 s = cadd(t1, t2);
      if (n < onv) {
        const double2 o = cadd(t0, s);
        out[n] = a.scale == 1.0 ? o : cscale(o, a.scale);
      }
      if (n + 256 < onv) {
        const double2 d = csub(t1, t2);
        const double2 o = make_double2(t0.x - 0.5 * s.x - kS3 * d.y, t0.y - 0.5 * s.y + kS3 * d.x);
        out[n + 256] = a.scale == 1.0 ? o : cscale(o, a.scale);
      }
    }
    // (the next pair's staging barrier orders these reads before its exchange writes)
  }
}

// pass C at L = 768 (conv_r16x3h): 1 launched, 0 not applicable, -1 error
int launch_conv_r16x3h(fusg_ctx* ctx, const WArgs& a, cudaStream_t s) {
  static const bool on = [] {  // FUSG_CONV_768=0 keeps the one-warp radix (8, 4, 3, 8) pass C
    const char* e = getenv("FUSG_CONV_768");
    return !(e && atoi(e) == 0);
  }();
  if (!on || a.in_nvalid < 1 || a.in_nvalid > 384 || a.out_nvalid > 384) return 0;
  const int64_t nl = int64_t(a.n_inner) * a.n_outer;
  if (nl >= (int64_t(1) << 31)) return 0;
  static std::atomic<uint64_t> attr_mask{0};
  if (!once_per_device(attr_mask, [] {
        double2 hw[48];
        for (int e = 0; e < 48; ++e) {  // the twiddle table's expression (L = 768, m = 16 e)
          const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (16 * e) / 768;
          hw[e] = make_double2(double(cosl(ang)), double(sinl(ang)));
        }
        return cudaMemcpyToSymbol(c_w48h, hw, sizeof(hw)) == cudaSuccess &&
               cudaFuncSetAttribute(conv_r16x3h, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(H3Smem::BYTES)) == cudaSuccess;
      })) {
    set_error(FUSG_CUDA, "pass C (768 = 3 x 256): cannot configure the kernel");
    return -1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_r16x3h, 96, H3Smem::BYTES) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  static const int waves = [] {  // CTAs per resident slot; 323^3 cascade grid: 4 / 16 / 64 -> 1.995 / 1.967 / 2.006 ms
    const char* e = getenv("FUSG_X3H_WAVES");
    return e ? std::max(1, atoi(e)) : 16;
  }();
  const int64_t pairs = (nl + 1) / 2;
  const int64_t grid = std::min<int64_t>(pairs, int64_t(per_sm) * ctx->num_sms * waves);
  WArgs b = a;
  b.ko.quad = 1;
  conv_r16x3h<<<unsigned(grid), 96, H3Smem::BYTES, s>>>(b);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "pass C (768 = 3 x 256)");
    return -1;
  }
  return 1;
}

}  // namespace fusg
